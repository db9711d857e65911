"""Small-grid workload for compute-sanitizer (racecheck / synccheck / memcheck).

Covers every kernel family on 16 x 12 x 10 grids (TMA tiles, mbarriers, shared-memory parking slots,
cp.async wrap tiles): CGKS-5th linear and GENO, GKS-2nd (Venkatakrishnan), line DOFs, box
inflow/outflow, a stretched mesh, the asynchronous pipeline, the in-process slab group and the
NCCL slab path with a self neighbour.  Run one tool per process:

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch  # noqa: F401  (libnccl.so.2 for the NCCL slab case)
    from cgks_inputs import random_smooth, shock_vortex, stretched_nodes
    from paper_2508_19911_b200 import Solver, decompose, nccl_unique_id, step_group

    n = (16, 12, 10)
    case = random_smooth(n, seed=4, jump=0.3)
    runs = [("cgks5-linear", dict(scheme=1, nonlinear=0)),
            ("cgks5-geno", dict(scheme=1, nonlinear=1)),
            ("gks2-venkat", dict(scheme=0, nonlinear=1)),
            ("gks2-s2o4", dict(scheme=0, nonlinear=0, time_scheme=2)),
            ("cgks5-lines", dict(scheme=1, nonlinear=1, lines=1)),
            ("cgks5-box", dict(scheme=1, nonlinear=1, bc=((2, 2), (0, 0), (0, 0)))),
            ("cgks5-nccl-self", dict(scheme=1, nonlinear=1, nccl_id="new"))]
    for name, kw in runs:
        kw = dict(kw)
        if kw.get("nccl_id") == "new":
            kw["nccl_id"] = nccl_unique_id()
        S = Solver.from_case(case, mu=1e-3, Pr=0.72, **kw)
        S.set_state(case.Q, case.G)
        S.step(2)
        Q, G = S.get_state()
        assert np.all(np.isfinite(Q)), name
        S.close()
        print("ok", name, flush=True)
    # stretched tensor-product mesh
    nodes = (stretched_nodes(16, case.lo[0], case.hi[0], 0.2), None, None)
    S = Solver.from_case(case, scheme=1, nonlinear=0, mu=1e-3, Pr=0.72, nodes=nodes)
    S.set_state(case.Q, case.G)
    S.step(2)
    S.close()
    print("ok stretched", flush=True)
    # 2-D box (shock-vortex geometry)
    sv = shock_vortex(nx=32, ny=16)
    S = Solver.from_case(sv, scheme=1)
    S.set_state(sv.Q, sv.G)
    S.step(2)
    S.close()
    print("ok shock-vortex 2-D", flush=True)
    # asynchronous host pipeline
    S = Solver.from_case(case, scheme=1, nonlinear=1, mu=1e-3, Pr=0.72)
    Qh = torch.from_numpy(np.ascontiguousarray(case.Q)).pin_memory()
    Gh = torch.from_numpy(np.ascontiguousarray(case.G)).pin_memory()
    Qo = torch.empty_like(Qh).pin_memory()
    Go = torch.empty_like(Gh).pin_memory()
    for _ in range(3):
        S.set_state_async(Qh, Gh)
        S.step_async(1)
        S.get_state_async(Qo, Go)
    S.sync()
    S.close()
    print("ok async", flush=True)
    # in-process slab group, 2 slabs
    solvers = []
    for r in range(2):
        S = Solver.from_case(case, scheme=1, nonlinear=1, mu=1e-3, Pr=0.72, nproc=(1, 1, 2), rank=r)
        off, nloc, _ = decompose(case.n, (1, 1, 2), r)
        z0, nz = off[2], nloc[2]
        S.set_state(np.ascontiguousarray(case.Q[:, z0:z0 + nz]), np.ascontiguousarray(case.G[:, :, z0:z0 + nz]))
        solvers.append(S)
    step_group(solvers, 2)
    for S in solvers:
        S.close()
    print("ok group", flush=True)
    print("SANITIZE_RUN_DONE", flush=True)


if __name__ == "__main__":
    main()
