"""z-slab decomposition on one GPU: P contexts of an in-process decomposition (halo copies,
shared dt; cgks_step_group) must reproduce the undecomposed run bit for bit, because every
cell and face is computed by the same code from the same inputs with the same global dt
(BASELINE configs[4] strategy for the 512^3 runs)."""
import numpy as np
import pytest

from cgks_inputs import random_smooth, tgv

pytestmark = pytest.mark.gpu


def _run_single(case, scheme, nl, steps, **kw):
    from paper_2508_19911_b200 import Solver
    S = Solver.from_case(case, scheme=scheme, nonlinear=nl, **kw)
    S.set_state(case.Q, case.G)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    S.close()
    return Q, G, t


def _run_group(case, scheme, nl, steps, P, **kw):
    from paper_2508_19911_b200 import Solver, decompose, step_group
    solvers = []
    for r in range(P):
        S = Solver.from_case(case, scheme=scheme, nonlinear=nl, nproc=(1, 1, P), rank=r, **kw)
        off, nloc, _ = decompose(case.n, (1, 1, P), r)
        z0, nz = off[2], nloc[2]
        S.set_state(np.ascontiguousarray(case.Q[:, z0:z0 + nz]), np.ascontiguousarray(case.G[:, :, z0:z0 + nz]))
        solvers.append(S)
    step_group(solvers, steps)
    Q = np.concatenate([s.get_state()[0] for s in solvers], axis=1)
    G = np.concatenate([s.get_state()[1] for s in solvers], axis=2)
    t = solvers[0].get_time()
    for s in solvers:
        s.close()
    return Q, G, t


@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("P", [2, 4])
def test_group_decomposition_bitwise(scheme, nl, P):
    case = random_smooth((20, 12, 16), seed=8, jump=0.4 if nl else 0.0)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, t1 = _run_single(case, scheme, nl, 5, **kw)
    Qp, Gp, tp = _run_group(case, scheme, nl, 5, P, **kw)
    assert t1 == tp
    assert np.array_equal(Q1, Qp)
    if scheme == 1:
        assert np.array_equal(G1, Gp)


def test_group_decomposition_tgv128_bitwise():
    case = tgv(128)
    Q1, G1, t1 = _run_single(case, 1, 0, 2)
    Qp, Gp, tp = _run_group(case, 1, 0, 2, 8)
    assert t1 == tp
    assert np.array_equal(Q1, Qp) and np.array_equal(G1, Gp)


def test_single_step_refused_for_group_member():
    from paper_2508_19911_b200 import CgksError, Solver
    case = random_smooth((8, 8, 8), seed=1)
    S = Solver.from_case(case, scheme=1, nproc=(1, 1, 2), rank=0)
    with pytest.raises(CgksError):
        S.step(1)
    S.close()
