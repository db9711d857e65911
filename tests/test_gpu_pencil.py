"""Pencil and y-slab decompositions nproc = (1, Py, Pz) (north_star "slab/pencil decomposition"; SURVEY
8(e): pencils, and 2-D grids split along y): the in-process group (pitched device copies of the 2-row y halos,
then the z halos, which carry the edge ghosts along) and the NCCL path with the rank as its own y (and z)
neighbour must reproduce the undecomposed run bit for bit -- same per-cell arithmetic, same global dt -- and so
match the oracle as the undecomposed run does."""
import os

import numpy as np
import pytest

from cgks_inputs import cases, random_smooth

pytestmark = pytest.mark.gpu


def _single(case, scheme, nl, steps, L=None, **kw):
    from paper_2508_19911_b200 import Solver
    S = Solver.from_case(case, scheme=scheme, nonlinear=nl, **kw)
    S.set_state(case.Q, case.G)
    if L is not None:
        S.set_lines(L)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    Lo = S.get_lines() if L is not None else None
    S.close()
    return Q, G, t, Lo


def _group(case, scheme, nl, steps, Py, Pz, L=None, **kw):
    from paper_2508_19911_b200 import Solver, decompose_pencil, step_group
    P = Py * Pz
    solvers, boxes = [], []
    for r in range(P):
        S = Solver.from_case(case, scheme=scheme, nonlinear=nl, nproc=(1, Py, Pz), rank=r, **kw)
        off, nloc, nbr = decompose_pencil(case.n, (1, Py, Pz), r)
        assert S.local_shape == (tuple(off), tuple(nloc))
        y0, ny, z0, nz = off[1], nloc[1], off[2], nloc[2]
        S.set_state(np.ascontiguousarray(case.Q[:, z0:z0 + nz, y0:y0 + ny]),
                    np.ascontiguousarray(case.G[:, :, z0:z0 + nz, y0:y0 + ny]))
        if L is not None:
            S.set_lines(np.ascontiguousarray(L[:, :, z0:z0 + nz, y0:y0 + ny]))
        solvers.append(S)
        boxes.append((y0, ny, z0, nz))
    step_group(solvers, steps)
    Q = np.zeros_like(case.Q)
    G = np.zeros_like(case.G)
    Lo = np.zeros_like(L) if L is not None else None
    for S, (y0, ny, z0, nz) in zip(solvers, boxes):
        q, g = S.get_state()
        Q[:, z0:z0 + nz, y0:y0 + ny] = q
        G[:, :, z0:z0 + nz, y0:y0 + ny] = g
        if L is not None:
            Lo[:, :, z0:z0 + nz, y0:y0 + ny] = S.get_lines()
    t = solvers[0].get_time()
    for S in solvers:
        S.close()
    return Q, G, t, Lo


@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("Py,Pz", [(2, 1), (2, 2), (3, 2), (4, 1)])
def test_pencil_group_bitwise(scheme, nl, Py, Pz):
    case = random_smooth((20, 24, 16), seed=8, jump=0.4 if nl else 0.0)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _single(case, scheme, nl, 5, **kw)
    Qp, Gp, tp, _ = _group(case, scheme, nl, 5, Py, Pz, **kw)
    assert t1 == tp
    assert np.array_equal(Q1, Qp)
    if scheme == 1:
        assert np.array_equal(G1, Gp)


@pytest.mark.parametrize("scheme", [1, 0])
def test_yslab_2d_box_bitwise(scheme):
    # BASELINE configs[3] shape (inflow / outflow in x, periodic y), 2-D: the only possible split is along y
    case = cases.shock_vortex(64, 32)
    Q1, G1, t1, _ = _single(case, scheme, 1, 6)
    Qp, Gp, tp, _ = _group(case, scheme, 1, 6, 4, 1)
    assert t1 == tp
    assert np.array_equal(Q1, Qp)
    if scheme == 1:
        assert np.array_equal(G1, Gp)


def test_yslab_2d_vortex_bitwise():
    case = cases.vortex(40)
    Q1, G1, t1, _ = _single(case, 1, 0, 5)
    Qp, Gp, tp, _ = _group(case, 1, 0, 5, 2, 1)
    assert t1 == tp and np.array_equal(Q1, Qp) and np.array_equal(G1, Gp)


@pytest.mark.parametrize("nl", [0, 1])
def test_pencil_group_lines_bitwise(nl):
    case = random_smooth((16, 16, 16), seed=9, jump=0.4 if nl else 0.0)
    rng = np.random.default_rng(5)
    L = case.G[np.array([1, 2, 1, 2, 2, 0, 2, 0, 0, 1, 0, 1])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
    kw = dict(mu=1e-3, Pr=0.72, lines=1)
    Q1, G1, t1, L1 = _single(case, 1, nl, 4, L=L, **kw)
    Qp, Gp, tp, Lp = _group(case, 1, nl, 4, 2, 2, L=L, **kw)
    assert t1 == tp
    assert np.array_equal(Q1, Qp) and np.array_equal(G1, Gp) and np.array_equal(L1, Lp)


def test_pencil_tgv32_vs_oracle():
    # SURVEY D4 option 2 for the pencil layout: oracle parity of a decomposed TGV (2 x 4 pencils), 10 steps
    import oracle
    from parity_util import hmin, rel_linf, worst
    case = cases.tgv(32)
    Qp, Gp, tp, _ = _group(case, 1, 0, 10, 2, 4)
    prob = oracle.Problem(**case.problem_kwargs(), scheme=1, time_scheme=2)
    Qo, Go, to, _, rc = oracle.run(prob, case.Q, case.G, 10)
    assert rc == 0
    assert abs(tp[0] - to) <= 1e-12 * abs(to)
    k, v = worst(rel_linf(Qp, Qo, Gp, Go, h=hmin(case), nsteps=10, tol=1e-10))
    assert v <= 1e-10, (k, v)


def _nccl_self(case, scheme, nl, steps, env, L=None, **kw):
    import torch  # noqa: F401  (loads the libnccl.so.2 the library binds at run time)
    from paper_2508_19911_b200 import Solver, nccl_unique_id
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        S = Solver.from_case(case, scheme=scheme, nonlinear=nl, nccl_id=nccl_unique_id(), **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    S.set_state(case.Q, case.G)
    if L is not None:
        S.set_lines(L)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    Lo = S.get_lines() if L is not None else None
    S.close()
    return Q, G, t, Lo


@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
def test_nccl_self_y_and_z_bitwise(scheme, nl):
    # one NCCL rank as its own y AND z neighbour (test hook CGKS_TEST_SELF_Y): pack, ncclSend/Recv, unpack of the
    # y strips, then the z planes with the edge ghosts, captured into the step graph
    case = random_smooth((20, 12, 16), seed=8, jump=0.4 if nl else 0.0)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _single(case, scheme, nl, 5, **kw)
    Qn, Gn, tn, _ = _nccl_self(case, scheme, nl, 5, {"CGKS_TEST_SELF_Y": "1"}, **kw)
    assert t1 == tn and np.array_equal(Q1, Qn)
    if scheme == 1:
        assert np.array_equal(G1, Gn)


def test_nccl_self_y_lines_bitwise():
    case = random_smooth((16, 12, 16), seed=9, jump=0.4)
    rng = np.random.default_rng(5)
    L = case.G[np.array([1, 2, 1, 2, 2, 0, 2, 0, 0, 1, 0, 1])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
    kw = dict(mu=1e-3, Pr=0.72, lines=1)
    Q1, G1, t1, L1 = _single(case, 1, 1, 4, L=L, **kw)
    Qn, Gn, tn, Ln = _nccl_self(case, 1, 1, 4, {"CGKS_TEST_SELF_Y": "1"}, L=L, **kw)
    assert t1 == tn and np.array_equal(Q1, Qn) and np.array_equal(G1, Gn) and np.array_equal(L1, Ln)


def test_nccl_self_2d_yslab_bitwise():
    # a 2-D grid with an NCCL id: the y path with the rank as its own neighbour (box BCs in x)
    case = cases.shock_vortex(64, 32)
    Q1, G1, t1, _ = _single(case, 1, 1, 6)
    Qn, Gn, tn, _ = _nccl_self(case, 1, 1, 6, {})
    assert t1 == tn and np.array_equal(Q1, Qn) and np.array_equal(G1, Gn)


def test_nccl_self_y_chunked_bitwise():
    # y halo + z-chunked stages (the chunk's ghost planes come from the z exchange after the y exchange)
    case = random_smooth((20, 12, 16), seed=8)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _single(case, 1, 0, 4, **kw)
    Qn, Gn, tn, _ = _nccl_self(case, 1, 0, 4, {"CGKS_TEST_SELF_Y": "1", "CGKS_CHUNK": "5"}, **kw)
    assert t1 == tn and np.array_equal(Q1, Qn) and np.array_equal(G1, Gn)


def test_nccl_self_y_stretched_bitwise():
    # stretched tensor-product mesh (NEXT-4) through the y + z self halos: the ghost rows / planes take the
    # periodic images' widths, as the plain context's wrap does
    from cgks_inputs import stretched_nodes
    case = random_smooth((16, 12, 16), seed=3)
    nodes = tuple(stretched_nodes(case.n[a], case.lo[a], case.hi[a], 0.2) for a in range(3))
    kw = dict(mu=1e-3, Pr=0.72, nodes=nodes)
    Q1, G1, t1, _ = _single(case, 1, 0, 4, **kw)
    Qn, Gn, tn, _ = _nccl_self(case, 1, 0, 4, {"CGKS_TEST_SELF_Y": "1"}, **kw)
    assert t1 == tn and np.array_equal(Q1, Qn) and np.array_equal(G1, Gn)


def test_pencil_config_errors():
    # cgks_create refuses: a split x axis, rows not divisible by Py, fewer than 4 rows per rank, a bounded y axis
    from paper_2508_19911_b200 import CgksError, Solver
    case = random_smooth((16, 12, 16), seed=1)
    for nproc in [(2, 1, 1), (1, 5, 1), (1, 4, 1), (1, 2, 3)]:  # 12 rows: 5 does not divide, 4 leaves 3 rows; 16 planes / 3
        with pytest.raises(CgksError) as e:
            Solver.from_case(case, scheme=1, nproc=nproc, rank=0)
        assert e.value.code == 2  # CGKS_ERR_CONFIG
    sv = cases.shock_vortex(64, 32)  # x is bounded: only y can be split, and y must be periodic
    bc = ((0, 0), (1, 2), (0, 0))
    with pytest.raises(CgksError):
        Solver(sv.n, sv.lo, sv.hi, scheme=1, bc=bc, bc_state=sv.bc_state, nproc=(1, 2, 1), rank=0)
