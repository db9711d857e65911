"""z-slab decomposition on one GPU: P contexts of an in-process decomposition (halo copies,
shared dt; cgks_step_group) must reproduce the undecomposed run bit for bit, because every
cell and face is computed by the same code from the same inputs with the same global dt
(BASELINE configs[4] strategy for the 512^3 runs)."""
import numpy as np
import pytest

from cgks_inputs import random_smooth, tgv

pytestmark = pytest.mark.gpu


def _run_single(case, scheme, nl, steps, L=None, **kw):
    from paper_2508_19911_b200 import Solver
    S = Solver.from_case(case, scheme=scheme, nonlinear=nl, **kw)
    S.set_state(case.Q, case.G)
    if L is not None:
        S.set_lines(L)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    Lout = S.get_lines() if L is not None else None
    S.close()
    return (Q, G, t) if L is None else (Q, G, t, Lout)


def _run_group(case, scheme, nl, steps, P, L=None, **kw):
    from paper_2508_19911_b200 import Solver, decompose, step_group
    solvers = []
    for r in range(P):
        S = Solver.from_case(case, scheme=scheme, nonlinear=nl, nproc=(1, 1, P), rank=r, **kw)
        off, nloc, _ = decompose(case.n, (1, 1, P), r)
        z0, nz = off[2], nloc[2]
        S.set_state(np.ascontiguousarray(case.Q[:, z0:z0 + nz]), np.ascontiguousarray(case.G[:, :, z0:z0 + nz]))
        if L is not None:
            S.set_lines(np.ascontiguousarray(L[:, :, z0:z0 + nz]))
        solvers.append(S)
    step_group(solvers, steps)
    Q = np.concatenate([s.get_state()[0] for s in solvers], axis=1)
    G = np.concatenate([s.get_state()[1] for s in solvers], axis=2)
    Lout = np.concatenate([s.get_lines() for s in solvers], axis=2) if L is not None else None
    t = solvers[0].get_time()
    for s in solvers:
        s.close()
    return (Q, G, t) if L is None else (Q, G, t, Lout)


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


@pytest.mark.parametrize("nl", [0, 1])
def test_group_decomposition_lines_bitwise(nl):
    # line DOFs (NEXT-1): their 2-plane halos travel with the state's, so the decomposed run is
    # again bit-identical to the single-context one
    case = random_smooth((16, 12, 20), seed=9, jump=0.4 if nl else 0.0)
    rng = np.random.default_rng(5)
    L = case.G[np.array([1, 2, 1, 2, 2, 0, 2, 0, 0, 1, 0, 1])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
    kw = dict(mu=1e-3, Pr=0.72, lines=1)
    Q1, G1, t1, L1 = _run_single(case, 1, nl, 5, L=L, **kw)
    Qp, Gp, tp, Lp = _run_group(case, 1, nl, 5, 4, L=L, **kw)
    assert t1 == tp
    assert np.array_equal(Q1, Qp) and np.array_equal(G1, Gp) and np.array_equal(L1, Lp)


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


def test_group_refuses_stretched_meshes():
    from paper_2508_19911_b200 import CgksError, Solver, step_group
    from cgks_inputs import stretched_nodes
    case = random_smooth((8, 8, 8), seed=1)
    nodes = (stretched_nodes(8, 0.0, 1.0, 0.2), None, None)
    S = [Solver.from_case(case, scheme=1, nproc=(1, 1, 2), rank=r, nodes=nodes) for r in range(2)]
    with pytest.raises(CgksError) as e:
        step_group(S, 1)
    assert e.value.code == 2 and "stretched" in str(e.value)
    for s in S:
        s.close()
