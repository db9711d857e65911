"""The NCCL slab path on one GPU: a single rank given an ncclUniqueId runs the z-slab machinery with
itself as both z neighbours (ghost planes, NCCL send/recv halo exchange = the periodic wrap, dt
allreduce, the exchange overlapped with the interior reconstruction on a second stream, all captured
in the step graph).  Same kernels and per-cell arithmetic as the periodic single-rank context, so
the two runs agree bit for bit."""
import numpy as np
import pytest

from cgks_inputs import random_smooth

pytestmark = pytest.mark.gpu


def _run(case, scheme, nl, steps, nccl, L=None, **kw):
    import torch  # noqa: F401  (loads the libnccl.so.2 the library binds at run time)
    from paper_2508_19911_b200 import Solver, nccl_unique_id
    S = Solver.from_case(case, scheme=scheme, nonlinear=nl, nccl_id=nccl_unique_id() if nccl else None, **kw)
    S.set_state(case.Q, case.G)
    if L is not None:
        S.set_lines(L)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    Lo = S.get_lines() if L is not None else None
    S.close()
    return Q, G, t, Lo


@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("graph", [1, 0])
@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
def test_nccl_self_halo_bitwise(scheme, nl, overlap, graph, monkeypatch):
    if not overlap:
        monkeypatch.setenv("CGKS_NO_OVERLAP", "1")
    if not graph:
        monkeypatch.setenv("CGKS_NO_GRAPH", "1")
    case = random_smooth((16, 12, 10), seed=4, jump=0.4 if nl else 0.0)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _run(case, scheme, nl, 4, False, **kw)
    Q2, G2, t2, _ = _run(case, scheme, nl, 4, True, **kw)
    assert t1 == t2
    assert np.array_equal(Q1, Q2)
    if scheme == 1:
        assert np.array_equal(G1, G2)


def test_nccl_self_halo_lines_bitwise():
    case = random_smooth((16, 12, 10), seed=6)
    rng = np.random.default_rng(2)
    L = case.G[np.array([0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
    kw = dict(mu=1e-3, Pr=0.72, lines=1)
    Q1, G1, t1, L1 = _run(case, 1, 0, 3, False, L=L, **kw)
    Q2, G2, t2, L2 = _run(case, 1, 0, 3, True, L=L, **kw)
    assert t1 == t2 and np.array_equal(Q1, Q2) and np.array_equal(G1, G2) and np.array_equal(L1, L2)


def test_nccl_self_halo_stretched_bitwise():
    # stretched nodes on all three axes: the slab path's ghost-plane widths come from the global
    # node arrays (periodic images), so the result equals the plain periodic context bit for bit
    from cgks_inputs import stretched_nodes
    case = random_smooth((16, 12, 10), seed=7, jump=0.3)
    nodes = (stretched_nodes(16, case.lo[0], case.hi[0], 0.2), stretched_nodes(12, case.lo[1], case.hi[1], 0.15),
             stretched_nodes(10, case.lo[2], case.hi[2], 0.25))
    kw = dict(mu=1e-3, Pr=0.72, nodes=nodes)
    Q1, G1, t1, _ = _run(case, 1, 1, 3, False, **kw)
    Q2, G2, t2, _ = _run(case, 1, 1, 3, True, **kw)
    assert t1 == t2 and np.array_equal(Q1, Q2) and np.array_equal(G1, G2)


def test_nccl_self_halo_async_pipeline():
    # the asynchronous calls on the NCCL slab path (exchange on the halo stream, copies on the copy
    # streams) give the synchronous results bit for bit
    import torch
    from paper_2508_19911_b200 import Solver, nccl_unique_id
    case = random_smooth((16, 12, 10), seed=5, jump=0.3)
    kw = dict(mu=1e-3, Pr=0.72)
    Q1, G1, _, _ = _run(case, 1, 1, 4, False, **kw)
    S = Solver.from_case(case, scheme=1, nonlinear=1, nccl_id=nccl_unique_id(), **kw)
    qi, gi = torch.from_numpy(case.Q).pin_memory(), torch.from_numpy(case.G).pin_memory()
    qo, go = torch.zeros_like(qi).pin_memory(), torch.zeros_like(gi).pin_memory()
    S.set_state_async(qi, gi)
    S.step_async(4)
    S.get_state_async(qo, go)
    S.sync()
    S.close()
    assert np.array_equal(qo.numpy(), Q1) and np.array_equal(go.numpy(), G1)


@pytest.mark.parametrize("graph", [1, 0])
def test_nccl_peer_failure_stops_at_the_same_step(graph, monkeypatch):
    """a rank that fails posts its error code through the dt allreduce-min; a healthy rank
    then fails the same step with the same code and keeps the state of the last completed step.  The
    peer is emulated by the CGKS_TEST_PEER_FAIL_STEP hook of the error-poison kernel (one GPU per call)."""
    import torch  # noqa: F401
    from paper_2508_19911_b200 import CgksError, Solver, nccl_unique_id
    if not graph:
        monkeypatch.setenv("CGKS_NO_GRAPH", "1")
    case = random_smooth((16, 12, 10), seed=4)
    kw = dict(mu=1e-3, Pr=0.72)
    Q2, G2, t2, _ = _run(case, 1, 0, 2, False, **kw)
    monkeypatch.setenv("CGKS_TEST_PEER_FAIL_STEP", "2")
    S = Solver.from_case(case, scheme=1, nccl_id=nccl_unique_id(), **kw)
    S.set_state(case.Q, case.G)
    with pytest.raises(CgksError) as e:
        S.step(5)
    assert e.value.code == 3
    assert "another rank" in S.last_error()
    t, steps, _ = S.get_time()
    assert steps == 2 and t == t2[0]
    Q, G = S.get_state()
    assert np.array_equal(Q, Q2) and np.array_equal(G, G2)
    S.close()
