"""z-chunked stages (large grids): each stage passes over z-chunks of C planes with
the chunk's own reconstruction (planes k0-1 .. k0+C) and face buffers, the periodic z images in two
stored ghost planes per side.  Same kernels and per-cell arithmetic as the whole-slab stage, every face
computed once: the run must equal the unchunked one bit for bit.  CGKS_CHUNK=C forces the chunk size
(the automatic choice chunks only grids whose whole-slab buffers do not fit)."""
import numpy as np
import pytest

from cgks_inputs import random_smooth, stretched_nodes

pytestmark = pytest.mark.gpu


def _run(case, steps, chunk, monkeypatch, L=None, nccl=False, **kw):
    import torch  # noqa: F401  (libnccl.so.2 for the NCCL case)
    from paper_2508_19911_b200 import Solver, nccl_unique_id
    if chunk:
        monkeypatch.setenv("CGKS_CHUNK", str(chunk))
    else:
        monkeypatch.delenv("CGKS_CHUNK", raising=False)
    S = Solver.from_case(case, nccl_id=nccl_unique_id() if nccl else None, **kw)
    S.set_state(case.Q, case.G)
    if L is not None:
        S.set_lines(L)
    S.step(steps)
    Q, G = S.get_state()
    t = S.get_time()
    Lo = S.get_lines() if L is not None else None
    S.close()
    return Q, G, t, Lo


@pytest.mark.parametrize("chunk", [3, 5])
@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
def test_chunked_bitwise(scheme, nl, chunk, monkeypatch):
    case = random_smooth((20, 12, 16), seed=8, jump=0.4 if nl else 0.0)
    kw = dict(scheme=scheme, nonlinear=nl, mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _run(case, 4, 0, monkeypatch, **kw)
    Q2, G2, t2, _ = _run(case, 4, chunk, monkeypatch, **kw)
    assert t1 == t2
    assert np.array_equal(Q1, Q2)
    if scheme == 1:
        assert np.array_equal(G1, G2)


def test_chunked_lines_box_x_bitwise(monkeypatch):
    # line DOFs and inflow / outflow x boundaries (z periodic) through the chunked stage
    case = random_smooth((16, 12, 14), seed=9, jump=0.3)
    rng = np.random.default_rng(5)
    L = case.G[np.array([1, 2, 1, 2, 2, 0, 2, 0, 0, 1, 0, 1])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
    bs = np.zeros((3, 2, 5))
    bs[:, :] = (1.0, 0.1, 0.0, 0.0, 1.0 / 0.4 + 0.005)
    kw = dict(scheme=1, nonlinear=1, mu=1e-3, Pr=0.72, lines=1, bc=((1, 2), (0, 0), (0, 0)), bc_state=bs)
    Q1, G1, t1, L1 = _run(case, 3, 0, monkeypatch, L=L, **kw)
    Q2, G2, t2, L2 = _run(case, 3, 4, monkeypatch, L=L, **kw)
    assert t1 == t2
    assert np.array_equal(Q1, Q2) and np.array_equal(G1, G2) and np.array_equal(L1, L2)


def test_chunked_stretched_bitwise(monkeypatch):
    case = random_smooth((16, 12, 12), seed=3)
    nodes = (stretched_nodes(16, case.lo[0], case.hi[0], 0.2), None,
             stretched_nodes(12, case.lo[2], case.hi[2], 0.2))
    kw = dict(scheme=1, mu=1e-3, Pr=0.72, nodes=nodes)
    Q1, G1, t1, _ = _run(case, 3, 0, monkeypatch, **kw)
    Q2, G2, t2, _ = _run(case, 3, 5, monkeypatch, **kw)
    assert t1 == t2
    assert np.array_equal(Q1, Q2) and np.array_equal(G1, G2)


@pytest.mark.parametrize("overlap", [1, 0])
def test_chunked_nccl_self_bitwise(overlap, monkeypatch):
    # the NCCL slab path with chunks: the exchange on the halo stream overlaps the interior chunks
    if not overlap:
        monkeypatch.setenv("CGKS_NO_OVERLAP", "1")
    case = random_smooth((16, 12, 20), seed=4, jump=0.3)
    kw = dict(scheme=1, nonlinear=1, mu=1e-3, Pr=0.72)
    Q1, G1, t1, _ = _run(case, 4, 0, monkeypatch, **kw)
    Q2, G2, t2, _ = _run(case, 4, 4, monkeypatch, nccl=True, **kw)
    assert t1 == t2
    assert np.array_equal(Q1, Q2) and np.array_equal(G1, G2)


def test_chunked_async_pipeline(monkeypatch):
    # the asynchronous host I/O calls on a chunked context
    import torch
    case = random_smooth((16, 12, 12), seed=2)
    kw = dict(scheme=1, mu=1e-3, Pr=0.72)
    Q1, G1, _, _ = _run(case, 2, 0, monkeypatch, **kw)
    from paper_2508_19911_b200 import Solver
    monkeypatch.setenv("CGKS_CHUNK", "5")
    S = Solver.from_case(case, **kw)
    qo = torch.zeros(case.Q.shape, dtype=torch.float64).pin_memory()
    go = torch.zeros(case.G.shape, dtype=torch.float64).pin_memory()
    S.set_state_async(case.Q, case.G)
    S.step_async(2)
    S.get_state_async(qo, go)
    S.sync()
    S.close()
    assert np.array_equal(qo.numpy(), Q1) and np.array_equal(go.numpy(), G1)
