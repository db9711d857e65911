"""Asynchronous host I/O (cgks_set_state_async / cgks_step_async / cgks_get_state_async / cgks_sync):
the pipelined calls give bit for bit the results of the synchronous ones, for every stage of a
pipeline whose input and output copies overlap the steps, and deferred step errors surface at
cgks_sync with the synchronous semantics (the state is the last completed step)."""
import numpy as np
import pytest

from cgks_inputs import random_smooth

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


@pytest.mark.parametrize("scheme", [1, 0])
@pytest.mark.parametrize("graph", [1, 0])
def test_async_pipeline_matches_sync(scheme, graph, monkeypatch):
    if not graph:
        monkeypatch.setenv("CGKS_NO_GRAPH", "1")
    from paper_2508_19911_b200 import Solver
    cases = [random_smooth((20, 12, 10), seed=s, jump=0.2) for s in (1, 2, 3)]
    kw = dict(mu=1e-3, Pr=0.72)
    ref = []
    S = Solver.from_case(cases[0], scheme=scheme, **kw)
    for c in cases:
        S.set_state(c.Q, c.G if scheme == 1 else None)
        S.step(3)
        ref.append(S.get_state())
    ins = [(_pinned(c.Q), _pinned(c.G)) for c in cases]
    outs = [(_pinned(np.zeros_like(c.Q)), _pinned(np.zeros_like(c.G))) for c in cases]
    for (qi, gi), (qo, go) in zip(ins, outs):  # three overlapped set / step / get stages, one sync
        S.set_state_async(qi, gi if scheme == 1 else None)
        S.step_async(3)
        S.get_state_async(qo, go)
    S.sync()
    for (Qr, Gr), (qo, go) in zip(ref, outs):
        assert np.array_equal(qo.numpy(), Qr)
        assert np.array_equal(go.numpy(), Gr)
    # numpy (pageable) buffers and device tensors work too
    import torch
    qd = torch.zeros(cases[0].Q.shape, dtype=torch.float64, device="cuda")
    S.set_state_async(cases[0].Q, cases[0].G if scheme == 1 else None)
    S.step_async(3)
    S.get_state_async(qd)
    S.sync()
    assert np.array_equal(qd.cpu().numpy(), ref[0][0])
    t, steps, _ = S.get_time()
    assert steps == 3
    S.close()


def test_async_deferred_positivity_error():
    from paper_2508_19911_b200 import CgksError, Solver
    case = random_smooth((16, 8, 6), seed=2)
    S = Solver.from_case(case, scheme=1)
    S.set_state(case.Q, case.G)
    S.step(2)
    Q2, G2 = S.get_state()
    Qb = Q2.copy()
    Qb[0, 2, 3, 4] = -1.0
    S.set_state_async(Qb, G2)
    S.step_async(3)  # fails in its first step; reported by sync
    with pytest.raises(CgksError) as e:
        S.sync()
    assert e.value.code == 3
    Q3, _ = S.get_state()
    assert np.array_equal(Q3, Qb)
    assert S.get_time()[1] == 0
    S.close()
