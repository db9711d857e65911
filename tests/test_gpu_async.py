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


def test_async_error_of_first_batch_is_not_wiped():
    # a failure in batch n must survive cgks_set_state_async of batch n+1 (sticky record)
    from paper_2508_19911_b200 import CgksError, Solver
    case = random_smooth((16, 8, 6), seed=2)
    good = [random_smooth((16, 8, 6), seed=s) for s in (3, 4)]
    S = Solver.from_case(case, scheme=1)
    Qb = case.Q.copy()
    Qb[0, 2, 3, 4] = -1.0
    outs = [(_pinned(np.zeros_like(case.Q)), _pinned(np.zeros_like(case.G))) for _ in range(3)]
    for (Q, G), (qo, go) in zip([(Qb, case.G)] + [(c.Q, c.G) for c in good], outs):
        S.set_state_async(Q, G)
        S.step_async(2)
        S.get_state_async(qo, go)
    with pytest.raises(CgksError) as e:
        S.sync()
    assert e.value.code == 3
    assert "earlier pipelined batch" in S.last_error()
    # the later batches ran normally
    R = Solver.from_case(case, scheme=1)
    for c, (qo, go) in zip(good, outs[1:]):
        R.set_state(c.Q, c.G)
        R.step(2)
        Qr, Gr = R.get_state()
        assert np.array_equal(qo.numpy(), Qr) and np.array_equal(go.numpy(), Gr)
    R.close()
    # the record is cleared by the sync that reported it
    S.set_state(good[0].Q, good[0].G)
    S.step(1)
    S.close()


def test_async_after_sync_steps_bookkeeping():
    # sync steps, then async steps, then a new batch that fails: the buffer index must stay valid
    from paper_2508_19911_b200 import CgksError, Solver
    case = random_smooth((16, 8, 6), seed=2)
    S = Solver.from_case(case, scheme=1)
    S.set_state(case.Q, case.G)
    S.step(4)
    S.step_async(1)
    Qb = case.Q.copy()
    Qb[0, 1, 1, 1] = -1.0
    S.set_state_async(Qb, case.G)
    S.step_async(5)
    with pytest.raises(CgksError) as e:
        S.sync()
    assert e.value.code == 3
    Q3, _ = S.get_state()
    assert np.array_equal(Q3, Qb)
    S.close()


def test_two_contexts_constants_ordered():
    # context B's constant upload must wait for context A's enqueued asynchronous steps
    from paper_2508_19911_b200 import Solver
    a = random_smooth((20, 12, 10), seed=1)
    b = random_smooth((12, 10, 8), seed=2)
    R = Solver.from_case(a, scheme=1, mu=1e-3, Pr=0.72)
    R.set_state(a.Q, a.G)
    R.step(4)
    Qr, Gr = R.get_state()
    R.close()
    A = Solver.from_case(a, scheme=1, mu=1e-3, Pr=0.72)
    B = Solver.from_case(b, scheme=1, nonlinear=1, mu=5e-3, Pr=1.0)
    qo, go = _pinned(np.zeros_like(a.Q)), _pinned(np.zeros_like(a.G))
    A.set_state_async(a.Q, a.G)
    A.step_async(4)
    A.get_state_async(qo, go)
    B.set_state(b.Q, b.G)  # takes the constants while A's steps may still be queued
    B.step(2)
    A.sync()
    assert np.array_equal(qo.numpy(), Qr) and np.array_equal(go.numpy(), Gr)
    A.close()
    B.close()
