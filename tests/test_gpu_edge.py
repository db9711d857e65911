"""Edge cases of the C ABI on the GPU: invalid configurations are refused with CGKS_ERR_CONFIG,
degenerate and tiny grids run and match the oracle, non-finite input is reported as an error instead
of propagating silently, an impossible allocation fails cleanly (and the next context still works),
and zero steps leave the state untouched."""
import numpy as np
import pytest

import oracle
from cgks_inputs import random_smooth, uniform
from parity_util import hmin, rel_linf, worst

pytestmark = pytest.mark.gpu


def _S():
    from paper_2508_19911_b200 import CgksError, Solver
    return Solver, CgksError


@pytest.mark.parametrize("kw", [
    dict(n=(0, 4, 4)),
    dict(gamma=0.9),
    dict(mu=-1.0),
    dict(scheme=0, lines=1),
    dict(sutherland_S=-1.0),
    dict(nodes=(np.array([0.0, 0.5, 0.4, 1.0]), None, None), n=(3, 4, 4)),
])
def test_invalid_configurations_are_refused(kw):
    Solver, CgksError = _S()
    args = dict(n=(4, 4, 4), lo=(0, 0, 0), hi=(1, 1, 1), scheme=1)
    args.update(kw)
    with pytest.raises(CgksError) as e:
        Solver(**args)
    assert e.value.code == 2


@pytest.mark.parametrize("n", [(3, 3, 3), (5, 1, 1), (3, 4, 1)])
@pytest.mark.parametrize("scheme", [1, 0])
def test_tiny_grids_match_oracle(n, scheme):
    Solver, _ = _S()
    c = random_smooth(n, seed=3)
    ts = 2 if scheme == 1 else 1
    p = oracle.Problem(**c.problem_kwargs(), scheme=scheme, time_scheme=ts)
    Qo, Go, _, _, rc = oracle.run(p, c.Q, c.G, 3)
    assert rc == 0
    S = Solver.from_case(c, scheme=scheme, time_scheme=ts)
    S.set_state(c.Q, c.G if scheme == 1 else None)
    S.step(3)
    Qg, Gg = S.get_state()
    S.close()
    k, v = worst(rel_linf(Qg, Qo, Gg if scheme == 1 else None, Go if scheme == 1 else None, h=hmin(c), nsteps=3))
    assert v <= 1e-10, (k, v)


def test_nonfinite_input_is_an_error():
    Solver, CgksError = _S()
    c = uniform((8, 8, 8))
    Q = c.Q.copy()
    Q[4, 3, 3, 3] = np.nan
    S = Solver.from_case(c, scheme=1)
    S.set_state(Q, c.G)
    with pytest.raises(CgksError) as e:
        S.step(1)
    assert e.value.code in (3, 4)
    S.close()


def test_impossible_allocation_fails_cleanly():
    Solver, CgksError = _S()
    with pytest.raises(CgksError) as e:
        Solver(n=(4096, 4096, 4096), lo=(0, 0, 0), hi=(1, 1, 1), scheme=1)
    assert e.value.code in (2, 5)  # 2: beyond the 2^32-element buffer limit (checked first), 5: allocation
    c = uniform((6, 6, 6))
    S = Solver.from_case(c, scheme=1)  # the device is still usable
    S.set_state(c.Q, c.G)
    S.step(1)
    S.close()


def test_zero_steps_leave_the_state():
    Solver, _ = _S()
    c = random_smooth((6, 5, 4), seed=1)
    S = Solver.from_case(c, scheme=1)
    S.set_state(c.Q, c.G)
    S.step(0)
    Q, G = S.get_state()
    t, steps, _ = S.get_time()
    S.close()
    assert steps == 0 and t == 0.0 and np.array_equal(Q, c.Q) and np.array_equal(G, c.G)


@pytest.mark.parametrize("graph", [0, 1])
def test_positivity_failure_in_large_run_is_clean(graph, monkeypatch):
    """A positivity failure raised mid-kernel on a large grid (high-speed TGV 116^3 without the
    collision-time jump term fails near step 470) is reported as CGKS_ERR_POSITIVITY with the state
    of the last completed step -- blocks that start after the flag is raised exit as a whole (a
    thread-divergent exit used to leave threads waiting on an uninitialised TMA barrier: launch
    failure)."""
    if not graph:
        monkeypatch.setenv("CGKS_NO_GRAPH", "1")
    from cgks_inputs import tgv_supersonic
    Solver, CgksError = _S()
    case = tgv_supersonic(116)
    S = Solver.from_case(case, scheme=1, tau_C=0.0)
    S.set_state(case.Q, case.G)
    S.step(455)
    with pytest.raises(CgksError) as e:
        S.step(40)
    assert e.value.code == 3, str(e.value)
    Q, _ = S.get_state()
    assert np.isfinite(Q).all() and Q[0].min() > 0
    S.close()
