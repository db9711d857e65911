"""GPU parity of the line-DOF variant of CGKS-5th:
the own cell's line-averaged derivatives replace its gradient as reconstruction data and are
updated from the interface values at corresponding Gauss points of opposite faces.  The library
(through cgks_set_lines / cgks_step / cgks_get_lines) against the oracle's run_lines on the same
inputs: relative L-infinity <= 1e-10 after 10 steps for averages, gradients and lines (R34 floors)."""
import math

import numpy as np
import pytest

import oracle
from cgks_inputs import line_derivatives, vortex
from cgks_inputs.cases import _vortex_prim, gl_average
from parity_util import floors, hmin, rel_linf, worst

pytestmark = pytest.mark.gpu


def _smooth3d():
    def prim(x, y, z):
        rho = 1.0 + 0.2 * np.sin(x) * np.cos(2 * y) + 0.1 * np.cos(z)
        u = 0.3 * np.sin(y + z)
        v = -0.2 * np.cos(x) * np.sin(z)
        w = 0.25 * np.sin(x + 2 * y)
        p = 1.0 + 0.1 * np.cos(x + y) * np.sin(z)
        return rho, u, v, w, p
    n = (20, 12, 10)
    lo, hi = (0.0, 0.0, 0.0), (2 * math.pi, 2 * math.pi, 2 * math.pi)
    Q, G = gl_average(prim, n, lo, hi, 1.4, nq=4)
    L = line_derivatives(prim, n, lo, hi, 1.4)
    return n, lo, hi, Q, G, L


def _compare(Qg, Gg, Lg, Qo, Go, Lo, h, tol, nsteps=10):
    r = rel_linf(Qg, Qo, Gg, Go, h=h, nsteps=nsteps, tol=tol)
    k, v = worst(r)
    assert v <= tol, (k, v)
    qs, gs = floors(Qo, Go, h, nsteps, tol)
    el = np.abs(Lg - Lo).max(axis=(0, 2, 3, 4)) / gs
    assert el.max() <= tol, el


@pytest.mark.parametrize("nl", [0, 1])
def test_lines_parity_3d(nl):
    from paper_2508_19911_b200 import Solver
    n, lo, hi, Q, G, L = _smooth3d()
    kw = dict(gamma=1.4, mu=2e-3, Pr=0.72, nonlinear=nl)
    prob = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, lines=1, cfl=0.3, **kw)
    Qo, Go, Lo, to, _, rc = oracle.run_lines(prob, Q, G, L, 10)
    assert rc == 0
    S = Solver(n, lo, hi, scheme=1, lines=1, cfl=0.3, **kw)
    S.set_state(Q, G)
    S.set_lines(L)
    S.step(10)
    Qg, Gg = S.get_state()
    Lg = S.get_lines()
    tg, _, _ = S.get_time()
    S.close()
    assert abs(tg - to) <= 1e-13 * to
    _compare(Qg, Gg, Lg, Qo, Go, Lo, hmin(n, lo, hi), 1e-10)


def test_lines_parity_vortex_2d():
    from paper_2508_19911_b200 import Solver
    c = vortex(40)
    L = line_derivatives(_vortex_prim(0.0), c.n, c.lo, c.hi, c.gamma)
    d = c.problem_kwargs()
    prob = oracle.Problem(**d, scheme=1, time_scheme=2, lines=1)
    Qo, Go, Lo, to, _, rc = oracle.run_lines(prob, c.Q, c.G, L, 20)
    assert rc == 0
    S = Solver.from_case(c, scheme=1, lines=1)
    S.set_state(c.Q, c.G)
    S.set_lines(L)
    S.step(20)
    Qg, Gg = S.get_state()
    Lg = S.get_lines()
    S.close()
    _compare(Qg, Gg, Lg, Qo, Go, Lo, hmin(c), 1e-10, 20)


def test_lines_default_from_gradients():
    # without cgks_set_lines the lines start from the gradients on both sides
    from paper_2508_19911_b200 import Solver
    n, lo, hi, Q, G, L = _smooth3d()
    prob = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, lines=1, cfl=0.3, mu=1e-3, Pr=0.72)
    Qo, Go, _, _, rc = oracle.run(prob, Q, G, 5)
    assert rc == 0
    S = Solver(n, lo, hi, scheme=1, lines=1, cfl=0.3, mu=1e-3, Pr=0.72)
    S.set_state(Q, G)
    S.step(5)
    Qg, Gg = S.get_state()
    S.close()
    k, v = worst(rel_linf(Qg, Qo, Gg, Go, h=hmin(n, lo, hi), nsteps=5))
    assert v <= 1e-10, (k, v)


def test_lines_diagnostics_and_qcriterion():
    from paper_2508_19911_b200 import Solver
    n, lo, hi, Q, G, L = _smooth3d()
    kw = dict(gamma=1.4, mu=2e-3, Pr=0.72)
    prob = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, lines=1, cfl=0.3, **kw)
    S = Solver(n, lo, hi, scheme=1, lines=1, cfl=0.3, **kw)
    S.set_state(Q, G)
    S.set_lines(L)
    S.step(3)
    Qg, Gg = S.get_state()
    Lg = S.get_lines()
    dg, qg = S.diagnostics(), S.qcriterion()
    S.close()
    do = oracle.diagnostics(prob, Qg, Gg, Lg)
    qo = oracle.qcriterion(prob, Qg, Gg, Lg)
    assert np.all(np.abs(dg - do) <= 1e-12 * np.abs(do) + 1e-300), (dg, do)
    assert np.abs(qg - qo).max() <= 1e-11 * np.abs(qo).max()


@pytest.mark.parametrize("nl", [0, 1])
@pytest.mark.parametrize("bc", [((2, 2), (0, 0), (0, 0)), ((0, 0), (1, 1), (2, 2))])
def test_lines_parity_box(nl, bc):
    # box boundaries: a ghost cell takes the boundary cell's lines (outflow) or none (inflow), as in
    # the oracle's ghost rule
    from paper_2508_19911_b200 import Solver
    n, lo, hi, Q, G, L = _smooth3d()
    bs = np.zeros((3, 2, 5))
    bs[:, :] = (1.0, 0.1, 0.0, 0.0, 1.0 / 0.4 + 0.005)  # inflow: rho = 1, u = 0.1, p = 1
    kw = dict(gamma=1.4, mu=2e-3, Pr=0.72, nonlinear=nl, bc=bc, bc_state=bs)
    prob = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, lines=1, cfl=0.3, **kw)
    Qo, Go, Lo, to, _, rc = oracle.run_lines(prob, Q, G, L, 10)
    assert rc == 0
    S = Solver(n, lo, hi, scheme=1, lines=1, cfl=0.3, **kw)
    S.set_state(Q, G)
    S.set_lines(L)
    S.step(10)
    Qg, Gg = S.get_state()
    Lg = S.get_lines()
    tg, _, _ = S.get_time()
    S.close()
    assert abs(tg - to) <= 1e-13 * to
    _compare(Qg, Gg, Lg, Qo, Go, Lo, hmin(n, lo, hi), 1e-10)
