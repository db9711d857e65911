"""GPU parity on stretched tensor-product meshes (reading R37): the
library with per-axis node arrays against the oracle on the same inputs, relative L-infinity <= 1e-10
after 10 steps (R34 floors), both schemes, periodic and box boundaries; uniform node arrays reproduce
the uniform path bit for bit."""
import math

import numpy as np
import pytest

import oracle
from cgks_inputs import gl_average, stretched_nodes, vortex
from cgks_inputs.cases import _vortex_prim
from parity_util import rel_linf, worst


def _hmin_nodes(nodes, n, lo, hi):
    hs = []
    for a in range(3):
        if n[a] > 1:
            hs.append(np.diff(nodes[a]).min() if nodes[a] is not None else (hi[a] - lo[a]) / n[a])
    return min(hs)

pytestmark = pytest.mark.gpu


def _solver(**kw):
    from paper_2508_19911_b200 import Solver
    return Solver(**kw)


def _both(n, lo, hi, nodes, Q, G, scheme, steps, **kw):
    ts = 2 if scheme == 1 else 1
    p = oracle.Problem(n=n, lo=lo, hi=hi, scheme=scheme, time_scheme=ts, nodes=nodes, **kw)
    Qo, Go, to, _, rc = oracle.run(p, Q, G if scheme == 1 else None, steps)
    assert rc == 0
    S = _solver(n=n, lo=lo, hi=hi, scheme=scheme, time_scheme=ts, nodes=nodes, **kw)
    S.set_state(np.ascontiguousarray(Q), np.ascontiguousarray(G) if scheme == 1 else None)
    S.step(steps)
    Qg, Gg = S.get_state()
    tg, _, _ = S.get_time()
    S.close()
    assert abs(tg - to) <= 1e-13 * to
    return Qg, Gg, Qo, Go


@pytest.mark.parametrize("scheme,nl", [(1, 0), (1, 1), (0, 1)])
def test_stretched_vortex_2d(scheme, nl):
    n = 32
    nodes = (stretched_nodes(n, 0.0, 10.0, 0.3), stretched_nodes(n, 0.0, 10.0, 0.2, "sine"), np.array([0.0, 1.0]))
    Q, G = gl_average(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=nodes)
    Qg, Gg, Qo, Go = _both((n, n, 1), (0, 0, 0), (10, 10, 1), nodes, Q, G, scheme, 10, mu=1e-3, Pr=0.72,
                           nonlinear=nl, cfl=0.3)
    k, v = worst(rel_linf(Qg, Qo, Gg if scheme == 1 else None, Go if scheme == 1 else None,
                          h=_hmin_nodes(nodes, (n, n, 1), (0, 0, 0), (10, 10, 1))))
    assert v <= 1e-10, (k, v)


@pytest.mark.parametrize("box", [0, 1])
def test_stretched_3d(box):
    n = (20, 12, 10)
    lo, hi = (0.0, 0.0, 0.0), (2 * math.pi,) * 3
    nodes = (stretched_nodes(20, 0.0, 2 * math.pi, 2.0, "tanh"), stretched_nodes(12, 0.0, 2 * math.pi, 0.25),
             None)

    def prim(x, y, z):
        return (1.0 + 0.2 * np.sin(x) * np.cos(2 * y) + 0.1 * np.cos(z), 0.3 * np.sin(y + z),
                -0.2 * np.cos(x) * np.sin(z), 0.25 * np.sin(x + 2 * y), 1.0 + 0.1 * np.cos(x + y) * np.sin(z))
    zn = np.linspace(0.0, 2 * math.pi, 11)
    Q, G = gl_average(prim, n, lo, hi, 1.4, nq=4, mesh_nodes=(nodes[0], nodes[1], zn))
    bc = ((2, 2), (0, 0), (0, 0)) if box else ((0, 0), (0, 0), (0, 0))
    Qg, Gg, Qo, Go = _both(n, lo, hi, nodes, Q, G, 1, 10, mu=2e-3, Pr=0.72, nonlinear=1, cfl=0.3, bc=bc)
    k, v = worst(rel_linf(Qg, Qo, Gg, Go, h=_hmin_nodes(nodes, n, lo, hi)))
    assert v <= 1e-10, (k, v)


def test_uniform_nodes_bitwise_gpu():
    c = vortex(40)  # h = 0.25: nodes k/4 are exact
    nodes = (np.arange(41) * 0.25, np.arange(41) * 0.25, np.array([0.0, 1.0]))
    kw = dict(n=c.n, lo=c.lo, hi=c.hi, scheme=1, mu=0.0, Pr=1.0, tau_eps=0.0, tau_C=0.0, cfl=0.5)
    out = []
    for nd in (None, nodes):
        S = _solver(nodes=nd, **kw)
        S.set_state(c.Q, c.G)
        S.step(5)
        out.append(S.get_state())
        S.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_stretched_diagnostics_and_qcriterion():
    n = 32
    nodes = (stretched_nodes(n, 0.0, 10.0, 0.3), stretched_nodes(n, 0.0, 10.0, 0.2), np.array([0.0, 1.0]))
    Q, G = gl_average(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=nodes)
    for scheme in (1, 0):
        p = oracle.Problem(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=scheme, mu=1e-3, nodes=nodes)
        S = _solver(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=scheme, mu=1e-3, nodes=nodes)
        S.set_state(Q, G if scheme == 1 else None)
        dg, qg = S.diagnostics(), S.qcriterion()
        S.close()
        do = oracle.diagnostics(p, Q, G if scheme == 1 else None)
        qo = oracle.qcriterion(p, Q, G if scheme == 1 else None)
        assert np.all(np.abs(dg - do) <= 1e-12 * np.abs(do) + 1e-300), (scheme, dg, do)
        assert np.abs(qg - qo).max() <= 1e-11 * np.abs(qo).max()


# ---- line DOFs (NEXT-1) on stretched meshes
@pytest.mark.parametrize("nl,box", [(0, 0), (1, 0), (1, 1)])
def test_stretched_lines_3d(nl, box):
    from cgks_inputs import line_derivatives
    n = (20, 12, 10)
    lo, hi = (0.0, 0.0, 0.0), (2 * math.pi,) * 3
    nodes = (stretched_nodes(20, 0.0, 2 * math.pi, 2.0, "tanh"), stretched_nodes(12, 0.0, 2 * math.pi, 0.25),
             None)

    def prim(x, y, z):
        return (1.0 + 0.2 * np.sin(x) * np.cos(2 * y) + 0.1 * np.cos(z), 0.3 * np.sin(y + z),
                -0.2 * np.cos(x) * np.sin(z), 0.25 * np.sin(x + 2 * y), 1.0 + 0.1 * np.cos(x + y) * np.sin(z))
    zn = np.linspace(0.0, 2 * math.pi, 11)
    mn = (nodes[0], nodes[1], zn)
    Q, G = gl_average(prim, n, lo, hi, 1.4, nq=4, mesh_nodes=mn)
    L = line_derivatives(prim, n, lo, hi, 1.4, mesh_nodes=mn)
    bc = ((2, 2), (0, 0), (0, 0)) if box else ((0, 0), (0, 0), (0, 0))
    kw = dict(mu=2e-3, Pr=0.72, nonlinear=nl, cfl=0.3, bc=bc, lines=1)
    p = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, nodes=nodes, **kw)
    Qo, Go, Lo, to, _, rc = oracle.run_lines(p, Q, G, L, 10)
    assert rc == 0
    S = _solver(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, nodes=nodes, **kw)
    S.set_state(Q, G)
    S.set_lines(L)
    S.step(10)
    Qg, Gg = S.get_state()
    Lg = S.get_lines()
    tg, _, _ = S.get_time()
    S.close()
    assert abs(tg - to) <= 1e-13 * to
    k, v = worst(rel_linf(Qg, Qo, Gg, Go, h=_hmin_nodes(nodes, n, lo, hi)))
    assert v <= 1e-10, (k, v)
    from parity_util import floors
    _, gs = floors(Qo, Go, _hmin_nodes(nodes, n, lo, hi))
    el = np.abs(Lg - Lo).max(axis=(0, 2, 3, 4)) / gs
    assert el.max() <= 1e-10, el


def test_stretched_lines_diagnostics():
    # diagnostics / Q-criterion of the line reconstruction on a stretched mesh against the oracle
    from cgks_inputs import line_derivatives
    n = 24
    nodes = (stretched_nodes(n, 0.0, 10.0, 0.3), stretched_nodes(n, 0.0, 10.0, 0.2, "sine"), np.array([0.0, 1.0]))
    Q, G = gl_average(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=nodes)
    L = line_derivatives(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, mesh_nodes=nodes)
    kw = dict(mu=1e-3, Pr=0.72, lines=1)
    p = oracle.Problem(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=1, time_scheme=2, nodes=nodes, **kw)
    do = oracle.diagnostics(p, Q, G, L)
    qo = oracle.qcriterion(p, Q, G, L)
    S = _solver(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=1, nodes=nodes, **kw)
    S.set_state(Q, G)
    S.set_lines(L)
    dg = S.diagnostics()
    qg = S.qcriterion()
    S.close()
    assert np.allclose(dg, do, rtol=1e-12, atol=0), (dg, do)
    assert np.abs(qg - qo).max() <= 1e-11 * np.abs(qo).max()
