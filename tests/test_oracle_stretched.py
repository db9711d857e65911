"""Pins of the oracle on stretched tensor-product meshes (P:255 reference-cell
transformation, reading R37: each cell maps affinely to the reference cell, the reconstruction uses
the uniform reference stencil with every cell's data in its own reference units, the update divides by
the cell's own widths).

Pinned by: uniform node arrays reproduce the uniform path bit for bit; exact conservation of
sum_c Q_c V_c on a periodic stretched mesh; bitwise preservation of uniform flow; convergence on the
isentropic vortex on a smoothly stretched mesh (the index-space reconstruction is second order on
non-uniform cells: the measured order falls from ~3.7 towards 2 as h -> 0, DESIGN R37); and the
Crocco-Busemann jet inflow relations."""
import math

import numpy as np
import pytest

import oracle
from cgks_inputs import gl_average, jet_inflow, stretched_nodes, uniform, vortex
from cgks_inputs.cases import _vortex_prim


def _vortex_on(n, beta):
    nx = stretched_nodes(n, 0.0, 10.0, beta)
    ny = stretched_nodes(n, 0.0, 10.0, beta)
    nz = np.array([0.0, 1.0])
    Q, G = gl_average(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=(nx, ny, nz))
    return (nx, ny, nz), Q, G


@pytest.mark.parametrize("scheme", [1, 0])
def test_uniform_nodes_reproduce_uniform_path(scheme):
    c = vortex(40)  # h = 0.25: node coordinates k/4 are exact, so the widths are exactly h
    nodes = (np.arange(41) * 0.25, np.arange(41) * 0.25, np.array([0.0, 1.0]))
    d = c.problem_kwargs()
    p0 = oracle.Problem(**d, scheme=scheme, time_scheme=2 if scheme else 1)
    p1 = oracle.Problem(**d, scheme=scheme, time_scheme=2 if scheme else 1, nodes=nodes)
    a = oracle.run(p0, c.Q, c.G, 5)
    b = oracle.run(p1, c.Q, c.G, 5)
    assert np.array_equal(a[0], b[0]) and (scheme == 0 or np.array_equal(a[1], b[1])) and a[2] == b[2]


@pytest.mark.parametrize("scheme", [1, 0])
def test_conservation_on_stretched_periodic_mesh(scheme):
    nodes, Q, G = _vortex_on(24, 0.3)
    V = np.diff(nodes[0])[None, :] * np.diff(nodes[1])[:, None] * 1.0
    p = oracle.Problem(n=(24, 24, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=scheme, time_scheme=2 if scheme else 1,
                       mu=1e-3, Pr=0.72, nodes=nodes, nonlinear=1)
    Q1, G1, t, dt, rc = oracle.run(p, Q, G, 6)
    assert rc == 0
    for v in range(5):
        m0 = (Q[v, 0] * V).sum()
        m1 = (Q1[v, 0] * V).sum()
        assert abs(m1 - m0) <= 1e-13 * max(1.0, abs(m0)), (v, m0, m1)


def test_uniform_flow_preserved_on_stretched_mesh():
    c = uniform((10, 8, 6), state=(1.2, 0.3, -0.4, 0.5, 0.9), L=1.0)
    nodes = (stretched_nodes(10, 0, 1, 0.3), stretched_nodes(8, 0, 1, 0.2, "sine"), stretched_nodes(6, 0, 1, 0.25))
    d = c.problem_kwargs()
    d.update(mu=1e-3, Pr=0.72)
    p = oracle.Problem(**d, scheme=1, time_scheme=2, nodes=nodes)
    Q1, G1, t, dt, rc = oracle.run(p, c.Q, c.G, 4)
    assert rc == 0 and np.array_equal(Q1, c.Q) and np.abs(G1).max() == 0.0


def test_vortex_converges_on_stretched_mesh():
    errs = []
    for n, ns in ((20, 10), (40, 24), (80, 57)):
        nodes, Q, G = _vortex_on(n, 0.2)
        p = oracle.Problem(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=1, time_scheme=2, fixed_dt=1.0 / ns,
                           mu=0.0, Pr=1.0, tau_eps=0.0, tau_C=0.0, nodes=nodes)
        Q1, _, t, _, rc = oracle.run(p, Q, G, ns)
        assert rc == 0
        Qe, _ = gl_average(_vortex_prim(t), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=nodes)
        errs.append(np.abs(Q1[0] - Qe[0]).mean())
    o = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert o[0] > 3.0 and o[1] > 1.8, (errs, o)


def test_jet_inflow_crocco_busemann():
    r = np.linspace(0.0, 1.0, 401)
    rho, u, p = jet_inflow(r, M_j=0.9, T_j=1.2, T_inf=1.0, R0=0.5, theta=0.01)
    gam = 1.4
    Uj = 0.9 * math.sqrt(1.2)
    T = gam * p / rho
    assert abs(u[0] - Uj) < 1e-12 * Uj and abs(u[-1]) < 1e-12
    assert abs(T[0] - 1.2) < 1e-9 and abs(T[-1] - 1.0) < 1e-9  # core and ambient temperatures
    f = u / Uj
    want = 1.0 + 0.2 * f + 0.5 * (gam - 1.0) * 0.81 * 1.2 * f * (1.0 - f)
    assert np.abs(T - want).max() < 1e-12
    assert np.all(np.diff(u) <= 1e-15)  # monotone profile


# ---- line DOFs (NEXT-1) on stretched meshes: the own cell's lines in its own reference units
def _vortex_lines_on(n, beta):
    from cgks_inputs import line_derivatives
    nodes, Q, G = _vortex_on(n, beta)
    L = line_derivatives(_vortex_prim(0.0), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, mesh_nodes=nodes)
    return nodes, Q, G, L


def test_lines_uniform_nodes_reproduce_uniform_path():
    from cgks_inputs import line_derivatives
    c = vortex(40)
    nodes = (np.arange(41) * 0.25, np.arange(41) * 0.25, np.array([0.0, 1.0]))
    L = line_derivatives(_vortex_prim(0.0), c.n, c.lo, c.hi, c.gamma)
    L2 = line_derivatives(_vortex_prim(0.0), c.n, c.lo, c.hi, c.gamma, mesh_nodes=nodes)
    assert np.array_equal(L, L2)
    d = c.problem_kwargs()
    p0 = oracle.Problem(**d, scheme=1, time_scheme=2, lines=1)
    p1 = oracle.Problem(**d, scheme=1, time_scheme=2, lines=1, nodes=nodes)
    a = oracle.run_lines(p0, c.Q, c.G, L, 5)
    b = oracle.run_lines(p1, c.Q, c.G, L, 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2]) and a[3] == b[3]


def test_lines_conservation_on_stretched_periodic_mesh():
    nodes, Q, G, L = _vortex_lines_on(24, 0.3)
    V = np.diff(nodes[0])[None, :] * np.diff(nodes[1])[:, None] * 1.0
    p = oracle.Problem(n=(24, 24, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=1, time_scheme=2, lines=1,
                       mu=1e-3, Pr=0.72, nodes=nodes, nonlinear=1)
    Q1, G1, L1, t, dt, rc = oracle.run_lines(p, Q, G, L, 6)
    assert rc == 0
    for v in range(5):
        m0 = (Q[v, 0] * V).sum()
        m1 = (Q1[v, 0] * V).sum()
        assert abs(m1 - m0) <= 1e-13 * max(1.0, abs(m0)), (v, m0, m1)


def test_lines_vortex_converges_on_stretched_mesh():
    """the line data scaled by the own widths (R37): high-order convergence on a stretched mesh, with
    errors of the size the gradient-DOF scheme has on the same meshes (a line scaled by a wrong width
    is an O(1) relative error in the own-cell data and costs orders of magnitude at n = 40)."""
    errs, errs_g = [], []
    for n, ns in ((20, 10), (40, 24)):
        nodes, Q, G, L = _vortex_lines_on(n, 0.2)
        kw = dict(n=(n, n, 1), lo=(0, 0, 0), hi=(10, 10, 1), scheme=1, time_scheme=2, fixed_dt=1.0 / ns,
                  mu=0.0, Pr=1.0, tau_eps=0.0, tau_C=0.0, nodes=nodes)
        Q1, _, _, t, _, rc = oracle.run_lines(oracle.Problem(**kw, lines=1), Q, G, L, ns)
        assert rc == 0
        Qg, _, tg, _, rc = oracle.run(oracle.Problem(**kw), Q, G, ns)
        assert rc == 0 and tg == t
        Qe, _ = gl_average(_vortex_prim(t), (n, n, 1), (0, 0, 0), (10, 10, 1), 1.4, nq=5, mesh_nodes=nodes)
        errs.append(np.abs(Q1[0] - Qe[0]).mean())
        errs_g.append(np.abs(Qg[0] - Qe[0]).mean())
    o = math.log2(errs[0] / errs[1])
    assert o > 3.0, (errs, o)
    assert errs[1] < 3.0 * errs_g[1], (errs, errs_g)
