"""Pins of the oracle's line-DOF variant of CGKS-5th (P:166-172, P:197-203,
P:219-228): the own cell's line-averaged derivatives replace its gradient as reconstruction
data and are updated from the interface values at corresponding Gauss points of opposite faces.

Pinned by: exact reproduction of random quartics from exactly integrated averages, gradients and line
derivatives (the line rows are differences of the polynomial along segments, written here from the
polynomial itself); a resting gas with a bilinear density (an exact steady Euler state) keeps its
averages and its line derivatives equal to the exact values at every transverse Gauss point; and
fifth-order convergence on the isentropic vortex."""
import math

import numpy as np
import pytest

import oracle
from cgks_inputs import line_derivatives, line_points, vortex, vortex_exact
from cgks_inputs.cases import _vortex_prim
from test_oracle_recon import poly_case


def _lines_of(f, dim, nn, h):
    """exact line derivatives of the polynomial f at every cell: [nl][5][nz][ny][nx]"""
    out = []
    for a in range(dim):
        for t in line_points(dim, a):
            L = np.zeros((5, nn[2], nn[1], nn[0]))
            for k in range(nn[2]):
                for j in range(nn[1]):
                    for i in range(nn[0]):
                        c = [(i + 0.5) * h[0], (j + 0.5) * h[1], (k + 0.5) * h[2]]
                        xp = [c[b] + t[b] * h[b] + (0.5 * h[a] if b == a else 0.0) for b in range(3)]
                        xm = [c[b] + t[b] * h[b] - (0.5 * h[a] if b == a else 0.0) for b in range(3)]
                        L[:, k, j, i] = (f(xp) - f(xm)) / h[a]
            out.append(L)
    return np.array(out)


@pytest.mark.parametrize("dim,seed", [(3, 0), (3, 5), (2, 2), (1, 3)])
def test_lines_cls_quartic_exactness(dim, seed):
    prob, Q, G, f, df, h, c = poly_case(dim, 4, seed)
    prob.lines = 1
    nn = Q.shape[1:][::-1]
    L = _lines_of(f, dim, nn, h)
    assert L.shape[0] == oracle.nlines(dim)
    rng = np.random.default_rng(seed + 7)
    x = rng.uniform(-0.5, 0.5, size=(6, 3))
    x[:, dim:] = 0.0
    W, dW, _ = oracle.recon_eval_lines(prob, Q, G, L, c, x)
    for q in range(x.shape[0]):
        xp = [(c[a] + 0.5 + x[q, a]) * h[a] if a < dim else 0.5 * h[a] for a in range(3)]
        assert np.allclose(W[q], f(xp), rtol=0, atol=1e-11 * np.abs(Q).max())
        assert np.allclose(dW[q][:dim], df(xp)[:dim], rtol=0, atol=1e-10 * np.abs(G).max())
    # the lines really are used: corrupting them changes the reconstruction
    W2, _, _ = oracle.recon_eval_lines(prob, Q, G, L * 1.01, c, x)
    assert np.abs(W2 - W).max() > 1e-9


def test_lines_steady_bilinear_density():
    """rho = 1 + e x y, U = 0, p = 1 is a steady Euler state; after one S2O4 step the interior cells keep
    their averages and every line derivative equals the exact value e y (x-lines) / e x (y-lines) / 0
    (z-lines) at its own transverse Gauss point."""
    n, e = 12, 0.3
    gam = 1.4

    def prim(x, y, z):
        one = np.ones_like(x + y + z)
        return 1.0 + e * x * y, 0.0 * one, 0.0 * one, 0.0 * one, one

    from cgks_inputs.cases import gl_average
    lo, hi = (-0.5, -0.5, -0.5), (0.5, 0.5, 0.5)
    Q, G = gl_average(prim, (n, n, n), lo, hi, gam, nq=4)
    L = line_derivatives(prim, (n, n, n), lo, hi, gam)
    prob = oracle.Problem(n=(n, n, n), lo=lo, hi=hi, gamma=gam, scheme=1, mu=0.0, Pr=1.0, lines=1,
                          tau_eps=0.0, tau_C=0.0, bc=((2, 2), (2, 2), (2, 2)), cfl=0.3)  # tau = 0: Euler (R18)
    Q1, G1, L1, t, dt, rc = oracle.run_lines(prob, Q, G, L, 1)
    assert rc == 0 and t > 0
    s = slice(5, 7)
    assert np.abs(Q1[:, s, s, s] - Q[:, s, s, s]).max() < 1e-12
    assert np.abs(L1[:, :, s, s, s] - L[:, :, s, s, s]).max() < 1e-11
    # the x-lines differ per Gauss point (e y at y_c +- h/(2 sqrt 3)): the layout is exercised
    assert np.abs(L[0, 0, 6, 6, 6] - L[2, 0, 6, 6, 6]) > 1e-3


@pytest.mark.slow
def test_lines_vortex_order():
    """fifth-order convergence of the line-DOF CGKS-5th on the isentropic vortex (linear, tau = 0)."""
    errs = []
    for n, ns in ((20, 10), (40, 24), (80, 57)):
        c = vortex(n)
        d = c.problem_kwargs()
        p = oracle.Problem(**d, scheme=1, time_scheme=2, fixed_dt=1.0 / ns, lines=1)
        L = line_derivatives(_vortex_prim(0.0), c.n, c.lo, c.hi, c.gamma)
        Q, G, L2, t, dt, rc = oracle.run_lines(p, c.Q, c.G, L, ns)
        assert rc == 0
        Qe, _ = vortex_exact(n, t)
        errs.append((np.abs(Q[0] - Qe[0]).mean(), np.abs(Q[0] - Qe[0]).max()))
    e = np.array(errs)
    o1 = np.log2(e[:-1, 0] / e[1:, 0])
    assert o1[-1] > 4.5, (e, o1)
