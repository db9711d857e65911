"""Pins of the oracle's flow diagnostics: quadrature of
the reconstructed state for E_k, the solenoidal and dilatational dissipation and the mass.

Pinned by closed forms that do not use the oracle's formulas: uniform flow (exact values, zero
dissipation), the Taylor-Green initial fields (E_k = U0^2 |Omega| / 8, int |curl U|^2 = 3/4 U0^2 |Omega|,
div U = 0), approached at the reconstruction's order under refinement, and the high-speed TGV whose
temperature is 1 everywhere (so the Sutherland mu equals mu0)."""
import math

import numpy as np
import pytest

import oracle
from cgks_inputs import tgv, tgv_supersonic, uniform


def _prob(case, **kw):
    d = case.problem_kwargs()
    d.update(kw)
    return oracle.Problem(**d)


@pytest.mark.parametrize("scheme", [1, 0])
def test_uniform_flow_exact(scheme):
    state = (1.3, 0.4, -0.2, 0.7, 2.0)  # rho, u, v, w, p
    c = uniform((6, 5, 4), state=state, L=2.0)
    d = oracle.diagnostics(_prob(c, scheme=scheme, mu=0.01), c.Q, c.G)
    vol = 2.0 ** 3
    rho, u, v, w = state[:4]
    assert abs(d[0] - 0.5 * rho * (u * u + v * v + w * w) * vol) < 1e-13
    assert abs(d[1]) < 1e-25 and abs(d[2]) < 1e-25
    assert abs(d[3] - rho * vol) < 1e-13


def test_tgv_initial_values_converge():
    """TGV (rho = 1, U0 = 1) on [-pi, pi]^3: E_k -> (2 pi)^3 / 8, int |curl U|^2 -> 3/4 (2 pi)^3,
    int (div U)^2 -> 0, at the quartic's order (values ~h^5-h^6, derivatives ~h^4: error ratio
    16^3 -> 32^3 above 32 for E_k and above 12 for the dissipation)."""
    V = (2 * math.pi) ** 3
    mu = 1e-3
    errs = []
    for n in (16, 32):
        c = tgv(n)
        d = oracle.diagnostics(_prob(c, scheme=1, mu=mu), c.Q, c.G)
        errs.append((abs(d[0] / V - 0.125), abs(d[1] / (mu * V) - 0.75), abs(d[2] / (mu * V))))
        assert abs(d[3] / V - 1.0) < 1e-13  # rho == 1
    assert errs[1][0] < errs[0][0] / 32.0 and errs[1][1] < errs[0][1] / 12.0, errs
    assert errs[1][0] < 1e-6 and errs[1][1] < 5e-4 and errs[1][2] < 1e-8, errs


def test_tgv_gks2_second_order():
    V = (2 * math.pi) ** 3
    errs = []
    for n in (16, 32):
        c = tgv(n)
        d = oracle.diagnostics(_prob(c, scheme=0, mu=1e-3), c.Q, None)
        errs.append(abs(d[1] / (1e-3 * V) - 0.75))
    assert errs[1] < errs[0] / 3.0, errs


def test_supersonic_tgv_initial_values():
    """P:455-474 at t = 0: E_k / (rho0 U0^2 |Omega|) = 1/8 exactly in the continuum (see the IC pin);
    T == 1 so mu(T) == mu0 and int mu |curl U|^2 = mu0 U0^2 3/4 |Omega|; approached under refinement
    (linear weights; with GENO the blend lowers the order where chi < 1)."""
    V = (2 * math.pi) ** 3
    U0sq = 1.4 * 4.0
    errs = []
    for n in (16, 32):
        c = tgv_supersonic(n)
        d = oracle.diagnostics(_prob(c, scheme=1, nonlinear=0), c.Q, c.G)
        errs.append((abs(d[0] / (U0sq * V) - 0.125), abs(d[1] / (c.mu * U0sq * V) - 0.75)))
        assert abs(d[3] / V - 1.0) < 1e-13
    assert errs[1][0] < errs[0][0] / 32.0 and errs[1][1] < errs[0][1] / 12.0, errs
    assert errs[1][0] < 1e-5 and errs[1][1] < 2e-3, errs


def _linear_velocity_case(n, grad, rho=1.0, p=1.0, U0=(0.0, 0.0, 0.0)):
    """Constant density and pressure, velocity U = U0 + grad . x (grad[b][a] = dU_b/dx_a): exact cell
    averages and gradients of the conservative variables on a box with inflow-free periodic copies
    is not possible, so the field is used only on interior cells (the reconstruction is exact there)."""
    L = 1.0
    h = L / n
    x = (np.arange(n) + 0.5) * h - 0.5
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    pos = [X, Y, Z]
    U = [U0[b] + sum(grad[b][a] * pos[a] for a in range(3)) for b in range(3)]
    gam = 1.4
    Q = np.zeros((5, n, n, n))
    G = np.zeros((3, 5, n, n, n))
    Q[0] = rho
    for b in range(3):
        Q[1 + b] = rho * U[b]
        for a in range(3):
            G[a, 1 + b] = rho * grad[b][a]
    # rho E = p/(gamma-1) + rho |U|^2 / 2: the cell average of a quadratic adds the variance term
    ke = 0.5 * rho * (U[0] ** 2 + U[1] ** 2 + U[2] ** 2)
    var = 0.5 * rho * sum(sum(grad[b][a] ** 2 for b in range(3)) * h * h / 12.0 for a in range(3))
    Q[4] = p / (gam - 1.0) + ke + var
    for a in range(3):
        G[a, 4] = rho * sum(U[b] * grad[b][a] for b in range(3))
    return Q, G


@pytest.mark.parametrize("scheme", [1, 0])
def test_qcriterion_linear_fields(scheme):
    """Q = (|Omega|^2 - |S|^2)/2: solid-body rotation about z with rate w gives w^2, pure strain
    (a x, -a y) gives -a^2, exactly (a linear velocity is reproduced by both reconstructions);
    checked on interior cells (the box boundary uses ghost rules)."""
    n = 8
    w, a = 0.7, 0.4
    cases = [([[0, -w, 0], [w, 0, 0], [0, 0, 0]], w * w), ([[a, 0, 0], [0, -a, 0], [0, 0, 0]], -a * a)]
    for grad, want in cases:
        Q, G = _linear_velocity_case(n, grad)
        prob = oracle.Problem(n=(n, n, n), lo=(-0.5,) * 3, hi=(0.5,) * 3, scheme=scheme, mu=0.0,
                              bc=((2, 2), (2, 2), (2, 2)))
        q = oracle.qcriterion(prob, Q, G if scheme == 1 else None)
        inner = q[2:-2, 2:-2, 2:-2]
        assert np.abs(inner - want).max() < 1e-12, (scheme, want, inner.min(), inner.max())
