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
