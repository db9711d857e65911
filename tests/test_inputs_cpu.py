"""Pins of the seeded input generators (cgks_inputs) that feed both the oracle and the GPU path:
the config-4 shock must satisfy the Rankine-Hugoniot jump conditions (textbook; SURVEY C3 row
"shock-vortex IC"), with the values of SURVEY D1 (BASELINE configs[3])."""
import numpy as np

from cgks_inputs import shock_vortex
from cgks_inputs.cases import rankine_hugoniot


def _euler_flux_x(rho, u, p, gamma):
    E = p / (gamma - 1.0) + 0.5 * rho * u * u
    return np.array([rho * u, rho * u * u + p, u * (E + p)])


def test_rankine_hugoniot_flux_continuity():
    gamma = 1.4
    (r1, u1, p1), (r2, u2, p2) = rankine_hugoniot(1.2, gamma)
    F1 = _euler_flux_x(r1, u1, p1, gamma)
    F2 = _euler_flux_x(r2, u2, p2, gamma)
    assert np.all(np.abs(F1 - F2) <= 4e-16 * np.abs(F1)), (F1, F2)
    # upstream Mach number 1.2 (c1 = 1), downstream subsonic, entropy increases
    assert abs(u1 / np.sqrt(gamma * p1 / r1) - 1.2) < 1e-15
    assert u2 / np.sqrt(gamma * p2 / r2) < 1.0
    assert p2 / r2 ** gamma > p1 / r1 ** gamma
    # SURVEY D1 values (7 digits)
    assert abs(r2 - 1.3416149) < 5e-8 and abs(u2 - 0.8944444) < 5e-8 and abs(p2 / p1 - 1.5133333) < 5e-8


def test_shock_vortex_ic_states():
    gamma = 1.4
    case = shock_vortex(nx=64, ny=32)
    (r1, u1, p1), (r2, u2, p2) = rankine_hugoniot(1.2, gamma)
    x = (np.arange(64) + 0.5) * 2.0 / 64
    down = x > 0.55  # cells entirely behind the shock at x = 0.5
    Q = case.Q[:, 0, :, down]  # (ncell_x, 5, ny) after fancy indexing
    Q = np.moveaxis(Q, 0, -1)
    E2 = p2 / (gamma - 1.0) + 0.5 * r2 * u2 * u2
    want = np.array([r2, r2 * u2, 0.0, 0.0, E2])
    assert np.allclose(Q, want[:, None, None], rtol=1e-14, atol=1e-15)
    # inflow Dirichlet state = the upstream RH state (R29)
    E1 = p1 / (gamma - 1.0) + 0.5 * r1 * u1 * u1
    assert np.allclose(case.bc_state[0, 0], [r1, r1 * u1, 0.0, 0.0, E1], rtol=1e-15)
