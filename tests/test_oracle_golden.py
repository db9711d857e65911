"""Oracle pinned to the worked values in tests/golden/worked_values.txt (each line cites the
paper or spec passage that prints it).  CPU only."""
import math
import os

import numpy as np

import oracle
from cgks_inputs import uniform

GAMMA = 1.4
HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    vals = {}
    with open(os.path.join(HERE, "golden", "worked_values.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                name, value = line.split()[:2]
                vals[name] = float(value)
    return vals


G = _golden()


def _state(p, rho=1.0):
    return np.array([rho, 0.0, 0.0, 0.0, p / (GAMMA - 1.0)])


def test_collision_time_golden():
    z = np.zeros((3, 5))
    dt = 0.01
    d = oracle.flux_point(_state(1.0), z, _state(1.0), z, GAMMA, dt=dt)
    assert abs(d["tau"] - G["tau_eps"] * dt) < 1e-18
    d = oracle.flux_point(_state(2.0), z, _state(1.0), z, GAMMA, dt=dt)
    assert abs(d["tau"] - (G["tau_eps"] + G["tau_C"] / 3.0) * dt) < 1e-16
    assert abs(d["tau"] - G["tau_pl2_pr1_dt001"]) < 1e-15
    d = oracle.flux_point(_state(1.0), z, _state(1.0), z, GAMMA, dt=dt, mu=1e-3)
    assert abs(d["tau"] - G["tau_viscous_mu1e-3_p1"]) < 1e-18


def test_relaxation_weight_golden():
    # tau0 = C0 |pl - pr| / (pl + pr) dt: jump 1/3 and C0 = 3 give dt / tau0 = 1
    z = np.zeros((3, 5))
    WL, WR = _state(2.0), _state(1.0)
    d = oracle.flux_point(WL, z, WR, z, GAMMA, dt=0.01, relax_C=3.0)
    # the weight w on Q^e, recovered from every component that differs between Q^e and W_L
    k = np.abs(d["Qn"] - WL) > 1e-3
    assert k.any()
    w = (np.asarray(d["QLn"])[k] - WL[k]) / (np.asarray(d["Qn"])[k] - WL[k])
    assert np.all(np.abs(w - G["relax_weight_at_1"]) < 5e-7)


def test_uniform_flux_golden():
    W = np.array([1.0, 1.0, 0.0, 0.0, 1.0 / (GAMMA - 1.0) + 0.5])
    z = np.zeros((3, 5))
    want = [G["uniform_flux_" + c] for c in ("rho", "mx", "my", "mz", "E")]
    for mu, Pr in [(0.0, 1.0), (1e-3, 0.72)]:
        d = oracle.flux_point(W, z, W, z, GAMMA, dt=0.01, mu=mu, Pr=Pr)
        assert np.allclose(d["Fn"], want, rtol=1e-13, atol=1e-13)


def _prob(c, cfl, mu=0.0):
    return oracle.Problem(**{**c.problem_kwargs(), "mu": mu, "cfl": cfl})


def test_dt_golden():
    c = uniform((4, 4, 4), state=(1.0, 0.0, 0.0, 0.0, 1.0 / GAMMA), L=2.0)
    assert abs(oracle.dt(_prob(c, 0.5), c.Q) - G["dt_convective"]) < 1e-15
    c = uniform((4, 4, 4), state=(1.0, 0.0, 0.0, 0.0, 1e-14), L=0.4)
    assert abs(oracle.dt(_prob(c, 0.3, mu=0.01), c.Q) - G["dt_viscous"]) < 1e-14


def test_sutherland_golden():
    # the oracle's viscous dt bound at T = p / rho = 4 carries mu(T) of P:474 (R25: nu = mu(T) / rho)
    c = uniform((4, 4, 4), state=(0.25, 0.0, 0.0, 0.0, 1.0), L=0.4)
    p = _prob(c, 0.3, mu=0.01)
    p.sutherland_S = G["sutherland_S"]
    T = 4.0
    mu_T = 0.01 * G["sutherland_a"] * T ** 1.5 / (T + G["sutherland_S"])
    want = 0.3 * min(0.1 / math.sqrt(GAMMA * T), 0.01 / (3.0 * mu_T / 0.25))
    assert abs(oracle.dt(p, c.Q) - want) < 1e-15 * want
