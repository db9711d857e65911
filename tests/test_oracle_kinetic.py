"""Pins of the oracle's kinetic layer (Maxwellian moments, micro-slopes, the
interface distribution of Eq. (flux) and its time integrals) against brute-force
velocity/time quadrature and closed physical limits -- never against the oracle's
own formulas.  PAPER.md: P:64-129."""
import math

import numpy as np
import pytest
from scipy import integrate, special

import oracle
from kinetic_quadrature import MaxwellQuad

GAMMA = 1.4


def test_internal_dof_value():
    # N = (5-3 gamma)/(gamma-1) = 2 for gamma = 1.4 (SPEC's N=1 is wrong).
    # The moment <xi^2> = N/(2 lam) enters the energy moment: check <psi5> = (3+N)/(4 lam) at U=0.
    q = MaxwellQuad(1.0, 0.0, 0.0, 0.0, 1.0)
    assert abs(q.mean(np.ones_like(q.u))[4] - 5.0 / 4.0) < 1e-12


@pytest.mark.parametrize("lam", [0.1, 1.0, 10.0])
@pytest.mark.parametrize("U", [-3.0, -0.7, 0.0, 1.3, 3.0])
@pytest.mark.parametrize("side", [-1, 0, 1])
def test_moments_vs_quadrature(lam, U, side):
    M = oracle.moments_1d(U, lam, side)
    sig = 1.0 / math.sqrt(2 * lam)
    pdf = lambda u: math.exp(-lam * (u - U) ** 2) * math.sqrt(lam / math.pi)
    lo, hi = (-np.inf, np.inf) if side == 0 else ((0.0, np.inf) if side > 0 else (-np.inf, 0.0))
    for k in range(9):
        ref, _ = integrate.quad(lambda u: u ** k * pdf(u), lo, hi, epsabs=0, epsrel=1e-13, limit=400)
        scale, _ = integrate.quad(lambda u: abs(u) ** k * pdf(u), -np.inf, np.inf, epsrel=1e-13, limit=400)
        assert abs(M[k] - ref) <= 1e-10 * max(scale, 1e-300), (k, M[k], ref)


def test_half_moment_value():
    # <u^1>_{u>0}(lam=1, U=0) = 1/(2 sqrt(pi)); <u^0>_{u>0} = 1/2
    M = oracle.moments_1d(0.0, 1.0, +1)
    assert abs(M[0] - 0.5) < 1e-16
    assert abs(M[1] - 1.0 / (2.0 * math.sqrt(math.pi))) < 1e-15


@pytest.mark.parametrize("U,lam", [(0.3, 0.7), (-2.0, 4.0), (2.5, 0.2)])
def test_half_complementarity(U, lam):
    a, b, f = oracle.moments_1d(U, lam, 1), oracle.moments_1d(U, lam, -1), oracle.moments_1d(U, lam, 0)
    assert np.allclose(a + b, f, rtol=1e-13, atol=1e-13 * np.abs(f).max())


def _rand_prim(rng):
    return np.array([rng.uniform(0.5, 2.0), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1),
                     rng.uniform(0.3, 3.0)])


def test_micro_slope_roundtrip():
    rng = np.random.default_rng(1)
    for _ in range(6):
        prim = _rand_prim(rng)
        b = rng.normal(size=5)
        a = oracle.micro_slope(prim, GAMMA, b)
        q = MaxwellQuad(prim[0], prim[1], prim[2], prim[3], prim[4])
        back = q.mean(q.slope(a))
        assert np.allclose(back, b, rtol=1e-10, atol=1e-10 * np.abs(b).max())


def test_micro_slope_zero_and_symmetry():
    assert np.all(oracle.micro_slope(np.array([1, 0, 0, 0, 1.0]), GAMMA, np.zeros(5)) == 0.0)
    # pure density slope at U=0: the odd coefficients vanish by symmetry
    a = oracle.micro_slope(np.array([1, 0, 0, 0, 1.0]), GAMMA, np.array([1.0, 0, 0, 0, 0]))
    assert np.allclose(a[1:4], 0.0, atol=1e-15)


def _coef_t(t, tau):
    """c_1..c_6(t) of Eq. (flux)."""
    if tau == 0.0:
        return np.array([1.0, 0.0, t, 0.0, 0.0, 0.0])
    e = math.exp(-t / tau)
    return np.array([1 - e, (t + tau) * e - tau, t - tau + tau * e, e, -(tau + t) * e, -tau * e])


@pytest.mark.parametrize("T,tau", [(0.01, 0.002), (1.0, 0.05), (0.3, 1.7), (0.2, 0.0)])
def test_time_integrals(T, tau):
    C = oracle.time_integrals(T, tau)
    for i in range(6):
        ref, _ = integrate.quad(lambda t: _coef_t(t, tau)[i], 0.0, T, epsabs=1e-15, epsrel=1e-13)
        assert abs(C[i] - ref) <= 1e-12 * max(T, T * T), (i, C[i], ref)


def test_uniform_state_flux():
    # rho=1, U=(1,0,0), p=1, gamma=1.4 -> F = (1,2,0,0,4); identical sides -> F_t = 0
    W = np.array([1.0, 1.0, 0.0, 0.0, 1.0 / 0.4 + 0.5])
    z = np.zeros((3, 5))
    for mu, Pr in [(0.0, 1.0), (1e-3, 0.72)]:
        d = oracle.flux_point(W, z, W, z, GAMMA, dt=0.01, mu=mu, Pr=Pr)
        assert np.allclose(d["Fn"], [1, 2, 0, 0, 4], rtol=1e-13, atol=1e-13)
        assert np.abs(d["Ft"]).max() < 1e-12
        assert np.allclose(d["Qn"], W, rtol=1e-13)


def test_collision_time_examples():
    # P:344-346 with eps=0.05, C=10; SPEC S:225-226 worked values
    def state(p):
        return np.array([1.0, 0, 0, 0, p / 0.4])
    z = np.zeros((3, 5))
    d = oracle.flux_point(state(1.0), z, state(1.0), z, GAMMA, dt=0.01)
    assert abs(d["tau"] - 0.05 * 0.01) < 1e-18
    d = oracle.flux_point(state(2.0), z, state(1.0), z, GAMMA, dt=0.01)
    assert abs(d["tau"] - (0.0005 + 10 * (1 / 3) * 0.01)) < 1e-15
    assert abs(d["tau"] - 0.0338333333333) < 1e-12
    # viscous smooth region: tau = mu/p
    d = oracle.flux_point(state(1.0), z, state(1.0), z, GAMMA, dt=0.01, mu=1e-3)
    assert abs(d["tau"] - 1e-3) < 1e-18


def test_relaxation_weight():
    # P:326-327 with tau0 = C0 |pl-pr|/(pl+pr) dt (R23): jump 1/3 and C0 = 3 give dt/tau0 = 1,
    # weight on Q^e = 1 - e^{-1} = 0.632121
    def state(p):
        return np.array([1.0, 0, 0, 0, p / 0.4])
    z = np.zeros((3, 5))
    WL, WR = state(2.0), state(1.0)
    d = oracle.flux_point(WL, z, WR, z, GAMMA, dt=0.01, relax_C=3.0)
    w = 0.6321205588285577
    assert np.allclose(d["QLn"], w * d["Qn"] + (1 - w) * WL, rtol=1e-14)
    assert np.allclose(d["QRn"], w * d["Qn"] + (1 - w) * WR, rtol=1e-14)
    # no pressure jump -> e^{-dt/tau0} = 0 -> both sides take Q^e
    d = oracle.flux_point(WL, z, WL * 1.0, z, GAMMA, dt=0.01)
    assert np.array_equal(d["QLn"], d["Qn"]) and np.array_equal(d["QRn"], d["Qn"])


def _random_face(rng, jump=0.2):
    def state():
        rho = rng.uniform(0.8, 1.2)
        u = rng.uniform(-0.5, 0.5, size=3)
        p = rng.uniform(0.8, 1.2)
        return np.array([rho, rho * u[0], rho * u[1], rho * u[2], p / 0.4 + 0.5 * rho * (u @ u)])
    WL = state()
    WR = WL + jump * (state() - WL)
    dWL = rng.normal(scale=0.3, size=(3, 5))
    dWR = rng.normal(scale=0.3, size=(3, 5))
    return WL, dWL, WR, dWR


def _prim(W):
    rho = W[0]
    U = W[1:4] / rho
    p = 0.4 * (W[4] - 0.5 * rho * U @ U)
    return rho, U, rho / (2 * p)


@pytest.mark.parametrize("seed", [3, 4])
def test_flux_intermediates_satisfy_definitions(seed):
    rng = np.random.default_rng(seed)
    WL, dWL, WR, dWR = _random_face(rng)
    d = oracle.flux_point(WL, dWL, WR, dWR, GAMMA, dt=0.01, mu=1e-3, Pr=1.0)
    rL, UL, lL = _prim(WL)
    rR, UR, lR = _prim(WR)
    qLh = MaxwellQuad(rL, *UL, lL, side=+1)
    qRh = MaxwellQuad(rR, *UR, lR, side=-1)
    qL = MaxwellQuad(rL, *UL, lL)
    qR = MaxwellQuad(rR, *UR, lR)
    # R13: W0 = int psi (g_l H + g_r (1-H))
    W0 = rL * qLh.mean(np.ones_like(qLh.u)) + rR * qRh.mean(np.ones_like(qRh.u))
    assert np.allclose(d["W0"], W0, rtol=1e-10)
    r0, U0, l0 = _prim(W0)
    q0 = MaxwellQuad(r0, *U0, l0)
    for al in range(3):
        # R15: <a psi> = dW / rho
        assert np.allclose(qL.mean(qL.slope(d["aL"][al])), dWL[al] / rL, atol=1e-10)
        assert np.allclose(qR.mean(qR.slope(d["aR"][al])), dWR[al] / rR, atol=1e-10)
        # R14: rho0 <abar psi> = rho_l <a^l psi>_{u>0} + rho_r <a^r psi>_{u<0}
        lhs = r0 * q0.mean(q0.slope(d["abar"][al]))
        rhs = rL * qLh.mean(qLh.slope(d["aL"][al])) + rR * qRh.mean(qRh.slope(d["aR"][al]))
        assert np.allclose(lhs, rhs, atol=1e-10)
    # R16: compatibility <(a.u + A) psi> = 0 (full moments)
    for q, a, A in [(qL, d["aL"], d["AL"]), (qR, d["aR"], d["AR"]), (q0, d["abar"], d["Abar"])]:
        f = sum(q.vel(al) * q.slope(a[al]) for al in range(3)) + q.slope(A)
        assert np.abs(q.mean(f)).max() < 1e-10


@pytest.mark.parametrize("seed,tau_mode", [(5, "visc"), (6, "inviscid"), (7, "zero")])
def test_flux_time_integral_brute_force(seed, tau_mode):
    """Fbar(T) = int_0^T int u psi f(t) dXi dt of Eq. (flux) by velocity quadrature of each
    term and Gauss-Legendre in time, using the oracle's coefficients; then F^n, F_t^n per P:115-116."""
    rng = np.random.default_rng(seed)
    WL, dWL, WR, dWR = _random_face(rng)
    dt = 0.02
    kw = dict(visc=dict(mu=2e-3), inviscid=dict(mu=0.0), zero=dict(mu=0.0, tau_eps=0.0, tau_C=0.0))[tau_mode]
    d = oracle.flux_point(WL, dWL, WR, dWR, GAMMA, dt=dt, Pr=1.0, **kw)
    tau = d["tau"]
    if tau_mode == "zero":
        assert tau == 0.0
    rL, UL, lL = _prim(WL)
    rR, UR, lR = _prim(WR)
    r0, U0, l0 = _prim(d["W0"])
    qLh, qRh, q0 = MaxwellQuad(rL, *UL, lL, side=+1), MaxwellQuad(rR, *UR, lR, side=-1), MaxwellQuad(r0, *U0, l0)

    def terms(q, rho, a, A, flux):
        fac = q.u if flux else np.ones_like(q.u)
        adotu = sum(q.vel(al) * q.slope(a[al]) for al in range(3))
        return [rho * q.mean(fac), rho * q.mean(fac * adotu), rho * q.mean(fac * q.slope(A))]

    for flux in (True, False):
        m0 = terms(q0, r0, d["abar"], d["Abar"], flux)
        mL = terms(qLh, rL, d["aL"], d["AL"], flux)
        mR = terms(qRh, rR, d["aR"], d["AR"], flux)
        vecs = [m0[0], m0[1], m0[2], mL[0] + mR[0], mL[1] + mR[1], mL[2] + mR[2]]
        g, gw = np.polynomial.legendre.leggauss(60)
        out = []
        for T in (dt, dt / 2):
            ts = 0.5 * T * (g + 1)
            Ci = sum(0.5 * T * w * _coef_t(t, tau) for t, w in zip(ts, gw))
            out.append(sum(Ci[i] * vecs[i] for i in range(6)))
        Fb, Fh = out
        if flux:
            assert np.allclose(d["Fbar_dt"], Fb, rtol=1e-9, atol=1e-12)
            assert np.allclose(d["Fbar_half"], Fh, rtol=1e-9, atol=1e-12)
            Fn, Ft = (4 * Fh - Fb) / dt, 4 * (Fb - 2 * Fh) / dt ** 2
            assert np.allclose(d["Fn"], Fn, rtol=1e-8, atol=1e-9)
            assert np.allclose(d["Ft"], Ft, rtol=1e-6, atol=1e-6 * np.abs(Fn).max() / dt)
        else:
            Qn, Qt = (4 * Fh - Fb) / dt, 4 * (Fb - 2 * Fh) / dt ** 2
            assert np.allclose(d["Qn"], Qn, rtol=1e-8, atol=1e-9)
            assert np.allclose(d["Qt"], Qt, rtol=1e-6, atol=1e-6 * np.abs(Qn).max() / dt)


def _ns_state(rho=1.0, p=1.0):
    return np.array([rho, 0.0, 0.0, 0.0, p / 0.4])


@pytest.mark.parametrize("Pr", [1.0, 0.72])
def test_navier_stokes_limit(Pr):
    """Chapman-Enskog limit of the BGK flux with tau = mu/p << dt (R20):
    shear stress mu dv/dx and Fourier heat flux -(mu c_p/Pr) dT/dx, c_p = gamma/(gamma-1)."""
    mu, dt, s = 1e-6, 1e-2, 0.1
    z = np.zeros((3, 5))
    W = _ns_state()
    # linear shear: v = s x (normal = x); d(rho v)/dx = s
    dW = z.copy()
    dW[0, 2] = s
    d = oracle.flux_point(W, dW, W, dW, GAMMA, dt=dt, mu=mu, Pr=Pr, tau_C=0.0)
    assert abs(d["Fn"][2] - (-mu * s)) < 1e-3 * mu * s
    # heat conduction: T = p/rho with p const: drho/dx = -s (T=1 at rho=p=1), d(rho E)/dx = 0
    dW = z.copy()
    dW[0, 0] = -s
    d = oracle.flux_point(W, dW, W, dW, GAMMA, dt=dt, mu=mu, Pr=Pr, tau_C=0.0)
    q_ref = -(GAMMA / (GAMMA - 1.0)) * mu / Pr * s
    assert abs(d["Fn"][4] - q_ref) < 2e-3 * abs(q_ref)
    assert abs(d["Fn"][1] - 1.0) < 1e-12  # pressure unchanged to first order


def _sutherland(mu0, T):
    # mu(T) = mu_0 1.4042 T^{3/2} / (T + 0.4042)
    return mu0 * 1.4042 * T ** 1.5 / (T + 0.4042)


@pytest.mark.parametrize("rho", [1.0, 0.5, 2.5])
def test_navier_stokes_limit_sutherland(rho):
    """High-speed TGV viscosity: with the Sutherland law the Chapman-Enskog shear
    stress of the BGK flux is mu(T) dv/dx with T = p/rho of the local state (here T = 1/rho), and
    mu(1) = mu_0."""
    mu0, dt, s = 1e-6, 1e-2, 0.1
    W = _ns_state(rho=rho, p=1.0)
    dW = np.zeros((3, 5))
    dW[0, 2] = rho * s  # v = s x
    d = oracle.flux_point(W, dW, W, dW, GAMMA, dt=dt, mu=mu0, Pr=1.0, tau_C=0.0, sutherland_S=0.4042)
    mu = _sutherland(mu0, 1.0 / rho)
    assert abs(d["Fn"][2] - (-mu * s)) < 1e-3 * mu * s
    if rho == 1.0:
        assert abs(mu - mu0) < 1e-22
    # collision time in a smooth region: tau = mu(T0) / p0
    z = np.zeros((3, 5))
    d = oracle.flux_point(W, z, W, z, GAMMA, dt=dt, mu=mu0, sutherland_S=0.4042)
    assert abs(d["tau"] - mu / 1.0) < 1e-15 * mu


def test_prandtl_fix_vanishes_in_euler_limit():
    # tau = 0: f = g0 + t Abar g0 is pure equilibrium, so the Pr fix must add nothing (R20 pitfall)
    rng = np.random.default_rng(11)
    WL, dWL, _, _ = _random_face(rng)
    a = oracle.flux_point(WL, dWL, WL, dWL, GAMMA, dt=0.01, Pr=0.72, tau_eps=0.0, tau_C=0.0)
    b = oracle.flux_point(WL, dWL, WL, dWL, GAMMA, dt=0.01, Pr=1.0, tau_eps=0.0, tau_C=0.0)
    assert np.allclose(a["Fn"], b["Fn"], rtol=1e-14, atol=1e-14)
    assert np.allclose(a["Ft"], b["Ft"], rtol=1e-12, atol=1e-12)
    # and with tau = 0 and smooth (WL == WR) data, F^n is the Euler flux of the state
    rho, U, lam = _prim(WL)
    p = rho / (2 * lam)
    euler = np.array([rho * U[0], rho * U[0] ** 2 + p, rho * U[0] * U[1], rho * U[0] * U[2], U[0] * (WL[4] + p)])
    assert np.allclose(b["Fn"], euler, rtol=1e-12)
