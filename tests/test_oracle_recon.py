"""Pins of the oracle's reconstructions against exactly integrated
polynomials (independent 1-D antiderivatives), rank checks and limiter limits."""
import numpy as np
import pytest

import oracle


def _avg1(k, a, b):
    """average of x^k over [a, b]"""
    return (b ** (k + 1) - a ** (k + 1)) / ((k + 1) * (b - a))


def poly_case(dim, deg, seed, n=5, h=(0.3, 0.25, 0.2)):
    """Random polynomial of total degree <= deg over the active axes; exact cell averages and exact
    cell-averaged gradients on an n^dim grid.  Returns (prob, Q, G, f, grad f)."""
    rng = np.random.default_rng(seed)
    terms = []
    for i in range(deg + 1):
        for j in range(deg + 1 - i):
            for k in range(deg + 1 - i - j):
                if (dim < 2 and j) or (dim < 3 and k):
                    continue
                terms.append(((i, j, k), rng.normal()))
    nn = [n if a < dim else 1 for a in range(3)]
    hh = [h[a] for a in range(3)]
    lo = [0.0, 0.0, 0.0]
    hi = [nn[a] * hh[a] for a in range(3)]
    edges = [lo[a] + hh[a] * np.arange(nn[a] + 1) for a in range(3)]
    Q = np.zeros((5, nn[2], nn[1], nn[0]))
    G = np.zeros((3, 5, nn[2], nn[1], nn[0]))
    for (e, c) in terms:
        A = [np.array([_avg1(e[a], edges[a][q], edges[a][q + 1]) for q in range(nn[a])]) for a in range(3)]
        D = [np.array([(edges[a][q + 1] ** e[a] - edges[a][q] ** e[a]) / hh[a] for q in range(nn[a])])
             for a in range(3)]
        Q[:] += c * (A[2][:, None, None] * A[1][None, :, None] * A[0][None, None, :])[None]
        G[0] += c * (A[2][:, None, None] * A[1][None, :, None] * D[0][None, None, :])[None]
        G[1] += c * (A[2][:, None, None] * D[1][None, :, None] * A[0][None, None, :])[None]
        G[2] += c * (D[2][:, None, None] * A[1][None, :, None] * A[0][None, None, :])[None]
    # make the five components different (scaled copies) and keep density/pressure positive
    scale = np.array([1.0, -0.5, 0.25, 0.7, 2.0])
    Q = Q * scale[:, None, None, None]
    G = G * scale[None, :, None, None, None]

    def f(x):
        return sum(c * x[0] ** e[0] * x[1] ** e[1] * x[2] ** e[2] for (e, c) in terms) * scale

    def df(x):
        out = np.zeros((3, 5))
        for (e, c) in terms:
            for a in range(3):
                if e[a] == 0:
                    continue
                ee = list(e)
                ee[a] -= 1
                out[a] += c * e[a] * x[0] ** ee[0] * x[1] ** ee[1] * x[2] ** ee[2] * scale
        return out

    prob = oracle.Problem(n=tuple(nn), lo=tuple(lo), hi=tuple(hi), scheme=1)
    return prob, Q, G, f, df, hh, [nn[a] // 2 for a in range(3)]


@pytest.mark.parametrize("dim,nb,nd", [(3, 34, 63), (2, 14, 26), (1, 4, 5)])
def test_cls_rank_and_sizes(dim, nb, nd):
    r = oracle.recon5_matrix(dim)
    assert r["rank_ok"] and r["nb"] == nb and r["nd"] == nd
    assert r["nc"] == {3: 18, 2: 8, 1: 2}[dim]
    # constant data (all differences and derivatives zero) -> zero coefficients: R @ 0 = 0 trivially;
    # the matrix must reproduce the exact constraints: C @ R[:, :nc] = I (checked via quartic exactness below)


@pytest.mark.parametrize("dim,seed", [(3, 0), (3, 1), (2, 2), (1, 3)])
def test_cls_quartic_exactness(dim, seed):
    # consistent data from any quartic are reproduced exactly (chi == 1, linear mode)
    prob, Q, G, f, df, h, c = poly_case(dim, 4, seed)
    rng = np.random.default_rng(seed + 100)
    x = rng.uniform(-0.5, 0.5, size=(6, 3))
    x[:, dim:] = 0.0
    W, dW, _ = oracle.recon_eval(prob, Q, G, c, x)
    for q in range(x.shape[0]):
        xp = [(c[a] + 0.5 + x[q, a]) * h[a] if a < dim else 0.5 * h[a] for a in range(3)]
        ref, dref = f(xp), df(xp)
        sc = np.abs(Q).max()
        assert np.allclose(W[q], ref, rtol=0, atol=1e-11 * sc)
        assert np.allclose(dW[q][:dim], dref[:dim], rtol=0, atol=1e-10 * np.abs(G).max())


def test_cls_quintic_is_not_reproduced():
    # sanity: the reconstruction is exactly quartic (a degree-5 field is not reproduced)
    prob, Q, G, f, df, h, c = poly_case(2, 5, 9)
    x = np.array([[0.5, 0.2, 0.0]])
    W, dW, _ = oracle.recon_eval(prob, Q, G, c, x)
    xp = [(c[a] + 0.5 + x[0, a]) * h[a] if a < 2 else 0.5 * h[a] for a in range(3)]
    assert np.abs(W[0] - f(xp)).max() > 1e-8


def test_constant_field_exact():
    prob, Q, G, f, df, h, c = poly_case(3, 0, 4)
    x = np.array([[0.5, 0.28, -0.28], [-0.5, 0.1, 0.4]])
    for nl in (0, 1):
        prob.nonlinear = nl
        W, dW, chi = oracle.recon_eval(prob, Q, G, c, x)
        assert np.array_equal(W, np.broadcast_to(Q[:, 2, 2, 2], W.shape))
        assert np.all(dW == 0.0)


def test_geno_linear_field_is_exact_and_chi_one():
    # equal smoothness indicators on linear data: omega_m = 1/6, chi = 1, reproduction exact
    prob, Q, G, f, df, h, c = poly_case(3, 1, 5)
    prob.nonlinear = 1
    x = np.array([[0.5, 0.288675, -0.288675], [0.1, -0.5, 0.3]])
    W, dW, chi = oracle.recon_eval(prob, Q, G, c, x)
    assert np.all(chi > 1 - 1e-12)
    for q in range(2):
        xp = [(c[a] + 0.5 + x[q, a]) * h[a] for a in range(3)]
        assert np.allclose(W[q], f(xp), atol=1e-12 * np.abs(Q).max())


def test_geno_step_is_eno():
    # a jump at the face between cells 1 and 2 along x: cell 2's reconstruction drops to
    # the ENO sub-stencils (chi -> 0) and its face values stay within the data range
    n = 5
    Q = np.zeros((5, n, n, n))
    Q[0] = 1.0
    Q[4] = 2.5
    Q[0][:, :, 2:] = 2.0
    Q[4][:, :, 2:] = 5.0
    G = np.zeros((3, 5, n, n, n))
    prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(1, 1, 1), scheme=1, nonlinear=1)
    x = np.array([[-0.5, 0.288675, 0.288675], [0.5, -0.288675, 0.288675], [-0.5, 0.0, 0.0]])
    W, dW, chi = oracle.recon_eval(prob, Q, G, (2, 2, 2), x)
    assert chi[0] < 1e-6 and chi[4] < 1e-6
    # chi ~ 1e-8 at an O(1) jump (R8): the overshoot left is chi * (Gibbs overshoot of P^4)
    assert np.all(W[:, 0] >= 1.0 - 1e-6) and np.all(W[:, 0] <= 2.0 + 1e-6)
    # the linear quartic overshoots here (Gibbs); GENO must not
    prob.nonlinear = 0
    Wl, _, _ = oracle.recon_eval(prob, Q, G, (2, 2, 2), x)
    assert Wl[:, 0].min() < 1.0 - 1e-3 or Wl[:, 0].max() > 2.0 + 1e-3


def test_gks2_linear_exact_and_venkat():
    prob, Q, G, f, df, h, c = poly_case(3, 1, 6)
    prob.scheme = 0
    x = np.array([[0.5, 0.0, 0.0], [0.0, -0.5, 0.0]])
    for nl in (0, 1):
        prob.nonlinear = nl
        W, dW, phi = oracle.recon_eval(prob, Q, G, c, x)
        # LS on a uniform stencil reproduces linear fields; Venkatakrishnan gives phi = 1 on monotone linear data
        assert np.all(np.abs(phi - 1.0) < 1e-12)
        for q in range(2):
            xp = [(c[a] + 0.5 + x[q, a]) * h[a] for a in range(3)]
            assert np.allclose(W[q], f(xp), atol=1e-12 * np.abs(Q).max())
            assert np.allclose(dW[q], df(xp), atol=1e-11 * np.abs(G).max())


def test_venkat_extremum_and_constant():
    n = 5
    Q = np.ones((5, n, n, n))
    Q[4] = 2.5
    G = np.zeros((3, 5, n, n, n))
    prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(1, 1, 1), scheme=0, nonlinear=1)
    W, dW, phi = oracle.recon_eval(prob, Q, G, (2, 2, 2), np.array([[0.5, 0, 0]]))
    assert np.all(phi == 1.0)
    # strict local maximum in x at cell 2 with asymmetric neighbours -> phi0 < 1
    Q[0][:, :, 1] = 0.9
    Q[0][:, :, 2] = 1.3
    Q[0][:, :, 3] = 1.0
    W, dW, phi = oracle.recon_eval(prob, Q, G, (2, 2, 2), np.array([[0.5, 0, 0]]))
    assert phi[0] < 1.0
    assert phi[0] >= 0.0


def test_venkat_closed_form_value():
    """Venkatakrishnan's limiter function (R11) on data that fix every term: along x the averages are
    0.5, 1, 3 (h = 1), so the LS slope is 1.25 per cell; at the + face D2 = 0.625, D1 = qmax - q0 = 2 gives
    phi > 1 (clipped), at the - face D2 = -0.625, D1 = qmin - q0 = -0.5 gives
    phi = (D1^2 + e2 + 2 D1 D2) / (D1^2 + 2 D2^2 + D1 D2 + e2), e2 = (K h)^3 = 0.027 (K = 0.3): the textbook form
    (Venkatakrishnan 1995).  The cell takes the minimum over its faces."""
    n = 5
    Q = np.ones((5, n, n, n))
    Q[4] = 2.5
    Q[0][:, :, 1] = 0.5
    Q[0][:, :, 2] = 1.0
    Q[0][:, :, 3] = 3.0
    G = np.zeros((3, 5, n, n, n))
    prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(n, n, n), scheme=0, nonlinear=1)
    W, dW, phi = oracle.recon_eval(prob, Q, G, (2, 2, 2), np.array([[0.5, 0, 0], [-0.5, 0, 0]]))
    d1, d2, e2 = -0.5, -0.625, 0.3 ** 3
    want = (d1 * d1 + e2 + 2 * d1 * d2) / (d1 * d1 + 2 * d2 * d2 + d1 * d2 + e2)
    assert want == pytest.approx(0.902 / 1.37075, rel=1e-14)
    assert phi[0] == pytest.approx(want, rel=1e-14)
    assert np.all(phi[1:] == 1.0)
    assert W[0, 0] == pytest.approx(1.0 + want * 0.625, rel=1e-14) and W[1, 0] == pytest.approx(1.0 - want * 0.625, rel=1e-14)
    assert dW[0, 0, 0] == pytest.approx(want * 1.25, rel=1e-14)
    # a smaller K sharpens the limiter: e2 -> 0 gives (D1^2 + 2 D1 D2) / (D1^2 + 2 D2^2 + D1 D2)
    prob.k_venkat = 1e-6
    _, _, phi0 = oracle.recon_eval(prob, Q, G, (2, 2, 2), np.array([[0.5, 0, 0]]))
    assert phi0[0] == pytest.approx((0.25 + 0.625) / (0.25 + 0.78125 + 0.3125), rel=1e-12)


def test_geno_chi_scale_closed_form():
    # chi_scale C divides zeta (R8): chi_C = 1 / (1 + (zeta_1 / C)^4), zeta_1 = (1/chi_1 - 1)^(1/4),
    # checked on a curved field where the sub-stencil contrast gives an intermediate chi
    n = 5
    ax = np.arange(n) - 2.0
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    Q = np.zeros((5, n, n, n))
    Q[0] = 1.0 + 0.05 * X + 0.01 * X ** 2 + 0.01 * Y
    Q[4] = 2.5 + 0.1 * Z ** 2
    G = np.zeros((3, 5, n, n, n))
    G[0, 0] = 0.05 + 0.02 * X
    G[1, 0] = 0.01
    G[2, 4] = 0.2 * Z
    x = np.array([[0.5, 0.0, 0.0]])
    chis = {}
    for C in (1.0, 4.0, 8.0):
        prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(n, n, n), scheme=1, nonlinear=1, chi_scale=C)
        _, _, chi = oracle.recon_eval(prob, Q, G, (2, 2, 2), x)
        chis[C] = chi
    c1 = chis[1.0][0]
    assert 0.01 < c1 < 0.99, c1
    z1 = (1.0 / c1 - 1.0) ** 0.25
    for C in (4.0, 8.0):
        assert chis[C][0] == pytest.approx(1.0 / (1.0 + (z1 / C) ** 4), rel=1e-12)
        assert chis[C][0] > c1


def test_geno_chi_scale_keeps_eno_at_a_jump():
    n = 5
    Q = np.zeros((5, n, n, n))
    Q[0] = 1.0
    Q[4] = 2.5
    Q[0][:, :, 2:] = 2.0
    Q[4][:, :, 2:] = 5.0
    G = np.zeros((3, 5, n, n, n))
    prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(1, 1, 1), scheme=1, nonlinear=1, chi_scale=8.0)
    _, _, chi = oracle.recon_eval(prob, Q, G, (2, 2, 2), np.array([[-0.5, 0.0, 0.0]]))
    assert chi[0] < 1e-4 and chi[4] < 1e-4


# ---- GENO nonlinear weights: omega_m = wbar_m / sum_k wbar_k, wbar_m = d_m / (IS_m + eps)^5,
# d_m = 1/6, eps = 1e-15 (SPEC S:374-376 lists the pins: equal IS => 1/6, power-5 suppression) --------
def _geno_block(slopes_minus, slopes_plus, own_grad, h=1.0, n=5):
    """3-D n^3 periodic block, centre cell c = (2,2,2): the six face neighbours differ from Q_0 by the
    given reference-unit slopes (minus side: Q_0 - Q_{-a} = slopes_minus[a]; plus side: Q_{+a} - Q_0 =
    slopes_plus[a]), own cell-averaged gradient own_grad (physical units, h = 1 so reference = physical).
    The same numbers in all five components (scaled), rho and rho E kept positive."""
    Q = np.zeros((5, n, n, n))
    G = np.zeros((3, 5, n, n, n))
    c = n // 2
    base = np.array([2.0, 0.3, -0.2, 0.1, 9.0])
    Q[:] = base[:, None, None, None]
    scale = np.array([1.0, 0.5, 0.25, 0.125, 2.0])
    for a in range(3):
        lo = [c, c, c]
        hi = [c, c, c]
        lo[a] -= 1
        hi[a] += 1
        Q[(slice(None), lo[2], lo[1], lo[0])] = base - scale * slopes_minus[a]
        Q[(slice(None), hi[2], hi[1], hi[0])] = base + scale * slopes_plus[a]
        G[a, :, c, c, c] = scale * own_grad[a] / h
    prob = oracle.Problem(n=(n, n, n), lo=(0, 0, 0), hi=(n * h,) * 3, scheme=1, nonlinear=1)
    return prob, Q, G, (c, c, c)


def test_geno_weights_equal_is_give_one_sixth():
    # linear data with equal reference slopes on every axis: all six IS_m equal => omega_m = d_m = 1/6
    prob, Q, G, c = _geno_block([0.3] * 3, [0.3] * 3, [0.3] * 3)
    IS, om, _, chi = oracle.geno_cell(prob, Q, G, c)
    assert np.allclose(IS, IS[0, 0] * np.array([1.0, 0.5, 0.25, 0.125, 2.0]) ** 2 / 1.0, rtol=1e-14)
    assert np.all(np.abs(om - 1.0 / 6.0) <= 4e-16), om
    assert np.all(chi == 1.0)


def test_geno_weights_power5_suppression():
    # one sub-stencil (plus side of x) with IS ~1.3e6 x the others: its weight is below 1e-29
    # (d/(r IS)^5 against five of d/IS^5: (1/r^5) / 5 ~ 5e-32), the other five share the rest equally
    prob, Q, G, c = _geno_block([0.3] * 3, [600.0, 0.3, 0.3], [0.3] * 3)
    IS, om, _, _ = oracle.geno_cell(prob, Q, G, c)
    ratio = IS[1] / IS[0]
    assert np.all(ratio > 1e6)
    assert np.all(om[1] < 1e-29), om[1]
    others = om[[0, 2, 3, 4, 5]]
    assert np.allclose(others, 0.2, rtol=1e-14, atol=0.0)


@pytest.mark.parametrize("r", [2.0, 4.0, 10.0])
def test_geno_weights_known_ratios(r):
    """IS ratios fixed by the data: the minus-x sub-stencil has IS_0 = 3 s^2 r, the other five IS = 3 s^2
    (plus its own transverse slopes), so omega_0 = r^-5 / (r^-5 + 5) and omega_m = 1 / (r^-5 + 5) --
    the exponent 5 of P:268 decides the values (exponent 1 would give 1/(5 r + 1))."""
    s = 0.3
    # minus-x slope b with b^2 + 2 s^2 = 3 s^2 r  =>  b = s sqrt(3 r - 2)
    b = s * np.sqrt(3.0 * r - 2.0)
    prob, Q, G, c = _geno_block([b, s, s], [s, s, s], [s, s, s])
    IS, om, _, chi = oracle.geno_cell(prob, Q, G, c)
    assert np.allclose(IS[0] / IS[1], r, rtol=1e-13)
    # R7: IS_m = sum of the squared reference slopes of sub-stencil m (component v scaled by scale[v])
    scale = np.array([1.0, 0.5, 0.25, 0.125, 2.0])
    assert np.allclose(IS[1], 3.0 * s * s * scale ** 2, rtol=1e-13)
    w0 = r ** -5 / (r ** -5 + 5.0)
    assert np.allclose(om[0], w0, rtol=1e-13), (om[0], w0)
    assert np.allclose(om[1:], 1.0 / (r ** -5 + 5.0), rtol=1e-13)
    # R8 (the reading DESIGN.md adopts; the paper defers chi to its references): chi = 1 / (1 + zeta^4),
    # zeta = (IS_max - IS_min) / (IS_min + eps + 0.01 IS_max) -- with IS_max = r IS_min a function of r alone
    # (r = 2 gives chi = 0.52: the blend is half ENO already at a factor 2 between the indicators)
    zeta = (r - 1.0) / (1.0 + 0.01 * r)
    assert np.allclose(chi, 1.0 / (1.0 + zeta ** 4), rtol=1e-10), chi


def test_geno_blend_value_1d_known_ratio():
    """The blended face value of P:259-263 in 1-D: Q(x_G) = chi P^4(x_G) + (1 - chi) sum_m omega_m P_m^1(x_G).
    Data (Q_{-1}, Q_0, Q_{+1}) = (Q_0 - c, Q_0, Q_0 + 2c): sub-stencil slopes c and 2c, IS ratio 4, so
    omega = (1024/1025, 1/1025) and sum_m omega_m P_m^1(1/2) = Q_0 + (1026/1025) c / 2.  P^4 is the linear
    scheme's value of the same data (nonlinear = 0); chi is the oracle's (R8, parity unpinned)."""
    n = 7
    h = 0.5
    c = 0.04
    Q = np.zeros((5, 1, 1, n))
    base = np.array([1.0, 0.2, 0.0, 0.0, 2.5])
    Q[:] = base[:, None, None, None]
    i0 = 3
    Q[:, 0, 0, i0 - 1] = base - c
    Q[:, 0, 0, i0 + 1] = base + 2 * c
    Q[2:4] = 0.0
    G = np.zeros((3,) + Q.shape)
    G[0, :, 0, 0, i0] = 1.5 * c / h
    G[0, 2:4] = 0.0
    kw = dict(n=(n, 1, 1), lo=(0, 0, 0), hi=(n * h, 1, 1), scheme=1)
    x = np.array([[0.5, 0.0, 0.0], [-0.5, 0.0, 0.0]])
    Wl, dWl, _ = oracle.recon_eval(oracle.Problem(**kw, nonlinear=0), Q, G, (i0, 0, 0), x)
    Wn, dWn, chi = oracle.recon_eval(oracle.Problem(**kw, nonlinear=1), Q, G, (i0, 0, 0), x)
    assert np.all((chi[[0, 1, 4]] > 0.0) & (chi[[0, 1, 4]] < 1.0))
    slope = 1026.0 / 1025.0 * c  # reference units
    for v in (0, 1, 4):
        for p, xr in enumerate((0.5, -0.5)):
            lin = base[v] + slope * xr
            want = chi[v] * Wl[p, v] + (1.0 - chi[v]) * lin
            assert abs(Wn[p, v] - want) <= 1e-14 * abs(want), (v, p, Wn[p, v], want)
            dwant = chi[v] * dWl[p, 0, v] + (1.0 - chi[v]) * slope / h
            assert abs(dWn[p, 0, v] - dwant) <= 1e-13 * abs(dwant), (v, p, dWn[p, 0, v], dwant)


def test_geno_weights_epsilon():
    """eps = 1e-15 of P:270 enters as (IS_m + eps): five flat sub-stencils (IS = 0) and one with IS = eps
    give omega = (2 eps)^-5 / ((2 eps)^-5 + 5 eps^-5) = 1/161 for that one (a dropped eps would give 0)."""
    s = np.sqrt(1e-15)
    prob, Q, G, c = _geno_block([0.0] * 3, [s, 0.0, 0.0], [0.0] * 3)
    IS, om, _, _ = oracle.geno_cell(prob, Q, G, c)
    assert abs(IS[1, 0] - 1e-15) <= 1e-22 and np.all(IS[[0, 2, 3, 4, 5], 0] == 0.0)
    assert abs(om[1, 0] - 1.0 / 161.0) <= 1e-6 / 161.0, om[1, 0]
    assert np.allclose(om[[0, 2, 3, 4, 5], 0], 32.0 / 161.0, rtol=1e-6)
