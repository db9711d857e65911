"""Initial-condition generators (seeded, synthetic) for the five BASELINE configs and
the verification problems.  Each returns a :class:`Case` with exact cell averages Q
and exact cell-averaged gradients G (Gauss theorem on Gauss-Legendre face averages,
reading R26), in the layout ``Q[5][nz][ny][nx]``, ``G[3][5][nz][ny][nx]``.

Definitions follow SURVEY.md section 8(d) D1 (BASELINE.json configs) and PAPER.md
P:379-395 (Taylor-Green vortex).  Nothing here implements the scheme.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PI = math.pi


@dataclass
class Case:
    name: str
    n: tuple
    lo: tuple
    hi: tuple
    Q: np.ndarray
    G: np.ndarray
    gamma: float = 1.4
    mu: float = 0.0
    Pr: float = 1.0
    bc: tuple = ((0, 0), (0, 0), (0, 0))
    bc_state: np.ndarray = field(default_factory=lambda: np.zeros((3, 2, 5)))
    # recommended scheme settings for this config (not part of the IC)
    cfl: float = 0.5
    nonlinear: int = 0
    tau_eps: float = 0.05
    tau_C: float = 10.0
    relax_C: float = 10.0
    steps: int = 10
    note: str = ""
    sutherland_S: float = 0.0  # 0: constant mu; 0.4042: Sutherland law

    @property
    def ncell(self) -> int:
        return int(np.prod(self.n))

    @property
    def dim(self) -> int:
        return 3 if self.n[2] > 1 else (2 if self.n[1] > 1 else 1)

    def problem_kwargs(self) -> dict:
        """Physical and scheme parameters as keyword arguments (shared by both arms)."""
        return dict(n=tuple(self.n), lo=tuple(self.lo), hi=tuple(self.hi), gamma=self.gamma, mu=self.mu,
                    Pr=self.Pr, bc=self.bc, bc_state=np.array(self.bc_state), cfl=self.cfl,
                    nonlinear=self.nonlinear, tau_eps=self.tau_eps, tau_C=self.tau_C, relax_C=self.relax_C,
                    sutherland_S=self.sutherland_S)


def prim_to_cons(rho, u, v, w, p, gamma):
    E = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
    return np.stack([rho, rho * u, rho * v, rho * w, E])


def _gl(nq):
    x, w = np.polynomial.legendre.leggauss(nq)
    return 0.5 * x, 0.5 * w  # nodes on [-1/2, 1/2], weights sum to 1


def gl_average(fprim, n, lo, hi, gamma, nq=4, nudge=1e-11, mesh_nodes=None):
    """Cell averages and cell-averaged gradients of cons(fprim(x, y, z)) by
    nq-point Gauss-Legendre per active axis; gradient by the Gauss theorem
    (face averages of the point values, evaluated just inside the cell).
    mesh_nodes: per-axis node coordinates of a stretched tensor-product mesh (or None: uniform)."""
    n = tuple(int(a) for a in n)
    dim = 3 if n[2] > 1 else (2 if n[1] > 1 else 1)
    if mesh_nodes is None:
        h = [(hi[a] - lo[a]) / n[a] * np.ones(n[a]) for a in range(3)]
        centres = [lo[a] + (np.arange(n[a]) + 0.5) * (hi[a] - lo[a]) / n[a] for a in range(3)]
    else:
        h = [np.diff(np.asarray(mesh_nodes[a], dtype=np.float64)) for a in range(3)]
        centres = [0.5 * (np.asarray(mesh_nodes[a])[1:] + np.asarray(mesh_nodes[a])[:-1]) for a in range(3)]
    xi, wi = _gl(nq)
    nodes = [(xi, wi) if a < dim else (np.zeros(1), np.ones(1)) for a in range(3)]

    def fcons(x, y, z):
        return prim_to_cons(*fprim(x, y, z), gamma)

    Q = np.zeros((5, n[2], n[1], n[0]))
    G = np.zeros((3, 5, n[2], n[1], n[0]))
    for k in range(n[2]):
        zc = centres[2][k]
        Z3, Y3, X3 = np.meshgrid([zc], centres[1], centres[0], indexing="ij")
        H3 = [h[0][None, None, :], h[1][None, :, None], np.array(h[2][k])[None, None, None]]
        # volume average
        acc = np.zeros((5, 1, n[1], n[0]))
        for (pz, wz) in zip(*nodes[2]):
            for (py, wy) in zip(*nodes[1]):
                for (px, wx) in zip(*nodes[0]):
                    acc += wx * wy * wz * fcons(X3 + px * H3[0], Y3 + py * H3[1], Z3 + pz * H3[2])
        Q[:, k] = acc[:, 0]
        # Gauss theorem: (face avg at +1/2 - face avg at -1/2)/h along each active axis
        for a in range(dim):
            face = []
            for side in (+1, -1):
                acc = np.zeros((5, 1, n[1], n[0]))
                off = side * (0.5 - nudge)
                tn = [nodes[b] if b != a else (np.array([off]), np.ones(1)) for b in range(3)]
                for (pz, wz) in zip(*tn[2]):
                    for (py, wy) in zip(*tn[1]):
                        for (px, wx) in zip(*tn[0]):
                            acc += wx * wy * wz * fcons(X3 + px * H3[0], Y3 + py * H3[1], Z3 + pz * H3[2])
                face.append(acc[:, 0])
            G[a, :, k] = (face[0] - face[1]) / H3[a][0]
    return Q, G


def stretched_nodes(n: int, lo: float, hi: float, beta: float = 0.0, kind: str = "sine"):
    """Node coordinates of a smoothly stretched axis (NEXT-4; tensor-product meshes of the jet runs,
    P:574-594): 'sine' x = lo + L (s + beta sin(2 pi s) / (2 pi)) on s = k/n (periodic-compatible,
    spacing ratio (1 + beta) / (1 - beta)); 'tanh' clusters nodes at the centre (jet shear layer):
    x = lo + L (1 + tanh(beta (s - 1/2)) / tanh(beta / 2)) / 2."""
    s_ = np.arange(n + 1) / n
    L = hi - lo
    if kind == "sine":
        return lo + L * (s_ + beta * np.sin(2 * math.pi * s_) / (2 * math.pi))
    if kind == "tanh":
        return lo + L * 0.5 * (1.0 + np.tanh(beta * (s_ - 0.5)) / math.tanh(0.5 * beta))
    raise ValueError(kind)


def jet_inflow(r, M_j=0.9, T_j=1.0, T_inf=1.0, R0=0.5, theta=0.02, gamma=1.4):
    """Round-jet inflow profile (NEXT-4 input generator, the jet runs of P:574-594 stay out of scope):
    hyperbolic-tangent axial velocity u(r) = (U_j/2)(1 + tanh((R0 - r)/(2 theta))), with the Crocco-Busemann
    relation for the temperature, T = T_inf + (T_j - T_inf) u/U_j + (gamma-1)/2 M_j^2 T_j (u/U_j)(1 - u/U_j),
    uniform pressure p = 1/gamma (sound speed 1 at T = 1), rho = gamma p / T.  Returns (rho, u, p)."""
    Uj = M_j * math.sqrt(T_j)
    u = 0.5 * Uj * (1.0 + np.tanh((R0 - np.asarray(r)) / (2.0 * theta)))
    f = u / Uj
    T = T_inf + (T_j - T_inf) * f + 0.5 * (gamma - 1.0) * M_j ** 2 * T_j * f * (1.0 - f)
    p = np.full_like(u, 1.0 / gamma)
    rho = gamma * p / T
    return rho, u, p


def line_points(dim: int, a: int):
    """Transverse Gauss-point offsets (reference units) of the line-averaged derivatives along axis a:
    g = p * n2 + q, p the sign (-, +) along t1 = (a+1)%3, q along t2 = (a+2)%3 (active axes only)."""
    gq = 0.5 / math.sqrt(3.0)
    t1, t2 = (a + 1) % 3, (a + 2) % 3
    n1 = 2 if t1 < dim else 1
    n2 = 2 if t2 < dim else 1
    pts = []
    for p_ in range(n1):
        for q_ in range(n2):
            t = [0.0, 0.0, 0.0]
            if t1 < dim:
                t[t1] = -gq if p_ == 0 else gq
            if t2 < dim:
                t[t2] = -gq if q_ == 0 else gq
            pts.append(t)
    return pts


def line_derivatives(fprim, n, lo, hi, gamma, mesh_nodes=None):
    """Exact line-averaged derivatives of cons(fprim(x, y, z)) for the line-DOF variant:
    (Q(x_c + h_a/2 e_a + t) - Q(x_c - h_a/2 e_a + t)) / h_a at the transverse Gauss points t of each axis
    (offsets in units of the cell's own widths); layout [nlines][5][nz][ny][nx] (see line_points).
    mesh_nodes: optional per-axis node arrays of a stretched mesh (NEXT-4), as in gl_average."""
    n = tuple(int(a) for a in n)
    dim = 3 if n[2] > 1 else (2 if n[1] > 1 else 1)
    c, hh = [], []
    for a in range(3):
        nd = None if mesh_nodes is None else mesh_nodes[a]
        if nd is None:
            ha = (hi[a] - lo[a]) / n[a]
            c.append(lo[a] + (np.arange(n[a]) + 0.5) * ha)
            hh.append(np.full(n[a], ha))
        else:
            nd = np.asarray(nd, dtype=np.float64)
            c.append(0.5 * (nd[1:] + nd[:-1]))
            hh.append(np.diff(nd))
    Z, Y, X = np.meshgrid(c[2], c[1], c[0], indexing="ij")
    HZ, HY, HX = np.meshgrid(hh[2], hh[1], hh[0], indexing="ij")
    h = [HX, HY, HZ]
    Z, Y, X = np.meshgrid(c[2], c[1], c[0], indexing="ij")
    pos = [X, Y, Z]
    out = []
    for a in range(dim):
        for t in line_points(dim, a):
            xp = [pos[b] + t[b] * h[b] + (0.5 * h[a] if b == a else 0.0) for b in range(3)]
            xm = [pos[b] + t[b] * h[b] - (0.5 * h[a] if b == a else 0.0) for b in range(3)]
            qp = prim_to_cons(*fprim(*xp), gamma)
            qm = prim_to_cons(*fprim(*xm), gamma)
            out.append((qp - qm) / h[a])
    return np.array(out)


# ---------------------------------------------------------------------------
# Config 1: 2-D isentropic vortex (BASELINE.json configs[0])
# ---------------------------------------------------------------------------
def _vortex_prim(t, gamma=1.4, eps=5.0, L=10.0):
    def f(x, y, z):
        xb = np.mod(x - 5.0 - t + L / 2, L) - L / 2
        yb = np.mod(y - 5.0 - t + L / 2, L) - L / 2
        r2 = xb * xb + yb * yb
        e = np.exp(0.5 * (1.0 - r2))
        du = -eps / (2 * PI) * e * yb
        dv = eps / (2 * PI) * e * xb
        T = 1.0 - (gamma - 1.0) * eps * eps / (8.0 * gamma * PI * PI) * np.exp(1.0 - r2)
        rho = T ** (1.0 / (gamma - 1.0))
        p = rho * T
        return rho, 1.0 + du, 1.0 + dv, np.zeros_like(x + y + z), p
    return f


def vortex(n: int = 40, nq: int = 5) -> Case:
    nn = (n, n, 1)
    lo, hi = (0.0, 0.0, 0.0), (10.0, 10.0, 1.0)
    Q, G = gl_average(_vortex_prim(0.0), nn, lo, hi, 1.4, nq=nq)
    return Case("vortex", nn, lo, hi, Q, G, gamma=1.4, mu=0.0, Pr=1.0, cfl=0.5, nonlinear=0,
                tau_eps=0.0, tau_C=0.0, relax_C=10.0, steps=20,
                note="accuracy mode tau=0 (R18); exact solution = IC translated by (t,t)")


def vortex_exact(n: int, t: float, nq: int = 5):
    nn = (n, n, 1)
    return gl_average(_vortex_prim(t), nn, (0.0, 0.0, 0.0), (10.0, 10.0, 1.0), 1.4, nq=nq)


# ---------------------------------------------------------------------------
# Config 2 / 5: Taylor-Green vortex (BASELINE.json configs[1], configs[4]; rho == 1)
# exact separable cell averages
# ---------------------------------------------------------------------------
def _avg1d(kind, a, b):
    h = b - a
    if kind == "sin":
        return (np.cos(a) - np.cos(b)) / h
    if kind == "cos":
        return (np.sin(b) - np.sin(a)) / h
    if kind == "sin2":
        return 0.5 - (np.sin(2 * b) - np.sin(2 * a)) / (4 * h)
    if kind == "cos2":
        return 0.5 + (np.sin(2 * b) - np.sin(2 * a)) / (4 * h)
    if kind == "k2":  # cos(2x)
        return (np.sin(2 * b) - np.sin(2 * a)) / (2 * h)
    if kind == "one":
        return np.ones_like(a)
    raise ValueError(kind)


def _pt1d(kind, x):
    return {"sin": np.sin(x), "cos": np.cos(x), "sin2": np.sin(x) ** 2, "cos2": np.cos(x) ** 2,
            "k2": np.cos(2 * x), "one": np.ones_like(x)}[kind]


def tgv(n: int = 64, Ma: float = 0.1, Re: float = 1600.0, Pr: float = 0.72, gamma: float = 1.4,
        zrep: int = 1, z0: int = 0, nzb: int = None) -> Case:
    """TGV on [-pi,pi]^2 x [-pi, -pi + 2 pi zrep] with n x n x (n zrep) cells (zrep periods along z,
    for weak scaling); optionally only the z-planes [z0, z0+nzb) of it (one rank's slab)."""
    nzg = n * zrep
    if nzb is None:
        nzb = nzg
    nn = (n, n, nzg)
    lo, hi = (-PI, -PI, -PI), (PI, PI, -PI + 2 * PI * zrep)
    h = 2 * PI / n
    edges = -PI + h * np.arange(n + 1)
    a, b = edges[:-1], edges[1:]
    zed = -PI + h * np.arange(z0, z0 + nzb + 1)
    az, bz = zed[:-1], zed[1:]
    p0 = 1.0 / (gamma * Ma * Ma)  # Ma = U0/sqrt(gamma p0/rho0), U0 = rho0 = 1
    # separable terms: list of (coef, kx, ky, kz)
    terms = {
        1: [(1.0, "sin", "cos", "cos")],
        2: [(-1.0, "cos", "sin", "cos")],
        3: [],
        4: [(p0 / (gamma - 1.0), "one", "one", "one"),
            (1.0 / 16.0 / (gamma - 1.0), "k2", "one", "k2"), (2.0 / 16.0 / (gamma - 1.0), "k2", "one", "one"),
            (1.0 / 16.0 / (gamma - 1.0), "one", "k2", "k2"), (2.0 / 16.0 / (gamma - 1.0), "one", "k2", "one"),
            (0.5, "sin2", "cos2", "cos2"), (0.5, "cos2", "sin2", "cos2")],
        0: [(1.0, "one", "one", "one")],
    }
    Q = np.zeros((5, nzb, n, n))
    G = np.zeros((3, 5, nzb, n, n))
    for v, tl in terms.items():
        for (c, kx, ky, kz) in tl:
            Ax, Ay, Az = _avg1d(kx, a, b), _avg1d(ky, a, b), _avg1d(kz, az, bz)
            Dx = (_pt1d(kx, b) - _pt1d(kx, a)) / h
            Dy = (_pt1d(ky, b) - _pt1d(ky, a)) / h
            Dz = (_pt1d(kz, bz) - _pt1d(kz, az)) / h
            Q[v] += c * Az[:, None, None] * Ay[None, :, None] * Ax[None, None, :]
            G[0, v] += c * Az[:, None, None] * Ay[None, :, None] * Dx[None, None, :]
            G[1, v] += c * Az[:, None, None] * Dy[None, :, None] * Ax[None, None, :]
            G[2, v] += c * Dz[:, None, None] * Ay[None, :, None] * Ax[None, None, :]
    mu = 1.0 / Re  # rho0 U0 L / Re
    return Case("tgv", nn, lo, hi, Q, G, gamma=gamma, mu=mu, Pr=Pr, cfl=0.3, nonlinear=0, steps=100,
                note=f"TGV Ma={Ma} Re={Re} rho=1 (BASELINE configs[1]); exact separable averages")


# 1-D trigonometric polynomials {("c"|"s", k): coef} (cos kx / sin kx), for exact separable cell averages
def _tp_mul(p, q):
    out = {}
    for (ta, ka), ca in p.items():
        for (tb, kb), cb in q.items():
            c = 0.5 * ca * cb
            if ta == "c" and tb == "c":
                terms = [("c", ka - kb, c), ("c", ka + kb, c)]
            elif ta == "s" and tb == "s":
                terms = [("c", ka - kb, c), ("c", ka + kb, -c)]
            elif ta == "s":  # sin a cos b
                terms = [("s", ka + kb, c), ("s", ka - kb, c)]
            else:  # cos a sin b
                terms = [("s", ka + kb, c), ("s", kb - ka, c)]
            for t, k, cc in terms:
                if k < 0:  # cos(-k x) = cos(k x), sin(-k x) = -sin(k x)
                    k, cc = -k, (cc if t == "c" else -cc)
                if t == "s" and k == 0:
                    continue
                out[(t, k)] = out.get((t, k), 0.0) + cc
    return out


def _tp_avg(p, a, b):
    h = b - a
    r = np.zeros_like(a)
    for (t, k), c in p.items():
        if k == 0:
            r = r + c
        elif t == "c":
            r = r + c * (np.sin(k * b) - np.sin(k * a)) / (k * h)
        else:
            r = r + c * (np.cos(k * a) - np.cos(k * b)) / (k * h)
    return r


def _tp_pt(p, x):
    r = np.zeros_like(x)
    for (t, k), c in p.items():
        r = r + c * (np.cos(k * x) if t == "c" else np.sin(k * x))
    return r


def tgv_supersonic(n: int = 116, Ma: float = 2.0, Re: float = 1600.0, Pr: float = 0.7, gamma: float = 1.4) -> Case:
    """High-speed Taylor-Green vortex: periodic [-pi, pi]^3 (L = 1),
    U = U0 sin x cos y cos z, V = -U0 cos x sin y cos z, W = 0, rho = p = 1 + (cos 2x + cos 2y)(cos 2z + 2)/16,
    U0 = sqrt(gamma) Ma, Re = 1600, Pr = 0.7, Sutherland viscosity mu(T) = mu0 1.4042 T^1.5 / (T + 0.4042),
    mu0 = rho0 U0 L / Re.  Every conservative field is a sum of separable trigonometric products, so the
    cell averages and averaged gradients (Gauss theorem) are exact.  Nonlinear schemes (GENO /
    Venkatakrishnan) as in the paper."""
    nn = (n, n, n)
    lo, hi = (-PI, -PI, -PI), (PI, PI, PI)
    U0 = math.sqrt(gamma) * Ma
    one, c1, s1, c2 = {("c", 0): 1.0}, {("c", 1): 1.0}, {("s", 1): 1.0}, {("c", 2): 1.0}
    # s = rho / rho0 = p / p0 = 1 + (c2x c2z + 2 c2x + c2y c2z + 2 c2y) / 16, as (coef, fx, fy, fz)
    sfac = [(1.0, one, one, one), (1 / 16, c2, one, c2), (2 / 16, c2, one, one), (1 / 16, one, c2, c2),
            (2 / 16, one, c2, one)]

    def times(terms, c, fx, fy, fz):
        return [(c * t[0], _tp_mul(t[1], fx), _tp_mul(t[2], fy), _tp_mul(t[3], fz)) for t in terms]

    fields = {
        0: sfac,
        1: times(sfac, U0, s1, c1, c1),
        2: times(sfac, -U0, c1, s1, c1),
        3: [],
        4: [(t[0] / (gamma - 1.0),) + t[1:] for t in sfac]
        + times(sfac, 0.5 * U0 * U0, _tp_mul(s1, s1), _tp_mul(c1, c1), _tp_mul(c1, c1))
        + times(sfac, 0.5 * U0 * U0, _tp_mul(c1, c1), _tp_mul(s1, s1), _tp_mul(c1, c1)),
    }
    h = 2 * PI / n
    e = -PI + h * np.arange(n + 1)
    a, b = e[:-1], e[1:]
    Q = np.zeros((5, n, n, n))
    G = np.zeros((3, 5, n, n, n))
    for v, tl in fields.items():
        for (c, fx, fy, fz) in tl:
            Ax, Ay, Az = _tp_avg(fx, a, b), _tp_avg(fy, a, b), _tp_avg(fz, a, b)
            Dx, Dy, Dz = [(_tp_pt(f, b) - _tp_pt(f, a)) / h for f in (fx, fy, fz)]
            Q[v] += c * Az[:, None, None] * Ay[None, :, None] * Ax[None, None, :]
            G[0, v] += c * Az[:, None, None] * Ay[None, :, None] * Dx[None, None, :]
            G[1, v] += c * Az[:, None, None] * Dy[None, :, None] * Ax[None, None, :]
            G[2, v] += c * Dz[:, None, None] * Ay[None, :, None] * Ax[None, None, :]
    c = Case("tgv_ss", nn, lo, hi, Q, G, gamma=gamma, mu=U0 / Re, Pr=Pr, cfl=0.3, nonlinear=1, steps=100,
             note=f"high-speed TGV Ma={Ma} Re={Re} Sutherland (P:455-474); exact separable averages")
    c.sutherland_S = 0.4042
    return c


# ---------------------------------------------------------------------------
# Config 3: decaying compressible isotropic turbulence (BASELINE.json configs[2])
# ---------------------------------------------------------------------------
def hit(n: int = 128, seed: int = 2508, k0: float = 8.0, Mat: float = 0.5, Re_lambda: float = 72.0,
        Pr: float = 0.7, gamma: float = 1.4) -> Case:
    import scipy.fft as sfft
    rng = np.random.default_rng(seed)
    L = 2 * PI
    h = L / n
    k1 = sfft.fftfreq(n, d=1.0 / n)
    KZ, KY, KX = np.meshgrid(k1, k1, k1, indexing="ij")
    K2 = KX ** 2 + KY ** 2 + KZ ** 2
    Kmag = np.sqrt(K2)
    Kmag[0, 0, 0] = 1.0
    # white noise -> spectrum shape sqrt(E(k)/(4 pi k^2)), random phases from the seed
    uh = []
    for c in range(3):
        wn = rng.standard_normal((n, n, n))
        uh.append(sfft.fftn(wn, workers=-1))
    Ek = Kmag ** 4 * np.exp(-2.0 * Kmag ** 2 / k0 ** 2)
    amp = np.sqrt(Ek / (4 * PI * Kmag ** 2))
    amp[0, 0, 0] = 0.0
    uh = [u * amp for u in uh]
    # solenoidal projection k . u_hat = 0
    kd = (KX * uh[0] + KY * uh[1] + KZ * uh[2]) / np.where(K2 == 0, 1.0, K2)
    uh = [uh[0] - KX * kd, uh[1] - KY * kd, uh[2] - KZ * kd]
    # rescale so that sqrt(<u.u>) = Mat * c, c = 1
    upt = [np.real(sfft.ifftn(u, workers=-1)) for u in uh]
    scale = Mat / math.sqrt(np.mean(upt[0] ** 2 + upt[1] ** 2 + upt[2] ** 2))
    uh = [u * scale for u in uh]
    kk = [KX, KY, KZ]
    sinc = [np.sinc(k * h / (2 * PI)) for k in kk]  # np.sinc(x) = sin(pi x)/(pi x)
    S = sinc[0] * sinc[1] * sinc[2]
    rho0, p0 = 1.0, 1.0 / gamma
    Q = np.zeros((5, n, n, n))
    G = np.zeros((3, 5, n, n, n))
    Q[0] = rho0
    for c in range(3):
        Q[1 + c] = np.real(sfft.ifftn(uh[c] * S, workers=-1)) * rho0
        for a in range(3):
            G[a, 1 + c] = np.real(sfft.ifftn(1j * kk[a] * uh[c] * S, workers=-1)) * rho0
    # rho E = p/(gamma-1) + |u|^2/2: average of |u|^2/2 and of u . du/dx_a by 2-point Gauss-Legendre
    xi, wi = _gl(2)
    ke = np.zeros((n, n, n))
    dke = np.zeros((3, n, n, n))
    for pz, wz in zip(xi, wi):
        for py, wy in zip(xi, wi):
            for px, wx in zip(xi, wi):
                ph = np.exp(1j * (KX * px + KY * py + KZ * pz) * h)
                w = wx * wy * wz
                up = [np.real(sfft.ifftn(u * ph, workers=-1)) for u in uh]
                ke += w * 0.5 * (up[0] ** 2 + up[1] ** 2 + up[2] ** 2)
                for a in range(3):
                    s = 0.0
                    for c in range(3):
                        s = s + up[c] * np.real(sfft.ifftn(1j * kk[a] * uh[c] * ph, workers=-1))
                    dke[a] += w * s
    Q[4] = p0 / (gamma - 1.0) + rho0 * ke
    for a in range(3):
        G[a, 4] = rho0 * dke[a]
    u_rms = Mat / math.sqrt(3.0)
    lam_taylor = 2.0 / k0
    mu = rho0 * u_rms * lam_taylor / Re_lambda
    return Case("hit", (n, n, n), (0.0, 0.0, 0.0), (L, L, L), Q, G, gamma=gamma, mu=mu, Pr=Pr, cfl=0.3,
                nonlinear=1, steps=10, note=f"HIT k0={k0} Ma_t={Mat} Re_lambda={Re_lambda} seed={seed}")


# ---------------------------------------------------------------------------
# Config 4: viscous shock-vortex interaction (BASELINE.json configs[3])
# ---------------------------------------------------------------------------
def rankine_hugoniot(M, gamma=1.4, rho1=1.0, p1=None):
    if p1 is None:
        p1 = 1.0 / gamma
    c1 = math.sqrt(gamma * p1 / rho1)
    u1 = M * c1
    r = (gamma + 1) * M * M / ((gamma - 1) * M * M + 2)
    rho2 = rho1 * r
    u2 = u1 / r
    p2 = p1 * (1 + 2 * gamma / (gamma + 1) * (M * M - 1))
    return (rho1, u1, p1), (rho2, u2, p2)


def shock_vortex(nx: int = 1024, ny: int = 512, Ms: float = 1.2, Mv: float = 0.25, R: float = 0.075,
                 Re: float = 800.0, Pr: float = 0.75, gamma: float = 1.4, nq: int = 4) -> Case:
    (r1, u1, p1), (r2, u2, p2) = rankine_hugoniot(Ms, gamma)
    xs, xc, yc = 0.5, 0.25, 0.5
    T1 = p1 / r1

    def f(x, y, z):
        dx, dy = x - xc, y - yc
        rr = np.sqrt(dx * dx + dy * dy)
        q = (rr / R) ** 2
        ut = Mv * (rr / R) * np.exp(0.5 * (1.0 - q))  # c_inf = 1
        rs = np.where(rr > 0, rr, 1.0)
        T = T1 * (1.0 - 0.5 * (gamma - 1.0) * Mv * Mv * np.exp(1.0 - q))
        rho = r1 * (T / T1) ** (1.0 / (gamma - 1.0))
        p = rho * T
        u = u1 - ut * dy / rs
        v = ut * dx / rs
        down = x > xs
        rho = np.where(down, r2, rho)
        p = np.where(down, p2, p)
        u = np.where(down, u2, u)
        v = np.where(down, 0.0, v)
        return rho, u, v, np.zeros_like(x + y + z), p

    nn = (nx, ny, 1)
    lo, hi = (0.0, 0.0, 0.0), (2.0, 1.0, 1.0 / ny)
    Q, G = gl_average(f, nn, lo, hi, gamma, nq=nq)
    bcs = np.zeros((3, 2, 5))
    bcs[0, 0] = prim_to_cons(np.array(r1), np.array(u1), np.array(0.0), np.array(0.0), np.array(p1), gamma)
    mu = r1 * 1.0 * R / Re  # Re = rho1 c1 R / mu, c1 = 1
    return Case("shock_vortex", nn, lo, hi, Q, G, gamma=gamma, mu=mu, Pr=Pr,
                bc=((1, 2), (0, 0), (0, 0)), bc_state=bcs, cfl=0.3, nonlinear=1, steps=10,
                note="Ms=1.2 stationary shock at x=0.5, vortex Mv=0.25 R=0.075 at (0.25,0.5); inflow/outflow in x")


# ---------------------------------------------------------------------------
# Verification problems
# ---------------------------------------------------------------------------
def double_sod(n: int = 100, gamma: float = 1.4) -> Case:
    """Periodic double Sod tube on [0,2): (1,0,1) on [0.5,1.5), (0.125,0,0.1) elsewhere."""
    nn = (n, 1, 1)
    lo, hi = (0.0, 0.0, 0.0), (2.0, 1.0, 1.0)
    x = (np.arange(n) + 0.5) * 2.0 / n
    inside = (x >= 0.5) & (x < 1.5)
    rho = np.where(inside, 1.0, 0.125)
    p = np.where(inside, 1.0, 0.1)
    z = np.zeros(n)
    Q = prim_to_cons(rho, z, z, z, p, gamma).reshape(5, 1, 1, n)
    G = np.zeros((3, 5, 1, 1, n))
    return Case("double_sod", nn, lo, hi, Q, G, gamma=gamma, mu=0.0, Pr=1.0, cfl=0.5, nonlinear=1,
                steps=0, note="t=0.2 compared with the exact Riemann solution of the Sod problem")


def uniform(n=(8, 8, 8), state=(1.0, 0.3, -0.2, 0.1, 1.0), gamma: float = 1.4, L: float = 1.0) -> Case:
    rho, u, v, w, p = state
    nn = tuple(n)
    Q = np.zeros((5,) + nn[::-1])
    q = prim_to_cons(np.array(rho), np.array(u), np.array(v), np.array(w), np.array(p), gamma)
    if nn[2] == 1:
        q[3] = 0.0
        if nn[1] == 1:
            q[2] = 0.0
        q[4] = p / (gamma - 1.0) + 0.5 * rho * (u * u + (v * v if nn[1] > 1 else 0.0) + (w * w if nn[2] > 1 else 0.0))
    for c in range(5):
        Q[c] = q[c]
    G = np.zeros((3,) + Q.shape)
    return Case("uniform", nn, (0.0, 0.0, 0.0), (L, L, L), Q, G, gamma=gamma)


def random_smooth(n=(12, 10, 8), seed: int = 7, amp: float = 0.2, gamma: float = 1.4, mu: float = 0.0,
                  Pr: float = 1.0, kmax: int = 2, nq: int = 4, jump: float = 0.0) -> Case:
    """Seeded smooth periodic field on [0,1]^dim: a few random Fourier modes per variable.
    ``jump`` > 0 adds a smoothed density/pressure step (for the nonlinear paths)."""
    nn = tuple(int(a) for a in n)
    dim = 3 if nn[2] > 1 else (2 if nn[1] > 1 else 1)
    rng = np.random.default_rng(seed)
    modes = []
    for var in range(5):
        ml = []
        for _ in range(4):
            k = rng.integers(-kmax, kmax + 1, size=3)
            k[dim:] = 0
            ml.append((k, rng.uniform(0, 2 * PI), rng.uniform(-1, 1) / 4.0))
        modes.append(ml)

    def field_(var, x, y, z):
        s = 0.0
        for (k, ph, a) in modes[var]:
            s = s + a * np.cos(2 * PI * (k[0] * x + k[1] * y + k[2] * z) + ph)
        return s

    def f(x, y, z):
        rho = 1.0 + amp * field_(0, x, y, z)
        u = 0.5 * field_(1, x, y, z)
        v = 0.5 * field_(2, x, y, z) if dim > 1 else 0.0 * x
        w = 0.5 * field_(3, x, y, z) if dim > 2 else 0.0 * x
        p = 1.0 + amp * field_(4, x, y, z)
        if jump > 0.0:
            s = 0.5 * (1.0 + np.tanh((np.abs(x - 0.5) - 0.25) / 0.01))
            rho = rho + jump * s
            p = p + jump * s
        return rho, u, v, w, p

    lo = (0.0, 0.0, 0.0)
    hi = tuple(1.0 if a < dim else 1.0 / max(nn[0], 1) for a in range(3))
    Q, G = gl_average(f, nn, lo, hi, gamma, nq=nq)
    return Case("random_smooth", nn, lo, hi, Q, G, gamma=gamma, mu=mu, Pr=Pr, cfl=0.4)


CASES = {"vortex": vortex, "tgv": tgv, "tgv_supersonic": tgv_supersonic, "hit": hit, "shock_vortex": shock_vortex, "double_sod": double_sod,
         "uniform": uniform, "random_smooth": random_smooth}


def make_case(name: str, **kw) -> Case:
    return CASES[name](**kw)
