"""Exact solution of the 1-D Riemann problem for an ideal gas (textbook: pressure
function + Newton iteration for p*, then wave sampling).  Used only as an
independent pin of the oracle on the Sod problem."""
import math

import numpy as np


def _fk(p, rk, pk, g):
    ck = math.sqrt(g * pk / rk)
    if p > pk:  # shock
        A = 2.0 / ((g + 1.0) * rk)
        B = (g - 1.0) / (g + 1.0) * pk
        f = (p - pk) * math.sqrt(A / (p + B))
        df = math.sqrt(A / (B + p)) * (1.0 - 0.5 * (p - pk) / (B + p))
    else:  # rarefaction
        f = 2.0 * ck / (g - 1.0) * ((p / pk) ** ((g - 1.0) / (2.0 * g)) - 1.0)
        df = 1.0 / (rk * ck) * (p / pk) ** (-(g + 1.0) / (2.0 * g))
    return f, df


def star_state(L, R, g):
    rl, ul, pl = L
    rr, ur, pr = R
    p = 0.5 * (pl + pr)
    for _ in range(100):
        fl, dfl = _fk(p, rl, pl, g)
        fr, dfr = _fk(p, rr, pr, g)
        dp = (fl + fr + ur - ul) / (dfl + dfr)
        p = max(p - dp, 1e-12)
        if abs(dp) < 1e-15 * p:
            break
    fl, _ = _fk(p, rl, pl, g)
    fr, _ = _fk(p, rr, pr, g)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def sample(L, R, g, s):
    """Primitive (rho, u, p) at similarity coordinate s = x/t (vectorised over s)."""
    rl, ul, pl = L
    rr, ur, pr = R
    ps, us = star_state(L, R, g)
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    out = np.zeros((3, len(s)))
    for i, si in enumerate(s):
        if si <= us:  # left of contact
            if ps > pl:  # left shock
                sl = ul - cl * math.sqrt((g + 1) / (2 * g) * ps / pl + (g - 1) / (2 * g))
                if si <= sl:
                    out[:, i] = (rl, ul, pl)
                else:
                    r = rl * (ps / pl + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pl + 1)
                    out[:, i] = (r, us, ps)
            else:  # left rarefaction
                shl = ul - cl
                csl = cl * (ps / pl) ** ((g - 1) / (2 * g))
                stl = us - csl
                if si <= shl:
                    out[:, i] = (rl, ul, pl)
                elif si >= stl:
                    out[:, i] = (rl * (ps / pl) ** (1 / g), us, ps)
                else:
                    u = 2 / (g + 1) * (cl + (g - 1) / 2 * ul + si)
                    c = 2 / (g + 1) * (cl + (g - 1) / 2 * (ul - si))
                    r = rl * (c / cl) ** (2 / (g - 1))
                    out[:, i] = (r, u, pl * (c / cl) ** (2 * g / (g - 1)))
        else:  # right of contact
            if ps > pr:  # right shock
                sr = ur + cr * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
                if si >= sr:
                    out[:, i] = (rr, ur, pr)
                else:
                    r = rr * (ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1)
                    out[:, i] = (r, us, ps)
            else:  # right rarefaction
                shr = ur + cr
                csr = cr * (ps / pr) ** ((g - 1) / (2 * g))
                stр = us + csr
                if si >= shr:
                    out[:, i] = (rr, ur, pr)
                elif si <= stр:
                    out[:, i] = (rr * (ps / pr) ** (1 / g), us, ps)
                else:
                    u = 2 / (g + 1) * (-cr + (g - 1) / 2 * ur + si)
                    c = 2 / (g + 1) * (cr - (g - 1) / 2 * (ur - si))
                    r = rr * (c / cr) ** (2 / (g - 1))
                    out[:, i] = (r, u, pr * (c / cr) ** (2 * g / (g - 1)))
    return out


def double_sod_density(x, t, g=1.4, nsub=20):
    """Cell-averaged exact density of the periodic double Sod problem on [0,2) at time t
    (valid while the two Riemann fans do not interact): high state on [0.5, 1.5)."""
    hi, lo = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    h = x[1] - x[0]
    off = (np.arange(nsub) + 0.5) / nsub - 0.5
    rho = np.zeros(len(x))
    for j, xc in enumerate(x):
        pts = xc + off * h
        vals = []
        for xp in pts:
            if xp < 1.0:  # Riemann problem at x = 0.5: low | high
                s = (xp - 0.5) / t
                vals.append(sample(lo, hi, g, [s])[0, 0])
            else:  # Riemann problem at x = 1.5: high | low
                s = (xp - 1.5) / t
                vals.append(sample(hi, lo, g, [s])[0, 0])
        rho[j] = np.mean(vals)
    return rho
