"""Parity metric (R34 of DESIGN.md): relative L-infinity per conservative variable and
per gradient component.

  Q_v      : |Q_v^gpu - Q_v^orc| / max |Q_v|   (the three momentum components share one floor);
  G_{a,v}  : |G^gpu - G^orc| / max( max_a |G_{a,v}|  (same momentum family rule),
                                    A_v / tol )
             with the rounding allowance A_v = 16 n eps max|Q_v| / h_min: a gradient is a
             difference of interface values of size |Q_v| over a cell width, so each of the n
             steps leaves rounding of order eps |Q_v| / h_min in it (the oracle's literal
             two-window formula P:116 puts eps |Q| / dt into Q_t, times dt in the update).  An
             absolute gradient error below A_v therefore counts as tol; above it the plain
             relative bound applies.  (Round 1 used max|Q_v| / L as the second term, which on the
             TGV was ~20x looser than max|G| for the energy gradient: VERDICT r01, weak item 2.)
"""
import numpy as np

EPS = np.finfo(np.float64).eps


def floors(Q, G=None, h=1.0, nsteps=10, tol=1e-10):
    qf = np.abs(Q).reshape(5, -1).max(axis=1)
    qf[1:4] = qf[1:4].max()
    qf = np.maximum(qf, 1e-300)
    if G is None:
        return qf, None
    gf = np.abs(G).reshape(3, 5, -1).max(axis=(0, 2))
    gf[1:4] = gf[1:4].max()
    allow = 16.0 * max(int(nsteps), 1) * EPS * qf / h
    gf = np.maximum(np.maximum(gf, allow / tol), 1e-300)
    return qf, gf


def rel_linf(Qg, Qo, Gg=None, Go=None, h=1.0, nsteps=10, tol=1e-10):
    out = {}
    qf, gf = floors(Qo, Go if (Gg is not None and Go is not None) else None, h, nsteps, tol)
    for v in range(5):
        out[f"Q{v}"] = float(np.abs(Qg[v] - Qo[v]).max() / qf[v])
    if gf is not None:
        for v in range(5):
            for a in range(3):
                out[f"G{a}{v}"] = float(np.abs(Gg[a, v] - Go[a, v]).max() / gf[v])
    return out


def hmin(case_or_n, lo=None, hi=None):
    """smallest uniform cell width over the active axes (a Case, or n, lo, hi)"""
    if lo is None:
        c = case_or_n
        n, lo, hi = c.n, c.lo, c.hi
    else:
        n = case_or_n
    return min((hi[a] - lo[a]) / n[a] for a in range(3) if n[a] > 1) if any(x > 1 for x in n) else hi[0] - lo[0]


def worst(d):
    k = max(d, key=d.get)
    return k, d[k]
