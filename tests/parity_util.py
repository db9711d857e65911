"""Parity metric (R34 of DESIGN.md): relative L-infinity per conservative variable and
per gradient component.  Floors keep near-zero fields from turning rounding noise
into large relative numbers:
  Q_v      : max |Q_v| (the three momentum components share one floor);
  G_{a,v}  : max( max_a |G_{a,v}|, max |Q_v| / L ) with the same momentum family rule,
             L = the largest active domain length (a gradient is a difference of values
             of size |Q_v|; e.g. the density gradient of the rho == 1 Taylor-Green
             vortex is ~0 while rho ~ 1)."""
import numpy as np


def floors(Q, G=None, L=1.0):
    qf = np.abs(Q).reshape(5, -1).max(axis=1)
    qf[1:4] = qf[1:4].max()
    qf = np.maximum(qf, 1e-300)
    if G is None:
        return qf, None
    gf = np.abs(G).reshape(3, 5, -1).max(axis=(0, 2))
    gf[1:4] = gf[1:4].max()
    gf = np.maximum(np.maximum(gf, qf / L), 1e-300)
    return qf, gf


def rel_linf(Qg, Qo, Gg=None, Go=None, L=1.0):
    out = {}
    qf, gf = floors(Qo, Go if (Gg is not None and Go is not None) else None, L)
    for v in range(5):
        out[f"Q{v}"] = float(np.abs(Qg[v] - Qo[v]).max() / qf[v])
    if gf is not None:
        for v in range(5):
            for a in range(3):
                out[f"G{a}{v}"] = float(np.abs(Gg[a, v] - Go[a, v]).max() / gf[v])
    return out


def worst(d):
    k = max(d, key=d.get)
    return k, d[k]
