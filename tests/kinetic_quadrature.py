"""Brute-force velocity-space quadrature of Maxwellian moments, independent of the
oracle's closed-form moment recursions (tests only).

The particle velocity (u, v, w) and N = 2 internal degrees of freedom (xi_1, xi_2)
(gamma = 1.4, N = (5-3 gamma)/(gamma-1) = 2) are integrated with tensor
Gauss-Hermite nodes; a half range u>0 or u<0 uses Gauss-Legendre on a truncated
interval.  Every expectation is normalised by rho (<.> = (1/rho) int . g dXi).
"""
import math

import numpy as np


class MaxwellQuad:
    def __init__(self, rho, U, V, W, lam, side=0, n_gh=14, n_xi=8, n_gl=120):
        self.rho = rho
        sig = 1.0 / math.sqrt(2.0 * lam)
        x, w = np.polynomial.hermite_e.hermegauss(n_gh)  # weight exp(-x^2/2)
        w = w / math.sqrt(2 * math.pi)
        xq, wq = np.polynomial.hermite_e.hermegauss(n_xi)
        wq = wq / math.sqrt(2 * math.pi)
        if side == 0:
            un, uw = U + sig * x, w
        else:
            # integrate the 1-D normal density over u>0 (side=+1) or u<0 (side=-1), truncated at 14 sigma
            if side > 0:
                a, b = 0.0, max(U, 0.0) + 14 * sig
            else:
                a, b = min(U, 0.0) - 14 * sig, 0.0
            if b <= a:
                un, uw = np.array([0.0]), np.array([0.0])
            else:
                g, gw = np.polynomial.legendre.leggauss(n_gl)
                un = 0.5 * (b - a) * g + 0.5 * (a + b)
                uw = 0.5 * (b - a) * gw * np.exp(-0.5 * ((un - U) / sig) ** 2) / (sig * math.sqrt(2 * math.pi))
        vn, vw = V + sig * x, w
        wn, ww = W + sig * x, w
        x1, w1 = sig * xq, wq
        grids = np.meshgrid(un, vn, wn, x1, x1, indexing="ij")
        wts = np.meshgrid(uw, vw, ww, w1, w1, indexing="ij")
        self.u, self.v, self.w = grids[0].ravel(), grids[1].ravel(), grids[2].ravel()
        self.xi2 = (grids[3] ** 2 + grids[4] ** 2).ravel()
        self.wt = (wts[0] * wts[1] * wts[2] * wts[3] * wts[4]).ravel()

    def psi(self):
        return np.stack([np.ones_like(self.u), self.u, self.v, self.w,
                         0.5 * (self.u ** 2 + self.v ** 2 + self.w ** 2 + self.xi2)])

    def slope(self, a):
        """Evaluate a = a1 + a2 u + a3 v + a4 w + a5 psi5 at the nodes."""
        P = self.psi()
        return np.tensordot(np.asarray(a), P, axes=(0, 0))

    def vel(self, axis):
        return [self.u, self.v, self.w][axis]

    def mean(self, f):
        """<f psi> as a 5-vector (normalised by rho)."""
        return self.psi() @ (self.wt * f)
