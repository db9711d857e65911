#!/usr/bin/env python
"""Chebyshev coefficients of f(t) = (1 + 2a) exp(a^2) erfc(a), a = K (1 + t) / (1 - t), t in [-1, 1]
(the Shepherd-Laframboise form of the scaled complementary error function), computed with mpmath
at 40 digits, and a check of the double-precision evaluation used by the flux kernel
(gks_flux.cuh: erfc_e) against mpmath's erfc.

  python tools/erfc_fit.py            # prints the C table and the measured max relative error
"""
import math

import mpmath as mp

mp.mp.dps = 40
K = mp.mpf(3.75)
NT = 25


def coeffs(n=NT, m=240):
    nodes = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / m) for k in range(m)]
    vals = []
    for t in nodes:
        a = K * (1 + t) / (1 - t)
        vals.append((1 + 2 * a) * mp.exp(a * a) * mp.erfc(a))
    return [2 * mp.fsum(vals[k] * mp.cos(j * mp.pi * (k + mp.mpf(1) / 2) / m) for k in range(m)) / m
            for j in range(n)]


def erfc_e(z, c):
    """double-precision mirror of the device code"""
    a = abs(z)
    e = math.exp(-a * a)
    r = 1.0 / ((a + float(K)) * (1.0 + 2.0 * a))
    t = (a - float(K)) * (1.0 + 2.0 * a) * r
    inv = (a + float(K)) * r
    t2 = 2.0 * t
    b1 = 0.0
    b2 = 0.0
    for cj in reversed(c[1:]):
        b1, b2 = cj + t2 * b1 - b2, b1
    f = 0.5 * c[0] + t * b1 - b2
    y = e * f * inv
    return y if z >= 0 else 2.0 - y


if __name__ == "__main__":
    c = coeffs()
    cd = [float(x) for x in c]
    print(f"// K = {float(K)}, {NT} terms")
    print("{" + ", ".join(repr(x) for x in cd) + "}")
    worst = 0.0
    z = -6.0
    while z < 26.0:
        ref = mp.erfc(mp.mpf(z))
        got = erfc_e(z, cd)
        if ref != 0:
            worst = max(worst, float(abs((got - ref) / ref)))
        z += 0.00731
    print("max relative error on [-6, 26):", worst)
