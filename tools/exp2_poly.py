"""Derives the polynomial used by the device exp in csrc/hk_exp.cuh.

2^(r/T) on r in [-1/2, 1/2] (T = table size) is written as 1 + r*g(r) with g
a degree-d polynomial fitted at Chebyshev nodes in 60-digit arithmetic
(mpmath.chebyfit, near-minimax).  Prints the coefficients and the maximum
relative error of the double-precision Horner evaluation, table multiply
included, measured on a dense grid against mpmath.
"""
import sys
import mpmath as mp
import numpy as np

mp.mp.dps = 60


def fit(T, d):
    f = lambda r: (mp.power(2, r / T) - 1) / r if r != 0 else mp.log(2) / T
    poly, err = mp.chebyfit(f, [-0.5, 0.5], d + 1, error=True)
    return [float(c) for c in poly[::-1]]  # c1 (constant of g) .. c_{d+1}


def check(T, coeffs, n=200001):
    rs = np.linspace(-0.5, 0.5, n)
    table = [float(mp.power(2, mp.mpf(j) / T)) for j in range(T)]
    worst = 0.0
    for j in (0, T // 3, T - 1):
        for r in rs[:: max(1, n // 20001)]:
            p = coeffs[-1]
            for c in reversed(coeffs[:-1]):
                p = np.fma(p, r, c) if hasattr(np, "fma") else p * r + c
            y = p * r + 1.0
            y = y * table[j]
            exact = mp.power(2, (mp.mpf(j) + mp.mpf(r)) / T)
            worst = max(worst, abs(float((mp.mpf(y) - exact) / exact)))
    return worst


if __name__ == "__main__":
    for T, d in ((16, 4), (32, 3), (16, 3), (64, 3)):
        c = fit(T, d)
        print(f"T={T} deg(g)={d}: coeffs={[repr(x) for x in c]}  max_rel_err={check(T, c):.3e}")
