"""Pade approximants [n/n] of R(w) = atanh(sqrt w) / sqrt w = sum_k w^k / (2k+1)
(the moderate-strain log of smpm_common.cuh: eps = 1/2 log B = atanh(Z) =
Z R(Z^2)) and the largest w up to which each keeps |sqrt(w) (P/Q - R)| <= 4e-9."""
from fractions import Fraction

import numpy as np
import sympy as sp

c = [Fraction(1, 2 * k + 1) for k in range(16)]


def pade(m, n):
    q = sp.symbols(f"q1:{n + 1}")
    eqs = [sum((1 if j == 0 else q[j - 1]) * sp.Rational(c[k - j].numerator, c[k - j].denominator)
               for j in range(n + 1) if k - j >= 0) for k in range(m + 1, m + n + 1)]
    sol = sp.solve(eqs, q, dict=True)[0]
    qq = [sp.Integer(1)] + [sol[x] for x in q]
    p = [sum(qq[j] * sp.Rational(c[k - j].numerator, c[k - j].denominator) for j in range(min(k, n) + 1))
         for k in range(m + 1)]
    return p, qq


w = np.linspace(1e-6, 0.36, 40001)
f = np.arctanh(np.sqrt(w)) / np.sqrt(w)
for n in (2, 3, 4):
    p, q = pade(n, n)
    P = sum(float(a) * w ** k for k, a in enumerate(p))
    Q = sum(float(a) * w ** k for k, a in enumerate(q))
    err = np.sqrt(w) * np.abs(P / Q - f)
    bad = np.argmax(err > 4e-9) if (err > 4e-9).any() else len(w)
    print(f"[{n}/{n}] ok up to w = {w[bad - 1]:.4f}, min Q = {Q.min():.3f}; P = {p}; Q = {q}")
