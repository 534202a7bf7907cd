"""Derive the constants of the builder's 14-point degree-5 tetrahedral rule.

Orbits (barycentric): S31 (a, a, a, 1-3a) ×2 and S22 (c, c, 1/2-c, 1/2-c). Six unknowns
(a1, w1, a2, w2, c, w3), solved by Gauss–Newton in 50-digit arithmetic on the moment equations
Σ w_q λ_q^α = 3! α! / (|α|+3)! for every |α| ≤ 5 (weights sum to 1), started from the
literature's 14-point values rounded to 4 digits. Prints 17 significant digits and the
worst monomial residual. The CUDA builder types the printed constants (egfem_build.cu).
"""
import itertools
from math import factorial

from mpmath import mp, mpf, matrix, lu_solve

mp.dps = 50


def points(x):
    a1, w1, a2, w2, c, w3 = x
    P = []
    for a, w in ((a1, w1), (a2, w2)):
        for q in range(4):
            P.append(([1 - 3 * a if i == q else a for i in range(4)], w))
    for (i, j) in itertools.combinations(range(4), 2):
        lam = [mpf(1) / 2 - c] * 4
        lam[i] = lam[j] = c
        P.append((lam, w3))
    return P


ALPHAS = [al for s in range(6) for al in itertools.product(range(6), repeat=4) if sum(al) == s]


def resid(x):
    P = points(x)
    out = []
    for al in ALPHAS:
        exact = mpf(factorial(3) * factorial(al[0]) * factorial(al[1]) * factorial(al[2]) * factorial(al[3])) / factorial(sum(al) + 3)
        got = mpf(0)
        for lam, w in P:
            t = w
            for l, e in zip(lam, al):
                t *= l ** e
            got += t
        out.append(got - exact)
    return out


x = [mpf("0.0927"), mpf("0.0735"), mpf("0.3109"), mpf("0.1127"), mpf("0.0455"), mpf("0.0425")]
for it in range(60):
    r = resid(x)
    J = []
    h = mpf(10) ** -30
    for k in range(6):
        xp = list(x)
        xp[k] += h
        rp = resid(xp)
        J.append([(a - b) / h for a, b in zip(rp, r)])
    # Gauss–Newton: (JᵀJ) dx = -Jᵀ r
    A = matrix(6, 6)
    g = matrix(6, 1)
    for p in range(6):
        for q in range(6):
            A[p, q] = sum(J[p][m] * J[q][m] for m in range(len(r)))
        g[p] = -sum(J[p][m] * r[m] for m in range(len(r)))
    dx = lu_solve(A, g)
    x = [x[k] + dx[k] for k in range(6)]
worst = max(abs(v) for v in resid(x))
names = ["a1", "w1", "a2", "w2", "c", "w3"]
for n_, v in zip(names, x):
    print(n_, mp.nstr(v, 17))
print("worst |moment residual| (|alpha|<=5):", mp.nstr(worst, 3))
print("sum of weights:", mp.nstr(4 * x[1] + 4 * x[3] + 6 * x[5], 20))
