"""Backward-error thresholds theta_m of the degree-m Taylor approximant of exp (used by the GPU expm).

For ||A|| small enough, T_m(A) = exp(A + dA) with dA = h_m(A),
    h_m(x) = log(exp(-x) T_m(x)) = sum_{k > m} c_k x^k,
and ||dA|| / ||A|| <= sum_k |c_k| a^(k-1) with a an upper bound of the growth of ||A^k||^(1/k)
(a = ||A|| or the sharper max(||A^3||^(1/3), ||A^4||^(1/4)), valid for m >= 5).  theta_m is the
largest a with that bound <= u = 2^-53.  The c_k are computed exactly (rational series arithmetic);
only the final bisection uses floats.  Run: python tools/taylor_theta.py
"""
from fractions import Fraction
from math import factorial

N = 160          # series truncation degree (terms beyond it are < 1e-40 at a <= 2)


def series_mul(a, b):
    out = [Fraction(0)] * (N + 1)
    for i, ai in enumerate(a):
        if ai == 0:
            continue
        for j in range(0, N + 1 - i):
            if b[j]:
                out[i + j] += ai * b[j]
    return out


def h_coeffs(m):
    # R(x) = 1 - exp(-x) T_m(x) = exp(-x) (exp(x) - T_m(x)); log(1 - R) = -sum_j R^j / j
    em = [Fraction((-1) ** k, factorial(k)) for k in range(N + 1)]
    tail = [Fraction(0)] * (N + 1)
    for k in range(m + 1, N + 1):
        tail[k] = Fraction(1, factorial(k))
    R = series_mul(em, tail)
    h = [Fraction(0)] * (N + 1)
    P = [Fraction(1)] + [Fraction(0)] * N
    j = 1
    while True:
        P = series_mul(P, R)
        if not any(P):
            break
        for k in range(N + 1):
            h[k] -= P[k] / j
        j += 1
    return [abs(float(c)) for c in h]


def theta(m, u=2.0 ** -53):
    c = h_coeffs(m)
    f = lambda a: sum(ck * a ** (k - 1) for k, ck in enumerate(c) if k >= 1)
    lo, hi = 0.0, 4.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(mid) <= u:
            lo = mid
        else:
            hi = mid
    return lo


if __name__ == "__main__":
    for m in (4, 8, 12, 16, 20):
        print(f"theta_{m} = {theta(m):.17g}")
