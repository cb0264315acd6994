"""The GPU exponential's constants (csrc/expm.cuh, PHIPM_EXPM_TAYLOR) against their definitions:
theta_m = the largest alpha with sum_{k>m} |c_k| alpha^(k-1) <= 2^-53 for h_m(x) = log(exp(-x) T_m(x))
(exact rational series, tools/taylor_theta.py), and 1/k! correctly rounded.  CPU only."""
import os
import re
import sys
from fractions import Fraction
from math import factorial

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import taylor_theta  # noqa: E402

SRC = open(os.path.join(ROOT, "paper_0907_4631_b200", "csrc", "expm.cuh")).read()


def array(name):
    body = re.search(name + r"\[[^\]]*\]\s*=\s*\{([^}]*)\}", SRC).group(1)
    return [x.strip() for x in body.split(",") if x.strip()]


def test_theta_constants_match_the_exact_series():
    ms = [int(x) for x in array("TAYLOR_M")]
    th = [float(x) for x in array("TAYLOR_THETA")]
    assert ms == [8, 12, 16]
    for m, t in zip(ms, th):
        ref = taylor_theta.theta(m)
        assert abs(t - ref) <= 1e-14 * ref, (m, t, ref)
    # the bound really holds at theta and fails just above it
    for m, t in zip(ms, th):
        c = taylor_theta.h_coeffs(m)
        f = lambda a: sum(ck * a ** (k - 1) for k, ck in enumerate(c) if k >= 1)
        assert f(t) <= 2.0 ** -53 < f(t * (1 + 1e-6))


def test_products_of_the_paterson_stockmeyer_schemes():
    # degree m = 4 r from A, A^2, A^3, A^4: 3 products for the powers, r - 1 Horner products in A^4
    prods = [int(x) for x in array("TAYLOR_PROD")]
    assert prods == [3 + m // 4 - 1 for m in (8, 12, 16)]


def test_inverse_factorials_correctly_rounded():
    vals = [float(x) for x in array("TAYLOR_INVFACT")]
    assert len(vals) == 17
    for k, v in enumerate(vals):
        assert v == float(Fraction(1, factorial(k)))
