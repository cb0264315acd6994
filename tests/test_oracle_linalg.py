"""Pins for the oracle's dense pieces: Pade-13 coefficients, expm, Eq. (8), Dot2.

Everything is compared with something other than the oracle: exact integer/rational arithmetic,
closed forms, algebraic identities, and scipy.linalg.expm (an independent implementation; the
oracle's expm is hand-written C and does not call it).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_pade13_coefficients_exact(orc):
    # degree-13 diagonal Pade; b_j = c_j/c_13 are the integers in golden/pade13.json
    b = [int(x) for x in json.load(open(os.path.join(GOLD, "pade13.json")))["b"]]
    c = orc.pade13_coeffs()
    assert c[0] == 1.0
    for j in range(14):
        exact = Fraction(b[j], b[0])                  # c_j = b_j / b_0 since c_0 = 1
        assert abs(c[j] - float(exact)) <= 2 * (j + 1) * 2.3e-16 * float(exact), j  # j roundings


def test_pade13_scalar_is_exp(orc):
    c = orc.pade13_coeffs()
    for z in (0.0, 0.1, -0.5, 1.0):
        p = sum(c[j] * z ** j for j in range(14))
        q = sum(c[j] * (-z) ** j for j in range(14))
        assert abs(p / q - math.exp(z)) <= 8e-16 * math.exp(z)   # a few roundings in p, q, p/q


def test_cost_M_examples(orc):
    # SPEC S:174-176 on Eq. (8)
    g = json.load(open(os.path.join(GOLD, "controller_examples.json")))["cost_M"]
    want = {"44/3": 44 / 3, "44/3+4": 44 / 3 + 4}
    for e in g:
        assert orc.cost_M(e["norm1"]) == pytest.approx(want[e["M"]], rel=1e-15)
    assert orc.expm_squarings(0.0) == 0
    assert orc.expm_squarings(5.37 * 2 ** 5) == 5
    assert orc.expm_squarings(5.37 * 2 ** 5 * 1.0001) == 6


@pytest.mark.parametrize("K", [1, 2, 7])
def test_expm_zero_is_identity(orc, K):
    assert np.array_equal(orc.expm(np.zeros((K, K))), np.eye(K))


def test_expm_closed_forms(orc):
    # nilpotent: series terminates
    assert np.allclose(orc.expm(np.array([[0.0, 1.0], [0.0, 0.0]])), [[1, 1], [0, 1]], atol=1e-15, rtol=0)
    # diagonal
    E = orc.expm(np.diag([1.0, 2.0]))
    assert abs(E[0, 0] - math.e) < 1e-14 and abs(E[1, 1] - math.e ** 2) < 1e-14
    assert E[0, 1] == 0 and E[1, 0] == 0
    # rotation generator: exp([[0,-a],[a,0]]) = [[cos,-sin],[sin,cos]]
    a = 7.3
    E = orc.expm(np.array([[0.0, -a], [a, 0.0]]))
    assert np.allclose(E, [[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]], atol=1e-13, rtol=0)
    # Jordan block: exp(l I + N) = e^l (I + N + N^2/2)
    l = -3.0
    J = np.array([[l, 1, 0], [0, l, 1], [0, 0, l]], dtype=float)
    want = math.exp(l) * np.array([[1, 1, 0.5], [0, 1, 1], [0, 0, 1]])
    assert np.allclose(orc.expm(J), want, atol=1e-15, rtol=1e-13)


def test_expm_identities(orc):
    rng = np.random.default_rng(7)
    for K in (3, 17, 40):
        A = rng.standard_normal((K, K))
        A *= 10.0 / np.abs(A).sum(axis=0).max()       # ||A||_1 = 10
        assert np.abs(orc.expm(A) @ orc.expm(-A) - np.eye(K)).max() < 1e-10
        S = A + A.T
        ES = orc.expm(S)
        assert np.abs(ES - ES.T).max() <= 1e-12 * np.abs(ES).max()
    B1, B2 = rng.standard_normal((4, 4)), rng.standard_normal((3, 3))
    Bd = scipy.linalg.block_diag(B1, B2)
    Ed = orc.expm(Bd)
    assert np.allclose(Ed[:4, :4], orc.expm(B1), atol=1e-12) and np.allclose(Ed[4:, 4:], orc.expm(B2), atol=1e-12)
    assert np.abs(Ed[:4, 4:]).max() == 0 and np.abs(Ed[4:, :4]).max() == 0


@pytest.mark.parametrize("K,norm", [(1, 0.3), (5, 1.0), (16, 40.0), (43, 300.0), (105, 80.0)])
def test_expm_vs_scipy(orc, K, norm):
    rng = np.random.default_rng(K)
    A = rng.standard_normal((K, K))
    A *= norm / np.abs(A).sum(axis=0).max()
    A -= 0.5 * norm * np.eye(K)                       # keep exp(A) of moderate size
    E, R = orc.expm(A), scipy.linalg.expm(A)
    assert np.linalg.norm(E - R) <= 1e-12 * np.linalg.norm(R) * max(1.0, norm / 5)


def test_expm_hessenberg_like_augmented(orc):
    # the matrices K4 sees: Hessenberg block + e1 column + shifted identity (Eq. hathm)
    rng = np.random.default_rng(3)
    m, p = 30, 3
    H = np.triu(rng.standard_normal((m, m)), -1) * 20.0
    K = m + p + 1
    Hh = np.zeros((K, K))
    Hh[:m, :m] = H
    Hh[0, m] = 1.0
    for i in range(1, p + 1):
        Hh[m + i - 1, m + i] = 1.0
    E, R = orc.expm(Hh), scipy.linalg.expm(Hh)
    assert np.linalg.norm(E - R) <= 1e-11 * np.linalg.norm(R)


def test_dot2_exact(orc):
    rng = np.random.default_rng(11)
    for n in (1, 10, 1000):
        x, y = rng.standard_normal(n), rng.standard_normal(n)
        exact = sum(Fraction(a) * Fraction(b) for a, b in zip(x.tolist(), y.tolist()))
        assert abs(orc.dot(x, y) - float(exact)) <= 2.3e-16 * abs(float(exact)) + 1e-300
    # ill-conditioned: huge cancellation, exact answer 1
    x = np.array([1e16, 1.0, -1e16])
    y = np.array([1.0, 1.0, 1.0])
    assert orc.dot(x, y) == 1.0
    assert orc.norm2(np.array([3.0, 4.0])) == 5.0
