"""Pins for the oracle's phi-function evaluation (augmented exponential, Eq. hathm).

phi_p(tau H) e1 and phi_{p+1}(tau H) e1 from one (mu+p+1)^2 exponential are checked against the
closed forms of Sec. 2, phi_l(0)=1/l!, the recurrence Eq. (phirelation) P:154-159,
a Taylor series of the integral definition, and an eigen-decomposition route.
"""
import json
import math
import os

import numpy as np
import pytest

from exact import phi_scalar

GOLD = os.path.join(os.path.dirname(__file__), "golden")
E = math.e


def closed(ell, z):
    # P:144-153
    return [math.exp(z), (math.exp(z) - 1) / z, (math.exp(z) - 1 - z) / z ** 2,
            (math.exp(z) - 1 - z - z * z / 2) / z ** 3][ell]


def test_golden_phi_z1(orc):
    g = json.load(open(os.path.join(GOLD, "phi_z1.json")))["z1_decimal"]
    vals = [float(g[f"phi{l}"]) for l in range(4)]
    for p in range(3):
        a, b, _ = orc.phi_pair([[1.0]], 1.0, p)
        assert a[0] == pytest.approx(vals[p], rel=2e-15)
        assert b[0] == pytest.approx(vals[p + 1], rel=4e-15)


@pytest.mark.parametrize("z", [1.0, -1.0, 3.0, -3.0, 0.5])
@pytest.mark.parametrize("p", [0, 1, 2])
def test_phi_closed_forms(orc, z, p):
    a, b, nh = orc.phi_pair([[z]], 1.0, p)
    assert a[0] == pytest.approx(closed(p, z), rel=1e-13)
    assert b[0] == pytest.approx(closed(p + 1, z), rel=1e-12)
    assert nh == abs(z)


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4])
def test_phi_at_zero(orc, p):
    # phi_l(0) = 1/l! from the integral
    a, b, _ = orc.phi_pair([[0.0]], 1.0, p)
    assert a[0] == pytest.approx(1 / math.factorial(p), rel=1e-15)
    assert b[0] == pytest.approx(1 / math.factorial(p + 1), rel=1e-15)


def test_phi_tau_scaling(orc):
    # R8: tau enters only through tau*H: phi_pair(H, tau) = phi(tau h)
    a, b, _ = orc.phi_pair([[-2.0]], 0.25, 2)
    assert a[0] == pytest.approx(closed(2, -0.5), rel=1e-13)
    assert b[0] == pytest.approx(closed(3, -0.5), rel=1e-12)


def test_phi_recurrence(orc):
    # Eq. (phirelation): phi_l(z) = z phi_{l+1}(z) + 1/l!, residual <= 1e-13
    rng = np.random.default_rng(5)
    for z in rng.uniform(-2, 2, 50):
        for l in range(1, 5):
            a, b, _ = orc.phi_pair([[z]], 1.0, l)
            assert abs(a[0] - z * b[0] - 1 / math.factorial(l)) <= 1e-13


def test_phi_matrix_recurrence(orc):
    # phi_p(tH)e1 = tH phi_{p+1}(tH)e1 + e1/p!
    rng = np.random.default_rng(9)
    m = 12
    H = np.triu(rng.standard_normal((m, m)), -1)
    for p in (1, 2, 3):
        a, b, _ = orc.phi_pair(H, 0.7, p)
        e1 = np.zeros(m); e1[0] = 1
        assert np.abs(a - 0.7 * H @ b - e1 / math.factorial(p)).max() <= 1e-11


def test_phi_vs_taylor(orc):
    # phi_p(tH) e1 = sum_k (tH)^k e1/(k+p)!  for ||tH||_1 <= 2
    rng = np.random.default_rng(13)
    for m in (1, 4, 10):
        H = rng.standard_normal((m, m))
        H *= 2.0 / np.abs(H).sum(axis=0).max()
        for p in range(5):
            e1 = np.zeros(m); e1[0] = 1
            acc_p = np.zeros(m); acc_q = np.zeros(m)
            v = e1.copy()
            for k in range(60):
                acc_p += v / math.factorial(k + p)
                acc_q += v / math.factorial(k + p + 1)
                v = H @ v
            a, b, _ = orc.phi_pair(H, 1.0, p)
            assert np.abs(a - acc_p).max() <= 1e-12
            assert np.abs(b - acc_q).max() <= 1e-12


def test_phi_diagonal_and_symmetric_large_norm(orc):
    # diagonal H: phi_p(tD) e1 = phi_p(t d_1) e1
    d = np.array([-40.0, -3.0, 0.5, 2.0])
    a, b, _ = orc.phi_pair(np.diag(d), 1.0, 2)
    assert a[0] == pytest.approx(float(phi_scalar(2, np.array([-40.0]))[0]), rel=1e-13)
    assert np.all(a[1:] == 0) and np.all(b[1:] == 0)
    # symmetric tridiagonal with large norm (scaling and squaring active): eigen route
    rng = np.random.default_rng(17)
    m = 40
    al = -rng.uniform(0, 400, m)
    be = rng.uniform(1, 100, m - 1)
    T = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    lam, Q = np.linalg.eigh(T)
    for p in (0, 1, 3):
        a, b, _ = orc.phi_pair(T, 0.01, p)
        ra = Q @ (phi_scalar(p, 0.01 * lam) * Q[0])
        rb = Q @ (phi_scalar(p + 1, 0.01 * lam) * Q[0])
        assert np.abs(a - ra).max() <= 1e-12 * max(1.0, np.abs(ra).max())
        assert np.abs(b - rb).max() <= 1e-12 * max(1.0, np.abs(rb).max())
