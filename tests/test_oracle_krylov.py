"""Pins for the oracle's Krylov projection (Algorithms 1-2)."""
import math

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp

import workloads as W
from exact import dense_from_csr


def _csr_dense(D):
    S = sp.csr_matrix(D)
    S.sort_indices()
    return (S.indptr.astype(np.int32), S.indices.astype(np.int32), S.data.astype(np.float64))


def test_arnoldi_relation_and_orthonormality(orc):
    P = W.make("c5_mini")
    A = sp.csr_matrix((P.csr[2], P.csr[1], P.csr[0]), shape=(P.n, P.n))
    V, H, k, brk, beta = orc.krylov(P.csr, P.u[0], 30, symmetric=False)
    assert k == 30 and not brk
    normA = orc.inf_norm(P.csr)
    R = A @ V[:, :k] - V[:, :k + 1] @ H[:k + 1, :k]          # A V_m = V_{m+1} Hbar_m
    assert np.abs(R).max() <= 1e-10 * normA
    assert np.allclose(np.tril(H[:k, :k], -2), 0)              # Hessenberg
    assert np.allclose(V[:, 0], P.u[0] / np.linalg.norm(P.u[0]), rtol=0, atol=1e-15)
    # MGS keeps orthonormality while the basis is well conditioned (SPEC S:261 at m=8; the solve
    # uses m=10-12 here); at m=30 the Krylov vectors of c5 converge and MGS loses it
    V, H, k, brk, beta = orc.krylov(P.csr, P.u[0], 8, symmetric=False)
    assert np.abs(V.T @ V - np.eye(k + 1)).max() <= 1e-10


def test_arnoldi_orthonormal_random_dense(orc):
    # random dense A, n <= 100, m <= 30
    rng = np.random.default_rng(2)
    D = rng.standard_normal((100, 100))
    csr = _csr_dense(D)
    V, H, k, brk, beta = orc.krylov(csr, rng.standard_normal(100), 30, symmetric=False)
    assert k == 30
    assert np.abs(V.T @ V - np.eye(31)).max() <= 1e-10


def test_lanczos_matches_arnoldi_on_symmetric(orc):
    P = W.make("c2_mini")
    csr = orc.operator_csr(P)
    Va, Ha, ka, _, _ = orc.krylov(csr, P.u[0], 10, symmetric=False)
    Vl, Hl, kl, _, _ = orc.krylov(csr, P.u[0], 10, symmetric=True)
    assert ka == kl == 10
    scale = orc.inf_norm(csr)
    assert np.abs(Ha - Hl).max() <= 1e-8 * scale
    assert np.allclose(Hl[:10, :10], Hl[:10, :10].T)            # tridiagonal T symmetric
    A = dense_from_csr(csr)
    R = A @ Vl[:, :10] - Vl[:, :11] @ Hl[:11, :10]
    assert np.abs(R).max() <= 1e-10 * scale


def test_lanczos_first_entry(orc):
    # 1-D Laplacian n=5, seed e1: t_11 = -2
    st = W.Stencil(1, 5, 1, 1, (-2.0, 1.0, 1.0, 0, 0, 0, 0))
    csr = orc.csr_from_stencil(st)
    e1 = np.zeros(5); e1[0] = 1
    V, H, k, brk, _ = orc.krylov(csr, e1, 3, symmetric=True)
    assert H[0, 0] == -2.0 and H[1, 0] == 1.0


def test_breakdown_examples(orc):
    # diag(1,2), seed e1 -> m truncates to 1, H=[1]
    csr = _csr_dense(np.diag([1.0, 2.0]))
    V, H, k, brk, _ = orc.krylov(csr, np.array([1.0, 0.0]), 2, symmetric=False)
    assert k == 1 and brk and H[0, 0] == 1.0
    # [[0,1],[0,0]], seed [0,1], m=2: v1=[0,1], v2=[1,0], H=[[0,0],[1,0]], breakdown at 2
    csr = _csr_dense(np.array([[0.0, 1.0], [0.0, 0.0]]))
    V, H, k, brk, _ = orc.krylov(csr, np.array([0.0, 1.0]), 2, symmetric=False)
    assert k == 2 and brk
    assert np.array_equal(V[:, 0], [0, 1]) and np.array_equal(V[:, 1], [1, 0])
    assert np.array_equal(H[:2, :2], [[0, 0], [1, 0]])


def test_full_dimension_is_exact(orc):
    # m = n -> beta V phi_p(tau H) e1 = phi_p(tau A) v (dense augmented reference)
    rng = np.random.default_rng(21)
    n = 12
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.4) + np.diag(rng.uniform(-3, 0, n))
    csr = _csr_dense(D)
    v = rng.standard_normal(n)
    V, H, k, brk, beta = orc.krylov(csr, v, n, symmetric=False)
    for p in (0, 1, 3):
        tau = 0.6
        a, b, _ = orc.phi_pair(H[:k, :k], tau, p)
        approx = beta * V[:, :k] @ a
        # phi_p(tau A) v from the (n+p) augmented matrix [[tau A, v, 0],[0,0,I],[0,0,0]]
        K = n + p
        Ah = np.zeros((K + (1 if p == 0 else 0),) * 2)
        if p == 0:
            ref = scipy.linalg.expm(tau * D) @ v
        else:
            Ah = np.zeros((n + p, n + p))
            Ah[:n, :n] = tau * D
            Ah[:n, n] = v
            for i in range(1, p):
                Ah[n + i - 1, n + i] = 1.0
            ref = scipy.linalg.expm(Ah)[:n, n + p - 1]
        assert np.linalg.norm(approx - ref) <= 1e-10 * np.linalg.norm(ref)
