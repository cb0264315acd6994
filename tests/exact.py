"""Exact / independent references used to PIN the oracle (and, transitively, the GPU path).

None of these call the oracle or the product.  Each is a textbook special case or a brute-force
construction that reaches the exact w(t) = phi_0(tA)u_0 + sum_k t^k phi_k(tA) u_k
(PAPER.md Eq. lincomb2/phide) by a route unrelated to the Krylov method:

  * phi_scalar       — phi_l(z) from the Taylor series of Eq. (phifunctions) for |z|<=1
                       and the recurrence Eq. (phirelation) upward from e^z otherwise;
  * brute_augmented  — first n entries of expm(t [[A, U],[0, J]]) [u0; e_p] (BASELINE.json
                       north_star: "brute-force dense exp of the (n+p)x(n+p) augmented matrix");
  * dst_solution     — Dirichlet Laplacians are diagonalised by the orthonormal DST-I
                       (eigenvalues -4/h^2 sin^2(k pi/(2(N+1))) per direction, Kronecker sum);
  * kron_quadrature  — 2-D operators I(x)Ax + Ay(x)I: exp(sA)v = vec(Ey(s) V Ex(s)^T), phi_k by
                       composite Gauss-Legendre quadrature of the integral definition;
  * taylor_augmented — scaled truncated Taylor series of the augmented operator applied to
                       [u0; e_p] (the paper's own "exact" references come from expmv).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.fft
import scipy.linalg
import scipy.sparse as sp


def phi_scalar(ell: int, z):
    """phi_ell(z) elementwise for real z (array)."""
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    small = np.abs(z) <= 1.0
    zs = z[small]
    acc = np.zeros_like(zs)
    for k in range(40, -1, -1):                       # sum_k z^k/(k+ell)!  (Horner)
        acc = acc * zs + 1.0 / math.factorial(k + ell)
    out[small] = acc
    zl = z[~small]
    ph = np.exp(zl)
    for l in range(ell):                              # phi_{l+1} = (phi_l - 1/l!)/z
        ph = (ph - 1.0 / math.factorial(l)) / zl
    out[~small] = ph
    return out


def combine_spectral(lam, uhat, t):
    """sum_k t^k phi_k(t lam) uhat_k for diagonal operators (lam, uhat_k in the eigenbasis)."""
    w = np.zeros_like(uhat[0])
    for k, uk in enumerate(uhat):
        w = w + (t ** k) * phi_scalar(k, t * lam) * uk
    return w


def brute_augmented(A_dense, u, t):
    A = np.asarray(A_dense, dtype=np.float64)
    n = A.shape[0]
    p = len(u) - 1
    Ahat = np.zeros((n + p, n + p))
    Ahat[:n, :n] = A
    for i in range(p):                                # column i holds u_{p-i}
        Ahat[:n, n + i] = u[p - i]
    for i in range(p - 1):                            # J: shift
        Ahat[n + i, n + i + 1] = 1.0
    y0 = np.zeros(n + p)
    y0[:n] = u[0]
    if p > 0:
        y0[n + p - 1] = 1.0
    return (scipy.linalg.expm(t * Ahat) @ y0)[:n]


def _dirichlet_eigs(N, inv_h2):
    k = np.arange(1, N + 1, dtype=np.float64)
    return -4.0 * inv_h2 * np.sin(k * np.pi / (2.0 * (N + 1))) ** 2


def dst_solution(stencil, u, t):
    """Exact w for the constant-coefficient Dirichlet Laplacian stencils of c1/c2/c4."""
    dims = [stencil.nx, stencil.ny, stencil.nz][: stencil.dim]
    inv_h2 = stencil.coeffs[1]
    shape = tuple(reversed(dims))                     # C order: x fastest
    lam = np.zeros(shape)
    for ax, N in enumerate(reversed(dims)):
        e = _dirichlet_eigs(N, inv_h2)
        sh = [1] * len(shape)
        sh[ax] = N
        lam = lam + e.reshape(sh)
    uhat = [scipy.fft.dstn(x.reshape(shape), type=1, norm="ortho") for x in u]
    what = combine_spectral(lam, uhat, t)
    return scipy.fft.idstn(what, type=1, norm="ortho").ravel()


def _tri(N, sub, diag, sup):
    return (np.diag(np.full(N, diag)) + np.diag(np.full(N - 1, sub), -1)
            + np.diag(np.full(N - 1, sup), 1))


def kron_quadrature(stencil, u, t, panels=8, nodes=16):
    """Exact-to-quadrature w for 2-D stencils (c3): A = I (x) Ax + Ay (x) I."""
    assert stencil.dim == 2
    c0, cxm, cxp, cym, cyp = stencil.coeffs[:5]
    nx, ny = stencil.nx, stencil.ny
    # split the centre coefficient between the directions: any split gives the same A
    dx = -(cxm + cxp)
    dy = c0 - dx
    Ax = _tri(nx, cxm, dx, cxp)
    Ay = _tri(ny, cym, dy, cyp)
    U = [x.reshape(ny, nx) for x in u]
    E = lambda s, X: scipy.linalg.expm(s * Ay) @ X @ scipy.linalg.expm(s * Ax).T
    w = E(t, U[0])
    if len(u) > 1:
        xg, wg = np.polynomial.legendre.leggauss(nodes)
        edges = np.linspace(0.0, 1.0, panels + 1)
        for a, b in zip(edges[:-1], edges[1:]):
            th = 0.5 * (b - a) * xg + 0.5 * (a + b)
            wt = 0.5 * (b - a) * wg
            for thi, wi in zip(th, wt):
                Ea = scipy.linalg.expm((1 - thi) * t * Ay)
                Eb = scipy.linalg.expm((1 - thi) * t * Ax).T
                for k in range(1, len(u)):
                    # t^k phi_k(tA) u_k = t^k/(k-1)! int e^{(1-th)tA} th^{k-1} u_k dth
                    w = w + (t ** k) / math.factorial(k - 1) * wi * thi ** (k - 1) * (Ea @ U[k] @ Eb)
    return w.ravel()


def taylor_augmented(csr, u, t, inf_norm_A):
    """Scaled Taylor series of exp(t Ahat) [u0; e_p], Ahat = [[A, U],[0, J]], via sparse products."""
    rp, col, val = csr
    n = len(rp) - 1
    A = sp.csr_matrix((val, col, rp), shape=(n, n))
    p = len(u) - 1
    Ucols = [u[p - i] for i in range(p)]

    def apply(y):
        x, z = y[:n], y[n:]
        out = np.empty_like(y)
        out[:n] = A @ x
        for i in range(p):
            out[:n] += Ucols[i] * z[i]
        out[n:] = 0.0
        out[n:n + p - 1] = z[1:]
        return out

    s = int(math.ceil(2.0 * t * (inf_norm_A + 1.0)))
    d = t / s
    y = np.zeros(n + p)
    y[:n] = u[0]
    if p > 0:
        y[n + p - 1] = 1.0
    for _ in range(s):
        term = y.copy()
        acc = y.copy()
        for k in range(1, 80):
            term = apply(term) * (d / k)
            acc += term
            if np.linalg.norm(term) <= 1e-18 * np.linalg.norm(acc):
                break
        y = acc
    return y[:n]


def dense_from_csr(csr):
    rp, col, val = csr
    n = len(rp) - 1
    return sp.csr_matrix((val, col, rp), shape=(n, n)).toarray()


def relerr(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))
