"""Pins for the oracle's operator pieces: stencil nnz / CSR build, SpMV, ||A||_inf, and the inputs."""
import numpy as np
import pytest
import scipy.sparse as sp

import workloads as W


def dense_stencil(st):
    """Independent dense construction: Kronecker sum of 1-D tridiagonal pieces + centre."""
    dims = [st.nx, st.ny, st.nz]
    c0, cxm, cxp, cym, cyp, czm, czp = st.coeffs
    def tri_off(N, lo, hi):
        return np.diag(np.full(N - 1, lo), -1) + np.diag(np.full(N - 1, hi), 1)
    nx, ny, nz = dims
    Ix, Iy, Iz = np.eye(nx), np.eye(ny), np.eye(nz)
    A = c0 * np.eye(nx * ny * nz)
    A = A + np.kron(Iz, np.kron(Iy, tri_off(nx, cxm, cxp)))
    if st.dim >= 2:
        A = A + np.kron(Iz, np.kron(tri_off(ny, cym, cyp), Ix))
    if st.dim >= 3:
        A = A + np.kron(tri_off(nz, czm, czp), np.kron(Iy, Ix))
    return A


STENCILS = [
    W.Stencil(1, 9, 1, 1, (-2.0, 1.0, 1.5, 0, 0, 0, 0)),
    W.Stencil(2, 5, 4, 1, (-4.0, 1.0, 2.0, 3.0, 4.0, 0, 0)),
    W.Stencil(2, 1, 6, 1, (-4.0, 1.0, 2.0, 3.0, 4.0, 0, 0)),
    W.Stencil(3, 3, 4, 5, (-6.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0)),
    W.Stencil(3, 1, 1, 1, (-6.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0)),
]


@pytest.mark.parametrize("st", STENCILS)
def test_csr_from_stencil_matches_dense(orc, st):
    rp, col, val = orc.csr_from_stencil(st)
    A = sp.csr_matrix((val, col, rp), shape=(st.n, st.n)).toarray()
    D = dense_stencil(st)
    # structural entries with coefficient 0 are kept; compare values
    assert np.array_equal(A, D)
    for r in range(st.n):
        seg = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(seg) > 0)


@pytest.mark.parametrize("dim,dims,formula", [
    (1, (1000, 1, 1), lambda n, x, y, z: 3 * n - 2),
    (2, (256, 256, 1), lambda n, x, y, z: 5 * n - 2 * (x + y)),
    (2, (7, 3, 1), lambda n, x, y, z: 5 * n - 2 * (x + y)),
    (3, (128, 128, 128), lambda n, x, y, z: 7 * n - 2 * (x * y + x * z + y * z)),
    (3, (3, 4, 5), lambda n, x, y, z: 7 * n - 2 * (x * y + x * z + y * z)),
])
def test_stencil_nnz_closed_forms(orc, dim, dims, formula):
    st = W.Stencil(dim, *dims, (0.0,) * 7)
    assert orc.stencil_nnz(st) == formula(st.n, *dims)


def test_spmv_and_infnorm_vs_scipy(orc):
    P = W.make("c5_mini")
    rp, col, val = P.csr
    A = sp.csr_matrix((val, col, rp), shape=(P.n, P.n))
    x = np.random.default_rng(1).standard_normal(P.n)
    y = orc.spmv(P.csr, x)
    ref = A @ x
    scale = abs(A) @ np.abs(x)
    assert np.all(np.abs(y - ref) <= 1e-15 * scale)
    assert orc.inf_norm(P.csr) == pytest.approx(np.abs(A).sum(axis=1).max(), rel=1e-15)


def test_config_norms(orc):
    # ||A||_inf values written out from the definitions (SURVEY §8 header table)
    assert orc.inf_norm(orc.csr_from_stencil(W.c1().stencil)) == 4 * 1001 ** 2
    assert orc.inf_norm(orc.csr_from_stencil(W.c2(nx=256).stencil)) == 8 * 257 ** 2
    c3 = W.c3(nx=64).stencil
    assert orc.inf_norm(orc.csr_from_stencil(c3)) == 8 * 0.01 * 65 ** 2 + 3 * 65 * 0.5 * 2


def test_c5_structure():
    P = W.make("c5_mini")
    rp, col, val = P.csr
    n = P.n
    assert np.all(np.diff(rp) == 16)
    C = col.reshape(n, 16).astype(np.int64)
    Vv = val.reshape(n, 16)
    rows = np.arange(n)[:, None]
    assert np.all(np.diff(C, axis=1) > 0)
    assert np.all(np.abs(C - rows) <= 64) and C.min() >= 0 and C.max() < n
    dmask = C == rows
    assert np.all(dmask.sum(axis=1) == 1)
    off = np.where(dmask, 0.0, np.abs(Vv))
    s = np.zeros(n)
    for c in range(16):
        s = s + off[:, c]
    assert np.array_equal(Vv[dmask], -s - 1.0)       # diagonal = -(row abs sum) - 1
    # Gershgorin: every disc in Re z <= -1 (spectrum in the left half-plane)
    assert np.all(Vv[dmask] + s <= -1.0 + 1e-12)


def test_generators_deterministic():
    a, b = W.make("c5_mini"), W.make("c5_mini")
    assert W.sha256_of(*a.csr, *a.u) == W.sha256_of(*b.csr, *b.u)
    c, d = W.make("c3_mini"), W.make("c3_mini")
    assert W.sha256_of(*c.u) == W.sha256_of(*d.u)
    assert W.make("c1").u[0].shape == (1000,)
