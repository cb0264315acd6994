"""Randomised GPU parity on shapes the fixed cases do not cover (seeded, reproducible): random grid sizes
and coefficients for every stencil form (CSR build and SpMV bit-exact vs the oracle), random CSR
matrices with empty and long rows (SpMV within 1e-13, ||A||_inf bit-exact), random-length dots, and a
few random small/streaming solves against the oracle."""
import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(20261019)


def rand_coefs(rng, dim, nine=False):
    c = rng.integers(-64, 64, 7) / 16.0                     # exact binary fractions
    if dim < 3:
        c[5:] = 0.0
    if dim < 2:
        c[3:5] = 0.0
    corn = tuple(rng.integers(-64, 64, 4) / 16.0) if nine else (0.0,) * 4
    return tuple(float(x) for x in c), corn


def csr_ref(dim, nx, ny, nz, c, corn, nine):
    """Row-by-row CSR of the stencil (ascending columns), built here independently."""
    rp, col, val = [0], [], []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = i + nx * (j + ny * k)
                ent = []
                if dim >= 3 and k > 0:
                    ent.append((r - nx * ny, c[5]))
                if nine:
                    for dx, cv in ((-1, corn[0]), (0, c[3]), (1, corn[1])):
                        if j > 0 and 0 <= i + dx < nx:
                            ent.append((r - nx + dx, cv))
                elif dim >= 2 and j > 0:
                    ent.append((r - nx, c[3]))
                if i > 0:
                    ent.append((r - 1, c[1]))
                ent.append((r, c[0]))
                if i < nx - 1:
                    ent.append((r + 1, c[2]))
                if nine:
                    for dx, cv in ((-1, corn[2]), (0, c[4]), (1, corn[3])):
                        if j < ny - 1 and 0 <= i + dx < nx:
                            ent.append((r + nx + dx, cv))
                elif dim >= 2 and j < ny - 1:
                    ent.append((r + nx, c[4]))
                if dim >= 3 and k < nz - 1:
                    ent.append((r + nx * ny, c[6]))
                for cc, v in ent:
                    col.append(cc)
                    val.append(v)
                rp.append(len(col))
    return np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.float64)


CASES = []
for _ in range(12):
    dim = int(RNG.integers(1, 4))
    nine = dim == 2 and bool(RNG.integers(0, 2))
    if dim == 1:
        dims = (int(RNG.integers(1, 20000)), 1, 1)
    elif dim == 2:
        dims = (int(RNG.integers(1, 300)), int(RNG.integers(1, 120)), 1)
    else:
        dims = tuple(int(x) for x in RNG.integers(1, 40, 3))
    CASES.append((dim, dims, nine, int(RNG.integers(0, 1 << 30))))


@pytest.mark.parametrize("dim,dims,nine,seed", CASES)
def test_random_stencil_csr_and_spmv_bit_exact(ctx, orc, dim, dims, nine, seed):
    rng = np.random.default_rng(seed)
    c, corn = rand_coefs(rng, dim, nine)
    S = P.Stencil(dim, *dims, c, corn, 9 if nine else 0)
    ref = csr_ref(dim, *dims, c, corn, nine)
    rp, col, val = ctx.csr_from_stencil(S)
    assert np.array_equal(rp.cpu().numpy(), ref[0]) and np.array_equal(col.cpu().numpy(), ref[1])
    assert np.array_equal(val.cpu().numpy(), ref[2])
    x = rng.standard_normal(S.n)
    assert np.array_equal(ctx.spmv_stencil(S, to_dev(x)).cpu().numpy(), orc.spmv(ref, x))
    assert P.inf_norm_stencil(S) == orc.inf_norm(ref)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_random_csr(ctx, orc, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60000))
    lens = rng.integers(0, 24, n)
    lens[rng.random(n) < 0.05] = 0
    lens[rng.random(n) < 0.01] = 200                        # a few long rows
    lens = np.minimum(lens, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32) \
        if rp[-1] else np.zeros(0, np.int32)
    val = rng.standard_normal(len(col))
    x = rng.standard_normal(n)
    A = (to_dev(rp), to_dev(col), to_dev(val))
    y = ctx.spmv_csr(A, to_dev(x)).cpu().numpy()
    ref = orc.spmv((rp, col, val), x)
    absAx = orc.spmv((rp, col, np.abs(val)), np.abs(x))
    assert np.all(np.abs(y - ref) <= 1e-13 * absAx)
    assert ctx.inf_norm_csr(A) == orc.inf_norm((rp, col, val))


@pytest.mark.parametrize("n", [int(x) for x in RNG.integers(1, 3_000_000, 6)])
def test_random_dot(ctx, orc, n):
    rng = np.random.default_rng(n)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    d = ctx.dot(to_dev(x), to_dev(y))
    assert abs(d - orc.dot(x, y)) <= 1e-13 * np.abs(x * y).sum()


@pytest.mark.parametrize("seed,n,p,symmetric", [(11, 700, 1, True), (12, 5000, 3, False), (13, 20000, 2, True),
                                                 (14, 150000, 0, False), (15, 9000, 4, False)])
def test_random_banded_solves(ctx, orc, seed, n, p, symmetric):
    # random banded operators (nonsymmetric unless symmetrised), small-kernel and streaming paths
    rng = np.random.default_rng(seed)
    rp, col, val = W.random_banded_csr(rng, n, band=min(64, n - 1), k_off=min(7, n - 1))
    if symmetric:
        import scipy.sparse as sp
        A = sp.csr_matrix((val, col, rp), shape=(n, n))
        A = ((A + A.T) * 0.5).tocsr()
        A.sort_indices()
        rp, col, val = A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data.copy()
    u = [rng.standard_normal(n)] + [rng.uniform(-1, 1, n) for _ in range(p)]
    t, tol = 0.3, 1e-9
    wo, so, _ = orc.phipm(t, (rp, col, val), u, tol, m_init=10, m_max=100, symmetric=symmetric)
    assert so["status"] == 0
    w, s = ctx.solve_csr(t, (to_dev(rp), to_dev(col), to_dev(val)), [to_dev(x) for x in u], tol=tol,
                         symmetric=symmetric)
    assert s.t_reached == t
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol)


@pytest.mark.parametrize("kind", ["uniform", "alternating", "one_long_row"])
def test_csr_analysis_streaming_path(orc, kind):
    # nnz = 8 n in every case, so the analysis takes the streaming uniform-row kernel first
    # (csr_analyze_ell_kernel); rows that are not all of length 8 must be caught (row_ptr check) and
    # the general pass rerun, or the x-ring SpMV would run with a wrong band.  Solve vs the oracle.
    rng = np.random.default_rng(77)
    n, L, band = 20000, 8, 200            # n > SMALL_N: the streaming (x-ring) SpMV uses the band
    if kind == "uniform":
        lens = np.full(n, L)
    elif kind == "alternating":
        lens = np.where(np.arange(n) % 2 == 0, 4, 12)
    else:
        lens = np.full(n, L)
        lens[0] = 1
        lens[1] = 2 * L - 1
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    assert rp[-1] == L * n
    col = np.empty(rp[-1], np.int32)
    val = np.empty(rp[-1], np.float64)
    for r in range(n):
        k = lens[r]
        lo, hi = max(0, r - band), min(n - 1, r + band)
        cs = np.sort(rng.choice(np.arange(lo, hi + 1), size=k, replace=False))
        if r not in cs:
            cs[np.argmin(np.abs(cs - r))] = r
            cs = np.sort(cs)
        v = rng.standard_normal(k) / 4
        v[cs == r] = 0.0
        v[cs == r] = -(np.abs(v).sum()) - 1.0
        col[rp[r]:rp[r + 1]] = cs
        val[rp[r]:rp[r + 1]] = v
    csr = (rp.astype(np.int32), col, val)
    u = [rng.standard_normal(n), rng.uniform(-1, 1, n)]
    t, tol = 0.5, 1e-8
    wo, so, _ = orc.phipm(t, csr, u, tol, m_init=10, m_max=100, symmetric=False)
    ctx = P.Context(n_max=n, m_max=100, p_max=2)
    w, s = ctx.solve_csr(t, tuple(to_dev(a) for a in csr), [to_dev(x) for x in u], tol=tol, symmetric=False)
    ctx.close()
    assert s.t_reached == t
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol), (s, so)
