"""NEXT-4: 2-D 9-point stencils (the class of the paper's gr_30_30) and Matrix Market
ingestion, through the whole GPU path, against the oracle on a CSR built here independently (plain
row-by-row loops, columns ascending).  Coefficients are distinct exact binary fractions so that an
index or ordering mistake changes bits."""
import os

import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev
from ninept import csr_9pt as _csr_9pt, gr9_coeffs, ROUNDTRIP

pytestmark = pytest.mark.gpu

# (centre, xm, xp, ym, yp) and corners (xmym, xpym, xmyp, xpyp)
COEF = (-4.0, 0.5, 0.25, 0.125, 1.5, 0.0, 0.0)
CORN = (0.0625, 0.375, 0.75, 1.25)


def csr_9pt(nx, ny, coef=COEF, corn=CORN):
    return _csr_9pt(nx, ny, coef, corn)


def stencil(nx, ny, coef=COEF, corn=CORN):
    return P.Stencil(2, nx, ny, 1, coef, corn, 9)


SIZES = [(30, 30), (37, 53), (301, 301), (5000, 30)]    # small kernel, ragged, streaming, nx > tile


@pytest.mark.parametrize("nx,ny", SIZES)
def test_csr_from_9pt_stencil_bit_exact(ctx, nx, ny):
    rp, col, val = ctx.csr_from_stencil(stencil(nx, ny))
    r2, c2, v2 = csr_9pt(nx, ny)
    assert ctx.stencil_nnz(stencil(nx, ny)) == len(c2) == (3 * nx - 2) * (3 * ny - 2)
    assert np.array_equal(rp.cpu().numpy(), r2)
    assert np.array_equal(col.cpu().numpy(), c2)
    assert np.array_equal(val.cpu().numpy(), v2)


@pytest.mark.parametrize("nx,ny", SIZES)
def test_spmv_9pt_stencil_bit_exact(ctx, orc, nx, ny):
    x = np.random.default_rng(nx * ny).standard_normal(nx * ny)
    y = ctx.spmv_stencil(stencil(nx, ny), to_dev(x)).cpu().numpy()
    assert np.array_equal(y, orc.spmv(csr_9pt(nx, ny), x))


def heat_9pt(nx, ny, seed):
    """gr_30_30-like problem: A = h^-2 (9-point Laplacian, 8 on the diagonal, -1 off it), heat sign
    (negative definite); u0 ~ N(0,1), u1, u2 ~ U[-1,1]; p = 2, Lanczos."""
    h2 = float((nx + 1) ** 2)
    coef = (-8.0 * h2, h2, h2, h2, h2, 0.0, 0.0)
    corn = (h2,) * 4
    rng = np.random.default_rng(seed)
    n = nx * ny
    u = [rng.standard_normal(n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    return coef, corn, u


@pytest.mark.parametrize("nx,ny", [(30, 30), (301, 301)])
def test_solve_9pt_parity(ctx, orc, nx, ny):
    coef, corn, u = heat_9pt(nx, ny, 11)
    csr = csr_9pt(nx, ny, coef, corn)
    t, tol = 1e-4, 1e-10
    wo, so, _ = orc.phipm(t, csr, u, tol, m_init=10, m_max=100, symmetric=True)
    assert so["status"] == 0
    ud = [to_dev(x) for x in u]
    ws, ss = ctx.solve_stencil(t, stencil(nx, ny, coef, corn), ud, tol=tol, symmetric=True)
    wc, sc = ctx.solve_csr(t, tuple(to_dev(a) for a in csr), ud, tol=tol, symmetric=True)
    for w in (ws, wc):
        assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol)


def test_matrix_market_roundtrip_solve(ctx, orc, tmp_path):
    # a 9-point matrix written by scipy.io.mmwrite, read by phipm_mm_read, solved on the GPU
    import scipy.io
    import scipy.sparse as sp
    coef, corn, u = heat_9pt(30, 30, 12)
    csr = csr_9pt(30, 30, coef, corn)
    path = os.path.join(tmp_path, "gr_30_30_like.mtx")
    scipy.io.mmwrite(path, sp.csr_matrix((csr[2], csr[1], csr[0]), shape=(900, 900)), precision=17)
    rp, col, val = P.read_matrix_market(path)
    assert np.array_equal(rp, csr[0]) and np.array_equal(col, csr[1]) and np.array_equal(val, csr[2])
    t, tol = 1e-3, 1e-10
    wo, so, _ = orc.phipm(t, (rp, col, val), u, tol, m_init=10, m_max=100, symmetric=True)
    w, s = ctx.solve_csr(t, (to_dev(rp), to_dev(col), to_dev(val)), [to_dev(x) for x in u], tol=tol, symmetric=True)
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol)
    # c5_mini (random banded, Arnoldi) through a Matrix Market file as well
    Pb = W.make("c5_mini")
    path = os.path.join(tmp_path, "c5_mini.mtx")
    scipy.io.mmwrite(path, sp.csr_matrix((Pb.csr[2], Pb.csr[1], Pb.csr[0]), shape=(Pb.n, Pb.n)), precision=17)
    A = P.read_matrix_market(path)
    w, s = ctx.solve_csr(Pb.t, tuple(to_dev(a) for a in A), [to_dev(x) for x in Pb.u], tol=Pb.tol)
    wo, so, _ = orc.solve(Pb)
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(Pb.tol)


@pytest.mark.parametrize("path", ["stencil", "csr"])
def test_roundtrip_gr30(ctx, orc, path):
    """NEXT-4, the paper's round trip: w = e^{tA} b0, then e^{-tA} w, b0 = ones, t = 2,
    Tol = 1e-14, on the gr_30_30-class 9-point operator (tests/ninept.py, reading R41).  The backward
    leg uses the ABI's negation rule (t >= 0 only: e^{-tA} = e^{t(-A)}, Stencil.negated()).
    Each GPU leg is held to the BASELINE bar against the oracle's leg on the same input; the round
    trip itself is compared with b0, the exact answer, and reported beside the paper's 3.9e-6."""
    nx, ny, t, tol = ROUNDTRIP["nx"], ROUNDTRIP["ny"], ROUNDTRIP["t"], ROUNDTRIP["tol"]
    coef, corn = gr9_coeffs(-1.0)
    S = P.Stencil(2, nx, ny, 1, coef, corn, 9)
    fwd = csr_9pt(nx, ny, coef, corn)
    bwd = csr_9pt(nx, ny, *gr9_coeffs(+1.0))
    n = nx * ny
    b0 = np.ones(n)
    if path == "stencil":
        run = lambda op, x: ctx.solve_stencil(t, op, [to_dev(x)], tol=tol, symmetric=True)
        ops = (S, S.negated())
    else:
        run = lambda op, x: ctx.solve_csr(t, op, [to_dev(x)], tol=tol, symmetric=True)
        ops = tuple(tuple(to_dev(a) for a in c) for c in (fwd, bwd))
    wg, sf = run(ops[0], b0)
    wg = wg.cpu().numpy()
    wo, so, _ = orc.phipm(t, fwd, [b0], tol, symmetric=True)
    assert relerr(wg, wo) <= parity_bound(tol), (sf, so)
    bg, sb = run(ops[1], wg)
    bg = bg.cpu().numpy()
    bo, so2, _ = orc.phipm(t, bwd, [wg], tol, symmetric=True)       # same input as the GPU leg
    assert relerr(bg, bo) <= parity_bound(tol), (sb, so2)
    err = relerr(bg, b0)
    print(f"gr30 round trip ({path}): GPU relerr vs b0 {err:.2e} (paper phipm {ROUNDTRIP['paper_phipm_error']:.1e}); "
          f"fwd {sf} bwd {sb}")
    assert err <= 1e-12
