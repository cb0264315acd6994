"""9-point stencil helpers shared by the CPU pins and the GPU parity tests (no method arithmetic):
a plain row-by-row CSR builder and the coefficients of the round-trip operator of NEXT-4."""
import numpy as np


def csr_9pt(nx, ny, coef, corn):
    """CSR of a 2-D 9-point stencil with Dirichlet truncation, entries of a row in ascending column
    order.  coef = (centre, xm, xp, ym, yp, ...), corn = (xmym, xpym, xmyp, xpyp)."""
    c0, cxm, cxp, cym, cyp = coef[:5]
    cmm, cpm, cmp, cpp = corn
    w = {(-1, -1): cmm, (0, -1): cym, (1, -1): cpm, (-1, 0): cxm, (0, 0): c0, (1, 0): cxp,
         (-1, 1): cmp, (0, 1): cyp, (1, 1): cpp}
    rp, col, val = [0], [], []
    for j in range(ny):
        for i in range(nx):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    ii, jj = i + dx, j + dy
                    if 0 <= ii < nx and 0 <= jj < ny:
                        col.append(ii + nx * jj)
                        val.append(w[(dx, dy)])
            rp.append(len(col))
    return np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.float64)


def gr9_coeffs(sign=1.0, h=1.0):
    """The 9-point Laplacian of SPEC gen_laplacian9, (1/(6h^2)) [1 4 1; 4 -20 4; 1 4 1],
    times `sign`.  sign = -1 is the positive-semidefinite-signed variant, the class of the paper's
    gr_30_30 (symmetric, 9-point, 30x30, n = 900, nnz = 7744).  h = 1 (reading R41):
    the round trip e^{-tA} e^{tA} at t = 2 needs a spectrum of O(1) width, as gr_30_30's is; with
    h = 1/31 the forward leg would amplify by e^{2 t ||A||} ~ e^{25600}.
    Returns (coef 7-tuple, corners 4-tuple)."""
    s = sign / (6.0 * h * h)
    return (-20.0 * s, 4.0 * s, 4.0 * s, 4.0 * s, 4.0 * s, 0.0, 0.0), (s, s, s, s)


# NEXT-4 round trip: t = 2, b0 = ones, Tol = 1e-14 on the 30 x 30 grid; the paper's
# Table 1 reports a phipm relative error of 3.9e-6 for this experiment on gr_30_30
ROUNDTRIP = dict(nx=30, ny=30, t=2.0, tol=1e-14, paper_phipm_error=3.9e-6)
