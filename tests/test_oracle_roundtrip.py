"""NEXT-4: the paper's exponential round trip (§4.2) on a gr_30_30-class operator,
oracle side.  The exact answer of e^{-tA} e^{tA} b0 is b0 itself ("Only the third example has a known
exact solution"), and the forward leg e^{tA} b0 is pinned to scipy's dense expm (an
independent implementation) at n = 900.  The paper's phipm reaches 3.9e-6 on gr_30_30 (Table 1,
P:1290); the oracle's error is reported next to it."""
import numpy as np
import scipy.linalg
import scipy.sparse as sp

from ninept import csr_9pt, gr9_coeffs, ROUNDTRIP as RT


def test_gr9_structure():
    # n = 900, nnz = 7744 ((3N-2)^2)
    coef, corn = gr9_coeffs(-1.0)
    rp, col, val = csr_9pt(30, 30, coef, corn)
    assert len(rp) - 1 == 900 and len(col) == 7744 == (3 * 30 - 2) ** 2
    D = sp.csr_matrix((val, col, rp), shape=(900, 900)).toarray()
    assert np.array_equal(D, D.T)
    ev = np.linalg.eigvalsh(D)
    assert ev.min() > 0 and ev.max() < 32 / 6          # positive definite, spectrum in (0, 16/3)


def test_roundtrip_oracle(orc):
    nx, ny, t, tol = RT["nx"], RT["ny"], RT["t"], RT["tol"]
    fwd = csr_9pt(nx, ny, *gr9_coeffs(-1.0))                 # A (positive-signed, like gr_30_30)
    bwd = csr_9pt(nx, ny, *gr9_coeffs(+1.0))                 # -A: e^{-tA} with t > 0 (ABI negation rule)
    n = nx * ny
    b0 = np.ones(n)
    w, s, _ = orc.phipm(t, fwd, [b0], tol, symmetric=True)
    assert s["status"] == 0 and s["t_reached"] == t
    D = sp.csr_matrix((fwd[2], fwd[1], fwd[0]), shape=(n, n)).toarray()
    w_dense = scipy.linalg.expm(t * D) @ b0
    assert np.linalg.norm(w - w_dense) / np.linalg.norm(w_dense) <= 1e-12
    b, s2, _ = orc.phipm(t, bwd, [w], tol, symmetric=True)
    assert s2["status"] == 0
    err = np.linalg.norm(b - b0) / np.linalg.norm(b0)
    print(f"oracle round trip: relerr {err:.2e} (paper's phipm on gr_30_30: {RT['paper_phipm_error']:.1e}); "
          f"fwd {s} bwd {s2}")
    assert err <= 1e-12
