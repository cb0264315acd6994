"""Seeded synthetic inputs for the five BASELINE.json configs (c1..c5) and scaled-down variants.

This module is shared by the oracle side (tests, cpu baseline) and the GPU side (tests, bench).
It holds NO arithmetic of the method: it only draws random vectors, writes down stencil
coefficients, and (for c5) builds a random CSR matrix.  The stencil -> CSR conversion is
deliberately NOT here: the oracle (oracle/phipm_oracle.c) and the product
(paper_0907_4631_b200/csrc) each own their own builder, and tests compare them bit-exactly.

Recipes; every draw uses numpy Generator(PCG64(seed)), in the
order listed:

  c1  1-D heat, n=1000, h=1/(n+1), A = h^-2 tridiag(1,-2,1) Dirichlet (h^-2 = (n+1)^2 exactly).
      u0 = sin(pi x) + 0.01 N(0,1); u1, u2 ~ U[-1,1].  p=2, t=1e-3, tol=1e-10, Lanczos.  seed 101.
  c2  2-D 5-point Laplacian on 256x256 interior points, h=1/257, negative definite (heat sign),
      index i + nx*j.  u0 ~ N(0,1); u1..u3 ~ U[-1,1].  p=3, t=1e-4, tol=1e-10, Lanczos.  seed 102.
  c3  2-D advection-diffusion eps*Lap_h - (a_x D_x^- + a_y D_y^-) (first-order upwind for the
      positive velocity (1, 0.5)), eps=1e-2, 1024x1024, h=1/1025, x fastest.
      u0 = exp(-((x-.3)^2+(y-.3)^2)/(2*.05^2)) + 1e-3 N(0,1); u1, u2 ~ U[-1,1].
      p=2, t=1e-3, tol=1e-8, Arnoldi.  seed 103.
  c4  3-D 7-point Laplacian 128^3, h=1/129, index i + nx*(j + ny*k).  u0 ~ N(0,1); u1..u4 ~ U[-1,1].
      p=4, t=1e-5, tol=1e-10, Lanczos.  seed 104.
  c5  random banded CSR, n=4,194,304, 16 nnz/row: the diagonal plus 15 distinct off-diagonal
      columns drawn uniformly from the row's valid offsets {o : 1<=|o|<=4096, 0<=i+o<n}
      (rows with a duplicate are redrawn whole), sorted ascending; off-diagonal values
      N(0,1)/4; diagonal = -(sum_j |a_ij| in ascending column order) - 1.  Draw order:
      offsets (+redraws), values, u0 ~ N(0,1), u1..u3 ~ U[-1,1].  p=3, t=0.5, tol=1e-8,
      Arnoldi.  seed 105.

The paper measures on a Heston finite-difference system and University of Florida matrices
(PAPER.md P:826-936); those are not available, and these configs stand in for them.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import List, Optional, Tuple

import numpy as np

__all__ = ["Stencil", "Problem", "make", "CONFIGS", "sha256_of"]


@dataclasses.dataclass(frozen=True)
class Stencil:
    """Constant-coefficient 3/5/7-point operator on an nx*ny*nz grid with zero Dirichlet data.

    Row r = i + nx*(j + ny*k).  Coefficient order matches include/phipm.h:
    (c_center, c_xm, c_xp, c_ym, c_yp, c_zm, c_zp); unused directions are 0.
    """
    dim: int
    nx: int
    ny: int
    nz: int
    coeffs: Tuple[float, float, float, float, float, float, float]

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    p: int
    t: float
    tol: float
    symmetric: bool
    u: List[np.ndarray]                       # p+1 vectors, float64, C-contiguous
    stencil: Optional[Stencil] = None        # operator as a stencil descriptor
    csr: Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]] = None  # (row_ptr i32, col i32, val f64)
    seed: int = 0
    m_init: int = 10
    m_max: int = 100

    @property
    def u_stack(self) -> np.ndarray:
        return np.ascontiguousarray(np.stack(self.u))


def sha256_of(*arrays: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _uniform(rng, n):
    return rng.uniform(-1.0, 1.0, n)


def c1(n: int = 1000, seed: int = 101) -> Problem:
    rng = _rng(seed)
    inv_h2 = float((n + 1) ** 2)                 # exact integer h^-2
    x = np.arange(1, n + 1, dtype=np.float64) / (n + 1)
    u0 = np.sin(np.pi * x) + 0.01 * rng.standard_normal(n)
    u = [u0, _uniform(rng, n), _uniform(rng, n)]
    st = Stencil(1, n, 1, 1, (-2.0 * inv_h2, inv_h2, inv_h2, 0.0, 0.0, 0.0, 0.0))
    return Problem("c1", n, 2, 1e-3, 1e-10, True, u, stencil=st, seed=seed)


def c2(nx: int = 256, seed: int = 102) -> Problem:
    rng = _rng(seed)
    n = nx * nx
    inv_h2 = float((nx + 1) ** 2)
    u = [rng.standard_normal(n)] + [_uniform(rng, n) for _ in range(3)]
    st = Stencil(2, nx, nx, 1, (-4.0 * inv_h2, inv_h2, inv_h2, inv_h2, inv_h2, 0.0, 0.0))
    return Problem("c2", n, 3, 1e-4, 1e-10, True, u, stencil=st, seed=seed)


def c3(nx: int = 1024, seed: int = 103, eps: float = 1e-2, ax: float = 1.0, ay: float = 0.5) -> Problem:
    rng = _rng(seed)
    n = nx * nx
    h = 1.0 / (nx + 1)
    d = eps * float((nx + 1) ** 2)               # eps / h^2
    cx, cy = ax * (nx + 1), ay * (nx + 1)        # a / h
    coeffs = (-4.0 * d - (cx + cy), d + cx, d, d + cy, d, 0.0, 0.0)
    g = np.arange(1, nx + 1, dtype=np.float64) * h
    X, Y = np.meshgrid(g, g, indexing="xy")      # X varies along axis 1 -> x fastest in ravel
    bump = np.exp(-((X - 0.3) ** 2 + (Y - 0.3) ** 2) / (2 * 0.05 ** 2)).ravel()
    u0 = bump + 1e-3 * rng.standard_normal(n)
    u = [u0, _uniform(rng, n), _uniform(rng, n)]
    st = Stencil(2, nx, nx, 1, coeffs)
    return Problem("c3", n, 2, 1e-3, 1e-8, False, u, stencil=st, seed=seed)


def c4(nx: int = 128, seed: int = 104) -> Problem:
    rng = _rng(seed)
    n = nx ** 3
    inv_h2 = float((nx + 1) ** 2)
    u = [rng.standard_normal(n)] + [_uniform(rng, n) for _ in range(4)]
    st = Stencil(3, nx, nx, nx, (-6.0 * inv_h2,) + (inv_h2,) * 6)
    return Problem("c4", n, 4, 1e-5, 1e-10, True, u, stencil=st, seed=seed)


def random_banded_csr(rng: np.random.Generator, n: int, band: int, k_off: int = 15):
    """Row i: diagonal + k_off distinct columns i+o, o uniform over {1<=|o|<=band, 0<=i+o<n}."""
    if n - 1 < k_off or band < k_off:
        raise ValueError("band/n too small for k_off distinct off-diagonals")
    i = np.arange(n, dtype=np.int64)
    lo = np.minimum(i, band)                     # number of valid negative offsets
    hi = np.minimum(n - 1 - i, band)             # number of valid positive offsets
    L = lo + hi
    if np.any(L < k_off):
        raise ValueError("some row has fewer than k_off valid offsets")
    r = rng.integers(0, L[:, None], size=(n, k_off))
    r.sort(axis=1)
    bad = np.nonzero(np.any(r[:, 1:] == r[:, :-1], axis=1))[0]
    while bad.size:                              # redraw rows holding a duplicate, whole
        rr = rng.integers(0, L[bad][:, None], size=(bad.size, k_off))
        rr.sort(axis=1)
        r[bad] = rr
        still = np.any(rr[:, 1:] == rr[:, :-1], axis=1)
        bad = bad[still]
    off = np.where(r < lo[:, None], r - lo[:, None], r - lo[:, None] + 1)   # sorted, no 0
    vals = rng.standard_normal((n, k_off)) / 4.0
    # insert the diagonal at its sorted position
    npos = np.sum(off < 0, axis=1)               # offdiag entries left of the diagonal
    cols = np.empty((n, k_off + 1), dtype=np.int64)
    v = np.empty((n, k_off + 1), dtype=np.float64)
    idx = np.arange(k_off + 1)[None, :]
    left = idx < npos[:, None]
    right = idx > npos[:, None]
    src = np.where(left, idx, idx - 1)
    src = np.clip(src, 0, k_off - 1)
    cols[:] = np.take_along_axis(off, src, axis=1) + i[:, None]
    v[:] = np.take_along_axis(vals, src, axis=1)
    diag_mask = ~(left | right)
    cols[diag_mask] = i
    # diagonal = -(sum |a_ij|, j != i, ascending column order) - 1, summed sequentially
    absv = np.where(diag_mask, 0.0, np.abs(v))
    s = np.zeros(n)
    for c in range(k_off + 1):                   # sequential ascending-column sum
        s = s + absv[:, c]
    v[diag_mask] = -s - 1.0
    row_ptr = (np.arange(n + 1, dtype=np.int64) * (k_off + 1)).astype(np.int32)
    return row_ptr, cols.astype(np.int32).ravel(), np.ascontiguousarray(v.ravel())


def c5(n: int = 4_194_304, band: int = 4096, seed: int = 105) -> Problem:
    rng = _rng(seed)
    csr = random_banded_csr(rng, n, band)
    u = [rng.standard_normal(n)] + [_uniform(rng, n) for _ in range(3)]
    return Problem("c5", n, 3, 0.5, 1e-8, False, u, csr=csr, seed=seed)


# full-size BASELINE.json configs and scaled-down variants with the same structure
CONFIGS = {
    "c1": lambda: c1(),
    "c2": lambda: c2(),
    "c3": lambda: c3(),
    "c4": lambda: c4(),
    "c5": lambda: c5(),
    "c1_mini": lambda: c1(n=200),
    "c2_mini": lambda: c2(nx=24),
    "c3_mini": lambda: c3(nx=48),
    "c4_mini": lambda: c4(nx=12),
    "c5_mini": lambda: c5(n=6000, band=64),
    # "medium": several tiles and a ragged tail for the GPU kernels, still seconds for the oracle
    "c2_med": lambda: c2(nx=181),
    "c3_med": lambda: c3(nx=301),
    "c4_med": lambda: c4(nx=45),
    "c5_med": lambda: c5(n=300_007, band=1024),
    # 3-D Laplacian 70^3 (n = 343,000 >= 303,104): the tensor-memory Lanczos kernel at a size the
    # oracle still solves in seconds
    "c4_tm": lambda: c4(nx=70),
}


def make(name: str) -> Problem:
    return CONFIGS[name]()
