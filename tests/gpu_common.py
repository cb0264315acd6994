"""Shared helpers for the -m gpu parity tests (product through the C ABI vs the oracle)."""
import numpy as np

import workloads as W


def to_dev(x, dtype=None):
    import torch
    a = np.ascontiguousarray(x)
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def stencil_of(problem):
    import paper_0907_4631_b200 as P
    return P.Stencil.of(problem.stencil)


def parity_bound(tol):
    """BASELINE.json north_star: ||w_gpu - w_ref||_2 / ||w_ref||_2 <= max(10 tol, 1e-12)."""
    return max(10 * tol, 1e-12)


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))
