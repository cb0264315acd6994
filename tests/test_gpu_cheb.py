"""NEXT-2: phi-functions of the symmetric Lanczos matrix computed directly (csrc/phicheb.cuh,
PHIPM_EXPM_CHEBYSHEV) against the oracle's augmented Pade-13
exponential (orc_phi_pair), and full Lanczos solves with that method against the oracle.

Kernel bar: ||phi_gpu - phi_ref||_inf <= 1e-12 max(1, ||phi_k(tau T)||_2): both methods are backward
stable, so their difference scales with the norm of the matrix function (e.g. e^{20} for a T with an
eigenvalue at 20, even when e1 barely touches that eigenvector), not with the entries of the result.
On symmetric tridiagonal T from random draws and from actual Lanczos runs, at
K = mu + p + 1 from 2 to 105 and tau ||T|| from 1e-3 to beyond the 512-point limit (which falls
back to the augmented exponential)."""
import math

import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev, stencil_of

pytestmark = pytest.mark.gpu


@pytest.fixture
def cheb(ctx):
    ctx.set_expm_method(P.EXPM_CHEBYSHEV)
    yield ctx
    ctx.set_expm_method(P.EXPM_TAYLOR)


def tridiag(mu, seed, center, spread):
    rng = np.random.default_rng(seed)
    a = center + spread * rng.uniform(-1, 1, mu)
    b = spread * 0.5 * np.abs(rng.standard_normal(mu - 1)) + 1e-3 * spread
    return np.diag(a) + np.diag(b, 1) + np.diag(b, -1)


def tridiag_nsd(mu, seed, width):
    """Negative semidefinite symmetric tridiagonal with spectrum in [-width, 0] (the heat configs'
    Lanczos matrices): a random tridiagonal shifted by its largest eigenvalue and scaled."""
    T = tridiag(mu, seed, 0.0, 1.0)
    ev = np.linalg.eigvalsh(T)
    T = T - ev.max() * np.eye(mu)
    return T * (width / max(ev.max() - ev.min(), 1e-300))


def phi_norm(T, tau, k):
    """||phi_k(tau T)||_2 = max_i phi_k(tau lambda_i) (phi_k > 0 and increasing on the real line)."""
    z = tau * np.linalg.eigvalsh(T).max()
    if abs(z) < 1e-8:
        return 1.0 / math.factorial(k)
    f = math.exp(z)
    for j in range(k):
        f = (f - 1.0 / math.factorial(j)) / z
    return abs(f)


def check_pair(ctx, orc, T, tau, p):
    import torch
    a, b, nh = ctx.phi_pair(torch.from_numpy(T).cuda(), tau, p)
    ra, rb, rnh = orc.phi_pair(T, tau, p)
    a, b = a.cpu().numpy(), b.cpu().numpy()
    assert np.abs(a - ra).max() <= 1e-12 * max(1.0, phi_norm(T, tau, p)), np.abs(a - ra).max()
    assert np.abs(b - rb).max() <= 1e-12 * max(1.0, phi_norm(T, tau, p + 1)), np.abs(b - rb).max()
    assert nh == pytest.approx(rnh, rel=1e-15)


@pytest.mark.parametrize("mu", [1, 2, 9, 14, 40, 64, 100])
@pytest.mark.parametrize("p", [0, 1, 2, 4])
@pytest.mark.parametrize("width", [1e-3, 1.0, 30.0, 300.0, 3000.0])
def test_phi_pair_cheb_random(cheb, orc, mu, p, width):
    # negative semidefinite like the heat configs' Lanczos T: spectrum in [-width, 0]
    T = tridiag_nsd(mu, seed=mu * 7 + p, width=width) if mu > 1 else np.array([[-width]])
    check_pair(cheb, orc, T, 1.0, p)


@pytest.mark.parametrize("center", [-5.0, 0.0, 5.0])
def test_phi_pair_cheb_indefinite_and_positive(cheb, orc, center):
    # the round-trip forward leg has a positive spectrum (e^{tA}, A > 0); indefinite T as well
    T = tridiag(30, seed=3, center=center, spread=4.0)
    for p in (0, 1, 3):
        check_pair(cheb, orc, T, 1.0, p)


def test_phi_pair_cheb_closed_forms(cheb):
    import torch
    for z in (-30.0, -3.0, -1.0, -1e-6, 0.0, 1e-6, 1.0, 3.0):
        a, b, _ = cheb.phi_pair(torch.tensor([[z]], dtype=torch.float64, device="cuda"), 1.0, 1)
        p1 = math.expm1(z) / z if z != 0 else 1.0
        p2 = (math.expm1(z) - z) / z ** 2 if abs(z) > 1e-3 else 0.5 + z / 6 + z * z / 24
        assert float(a[0]) == pytest.approx(p1, rel=1e-13, abs=1e-16)
        assert float(b[0]) == pytest.approx(p2, rel=1e-12, abs=1e-16)


def test_phi_pair_cheb_wide_interval_falls_back(cheb, orc):
    # spectrum [-8000, 0]: half-width 4000, 9.5 sqrt(r) + 24 > 512 points -> the augmented Taylor
    # exponential (the kernel publishes status 7 and the host reruns the attempt)
    T = tridiag_nsd(20, seed=5, width=8000.0)
    check_pair(cheb, orc, T, 1.0, 2)


@pytest.mark.parametrize("name", ["c1_mini", "c2_mini", "c4_mini", "c2_med"])
def test_phi_pair_cheb_lanczos_T(cheb, orc, name):
    # T from an actual Lanczos run (the matrices the solve exponentiates), tau of the first step
    Pb = W.make(name)
    csr = orc.operator_csr(Pb)
    V, H, k, brk, beta = orc.krylov(csr, Pb.u[-1], 40 if Pb.n > 40 else Pb.n - 1, symmetric=True)
    T = H[:k, :k]
    T = np.triu(np.tril(T, 1), -1)
    T = 0.5 * (T + T.T)
    for tau in (Pb.t, Pb.t / 10, Pb.t / 300):
        check_pair(cheb, orc, T, tau, Pb.p)


CASES = [("c1_mini", "stencil"), ("c1", "stencil"), ("c1", "csr"), ("c2_mini", "stencil"), ("c2", "stencil"),
         ("c2", "csr"), ("c4_mini", "stencil"), ("c4_med", "stencil"), ("c4", "stencil")]


@pytest.mark.parametrize("name,path", CASES)
def test_solve_cheb_vs_oracle(ctx, orc, name, path):
    """Lanczos solves with the Chebyshev phi-functions against the oracle (augmented Pade-13)."""
    Pb = W.make(name)
    u = [to_dev(x) for x in Pb.u]
    kw = dict(tol=Pb.tol, symmetric=True, m_init=Pb.m_init, expm_method=P.EXPM_CHEBYSHEV)
    if path == "stencil":
        w, s = ctx.solve_stencil(Pb.t, stencil_of(Pb), u, **kw)
    else:
        A = ctx.csr_from_stencil(stencil_of(Pb))
        w, s = ctx.solve_csr(Pb.t, A, u, **kw)
    wo, so, _ = orc.solve(Pb)
    assert s.t_reached == Pb.t
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(Pb.tol), (s, so)


def test_solve_cheb_arnoldi_uses_taylor(ctx):
    # Arnoldi H is not symmetric: the method applies to Lanczos only, Arnoldi solves are unchanged
    Pb = W.make("c3_mini")
    u = [to_dev(x) for x in Pb.u]
    a, sa = ctx.solve_stencil(Pb.t, stencil_of(Pb), u, tol=Pb.tol, expm_method=P.EXPM_CHEBYSHEV)
    b, sb = ctx.solve_stencil(Pb.t, stencil_of(Pb), u, tol=Pb.tol, expm_method=P.EXPM_TAYLOR)
    assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())
