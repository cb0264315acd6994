"""The persistent Lanczos kernel with y / v~_j in tensor memory (csrc/persist_tm.cuh) and the persistent
w-recurrence (csrc/persist_wrec.cuh) against the oracle.

The host dispatches Lanczos extensions on stencils to it when n >= 4096 * 148 / 2 = 303,104 rows (a
4096-row tile per half CTA at least) and every CTA's range fits 4 tiles of 4096 rows.  The cases
cover every dimension class (1-D, 2-D 5-point, 2-D 9-point, 3-D), even nx (the fast pair path of
the stencil rows) and odd nx (the per-term path inside the same kernel), ragged last tiles, and
t large enough that attempts are rejected and m grows, so the kernel is relaunched with k0 > 0
(its first step then reads v~_{j-1} from global memory, the later ones from TMEM slot B).
Bar: ||w_gpu - w_ref|| / ||w_ref|| <= max(10 tol, 1e-12) (BASELINE.json north_star).
"""
import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev

pytestmark = pytest.mark.gpu


def laplacian(dim, nx, ny, nz, seed, p=2):
    """Dirichlet Laplacian (heat sign) on an nx x ny x nz grid, h = 1/(nx+1) in every direction."""
    h2 = float((nx + 1) ** 2)
    coef = [-2.0 * dim * h2, h2, h2, 0.0, 0.0, 0.0, 0.0]
    if dim >= 2:
        coef[3] = coef[4] = h2
    if dim >= 3:
        coef[5] = coef[6] = h2
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    u = [rng.standard_normal(n)] + [rng.uniform(-1, 1, n) for _ in range(p)]
    return W.Stencil(dim, nx, ny, nz, tuple(coef)), u


CASES = [
    # (dim, nx, ny, nz, t, tol): t chosen so that m has to grow past m_init = 10
    (3, 72, 70, 68, 2e-4, 1e-10),      # even nx: fast pair path, 3 of 4 tiles in the last CTA ragged
    (3, 71, 70, 69, 2e-4, 1e-10),      # odd nx: per-term rows inside the TMEM kernel
    (2, 640, 500, 1, 2e-5, 1e-10),     # 2-D 5-point
    (1, 400_001, 1, 1, 1e-11, 1e-10),  # 1-D, odd n
]


@pytest.mark.parametrize("dim,nx,ny,nz,t,tol", CASES)
def test_tmem_lanczos_parity(ctx, orc, dim, nx, ny, nz, t, tol):
    st, u = laplacian(dim, nx, ny, nz, seed=nx + ny + nz)
    n = st.n
    assert n >= 303_104
    Pb = W.Problem(name="tm", n=n, p=len(u) - 1, t=t, tol=tol, symmetric=True, u=u, stencil=st, seed=0)
    wo, so, _ = orc.solve(Pb)
    assert so["status"] == 0
    w, s = ctx.solve_stencil(t, P.Stencil.of(st), [to_dev(x) for x in u], tol=tol, symmetric=True)
    assert s.t_reached == t
    assert s.m_peak > 10, s                         # the extension was relaunched with k0 > 0
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol), (s, so)


def test_tmem_lanczos_9pt(ctx, orc):
    # 2-D 9-point Laplacian (DIM class 4 of the kernel), h^-2 (8 on the diagonal, 1 off it)
    from test_gpu_ninept import csr_9pt
    nx, ny = 620, 500
    h2 = float((nx + 1) ** 2)
    coef = (-8.0 * h2, h2, h2, h2, h2, 0.0, 0.0)
    corn = (h2,) * 4
    rng = np.random.default_rng(7)
    n = nx * ny
    u = [rng.standard_normal(n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    t, tol = 1e-5, 1e-10
    wo, so, _ = orc.phipm(t, csr_9pt(nx, ny, coef, corn), u, tol, m_init=10, m_max=100, symmetric=True)
    assert so["status"] == 0
    w, s = ctx.solve_stencil(t, P.Stencil(2, nx, ny, 1, coef, corn, 9), [to_dev(x) for x in u], tol=tol,
                             symmetric=True)
    assert s.t_reached == t
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol), (s, so)


@pytest.mark.parametrize("var", ["tmem", "wrec"])
def test_persistent_variants_agree(var):
    # c4 with the default kernels and with one persistent variant switched off (context option):
    #   tmem = 0: the Lanczos kernel keeps y in shared memory instead of tensor memory;
    #   wrec = 0: the w-recurrence runs as p streaming launches instead of one cooperative kernel.
    # Each pair differs only in the order some sums are reduced, so w agrees far below the parity bar
    Pb = W.make("c4")
    u = [to_dev(x) for x in Pb.u]
    out = {}
    for flag in (1, 0):
        c = P.Context(n_max=Pb.n, m_max=100, p_max=4, options={var: flag})
        w, s = c.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=True)
        out[flag] = w.cpu().numpy()
        c.close()
    assert relerr(out[1], out[0]) <= 1e-12


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5, 6])
def test_wrec_persistent_all_p_multistep(orc, p):
    # 2-D Laplacian 181^2 (n > 8192: the cooperative w-recurrence), t = 5e-4: two steps, so every u-term of
    # Eq. (wrecurrence) has a nonzero t_k^l / l! on the second.  Eq. (step) sums terms of size
    # ||tau A||^j ||u|| that cancel to O(||u||), so the accuracy any implementation reaches degrades with p
    # (the oracle vs the exact DST solution: 1e-14 at p = 0, 6e-12 at p = 3, 4e-8 at p = 6): up to p = 4
    # the GPU meets the BASELINE bar against the oracle; for p = 5, 6 both are held to the exact solution,
    # the GPU within 10x the oracle's own error
    import torch
    import exact as X
    st, u = laplacian(2, 181, 181, 1, seed=900 + p, p=p)
    Pb = W.Problem(name="wr", n=st.n, p=p, t=5e-4, tol=1e-9, symmetric=True, u=u, stencil=st, seed=0)
    wo, so, _ = orc.solve(Pb)
    assert so["status"] == 0
    ctx6 = P.Context(n_max=st.n, m_max=100, p_max=6)
    w, s = ctx6.solve_stencil(Pb.t, P.Stencil.of(st), [to_dev(x) for x in u], tol=Pb.tol, symmetric=True)
    assert s.t_reached == Pb.t and s.nsteps > 1, s
    wg = w.cpu().numpy()
    if p <= 4:
        assert relerr(wg, wo) <= parity_bound(Pb.tol), (s, so)
    else:
        ref = X.dst_solution(st, u, Pb.t)
        assert relerr(wg, ref) <= 10 * max(relerr(wo, ref), parity_bound(Pb.tol)), (s, so)
    torch.cuda.synchronize()


@pytest.mark.parametrize("modes,p", [(1, 0), (2, 0), (3, 0)])
def test_tmem_lanczos_breakdown(ctx, orc, modes, p):
    # u_0 = a combination of `modes` eigenvectors (separable sines) of the 3-D Dirichlet Laplacian: the
    # Krylov space is that invariant subspace, so Lanczos breaks down at j = modes inside the TMEM kernel
    # (h_{j+1,j} <= n eps ||A||, R22); the step's pre-issued halo tiles are drained before the CTAs exit.
    # (p > 0 would apply A^p to the sines' ~1e-14 rounding, high-frequency and amplified by ||A||^p, and
    # the space no longer closes at j = modes.)
    nx, ny, nz = 72, 70, 68
    st, _ = laplacian(3, nx, ny, nz, seed=0)
    gx = np.arange(1, nx + 1) / (nx + 1)
    gy = np.arange(1, ny + 1) / (ny + 1)
    gz = np.arange(1, nz + 1) / (nz + 1)

    def mode(k):
        return np.einsum("k,j,i->kji", np.sin(k * np.pi * gz), np.sin((k + 1) * np.pi * gy),
                         np.sin((k + 2) * np.pi * gx)).ravel()

    u = []
    for i in range(p + 1):
        v = np.zeros(st.n)
        for k in range(1, modes + 1):
            v += (1.0 + 0.5 * i) / k * mode(k)
        u.append(v)
    Pb = W.Problem(name="bd", n=st.n, p=p, t=1e-4, tol=1e-10, symmetric=True, u=u, stencil=st, seed=0)
    wo, so, _ = orc.solve(Pb)
    assert so["status"] == 0
    w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(st), [to_dev(x) for x in u], tol=Pb.tol, symmetric=True)
    assert s.t_reached == Pb.t
    assert s.nspmv - p * s.nsteps <= modes * s.nexpm, s    # the basis never grew past the invariant subspace
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(Pb.tol), (s, so)


def test_u0_in_place_and_copied_agree(ctx):
    # the first step reads u_0 in place when n is even and u_0 is 16-B aligned, otherwise from a workspace
    # copy; both run the same arithmetic, so w is bit-identical (also with w aliasing u_0)
    import torch
    Pb = W.make("c3_med")                                  # n = 301^2 odd: always the copy
    Pb2 = W.make("c4")                                     # n even
    for Q in (Pb, Pb2):
        u = [to_dev(x) for x in Q.u]
        S = P.Stencil.of(Q.stencil)
        w1, s1 = ctx.solve_stencil(Q.t, S, u, tol=Q.tol, symmetric=Q.symmetric)
        big = torch.zeros(Q.n + 1, dtype=torch.float64, device="cuda")
        big[1:] = u[0]
        u_mis = [big[1:]] + u[1:]                          # 8-B aligned view: the copy path
        w2, s2 = ctx.solve_stencil(Q.t, S, u_mis, tol=Q.tol, symmetric=Q.symmetric)
        assert torch.equal(w1, w2) and s1.nspmv == s2.nspmv
        u_alias = [u[0].clone()] + u[1:]
        w3, s3 = ctx.solve_stencil(Q.t, S, u_alias, out=u_alias[0], tol=Q.tol, symmetric=Q.symmetric)
        assert w3.data_ptr() == u_alias[0].data_ptr() and torch.equal(w1, w3)
