"""The cluster Lanczos kernel (csrc/persist_cl.cuh: Alg. 2, on one thread-block cluster with
the vectors in shared memory, DSMEM reductions and halo pushes) against the oracle.

Auto dispatch takes Lanczos extensions of stencils with 8192 < n <= 65536 (c2); the option
`cluster_lz` forces a cluster size (2/4/8/16) or a single CTA (-1) on other sizes.  The cases cover
every dimension class (1-D, 2-D 5-point, 2-D 9-point, 3-D with a plane-sized halo), ragged last CTAs,
relaunches with k0 > 0 (m grows inside an attempt sequence), a breakdown inside the kernel and
determinism.  Bars: H vs the oracle's Lanczos to 1e-9 ||A||_inf (test_gpu_kernels' Lanczos bar);
w: ||w_gpu - w_ref|| / ||w_ref|| <= max(10 tol, 1e-12) (BASELINE.json north_star).
"""
import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev

pytestmark = pytest.mark.gpu


def laplacian(orc, dim, nx, ny, nz, seed, p=2, ninept=False):
    """Dirichlet Laplacian (heat sign), h = 1/(nx+1) in every direction, or the 2-D 9-point one:
    (product stencil descriptor, oracle CSR built independently of the product, u_0..u_p)."""
    h2 = float((nx + 1) ** 2)
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    u = [rng.standard_normal(n)] + [rng.uniform(-1, 1, n) for _ in range(p)]
    if ninept:
        from test_gpu_ninept import csr_9pt
        coef, corn = (-8.0 * h2, h2, h2, h2, h2, 0.0, 0.0), (h2,) * 4
        return P.Stencil(2, nx, ny, 1, coef, corn, 9), csr_9pt(nx, ny, coef, corn), u
    coef = [-2.0 * dim * h2, h2, h2, 0.0, 0.0, 0.0, 0.0]
    if dim >= 2:
        coef[3] = coef[4] = h2
    if dim >= 3:
        coef[5] = coef[6] = h2
    st = W.Stencil(dim, nx, ny, nz, tuple(coef))
    return P.Stencil.of(st), orc.csr_from_stencil(st), u


# (dim, nx, ny, nz, ninept, cluster option)
KCASES = [
    (2, 256, 256, 1, False, 1),        # c2's operator, auto: 16 CTAs of 4096 rows
    (2, 181, 181, 1, False, 1),        # odd n = 32761: ragged last CTA
    (2, 150, 140, 1, True, 1),         # 9-point, halo nx + 1
    (3, 40, 40, 40, False, 1),         # 3-D: halo = one 1600-row plane
    (1, 20001, 1, 1, False, 1),        # 1-D, halo 1 row
    (2, 256, 256, 1, False, 2),        # forced cluster sizes
    (2, 256, 256, 1, False, 4),
    (2, 256, 256, 1, False, 8),
    (2, 40, 50, 1, False, -1),         # single CTA (n = 2000)
    (1, 1000, 1, 1, False, -1),        # c1-sized, single CTA
    (3, 12, 11, 10, False, 2),         # 3-D on 2 CTAs
]


@pytest.mark.parametrize("dim,nx,ny,nz,ninept,cl", KCASES)
def test_cluster_lanczos_vs_oracle(orc, dim, nx, ny, nz, ninept, cl):
    st, csr, u = laplacian(orc, dim, nx, ny, nz, seed=nx + ny + nz, ninept=ninept)
    n = nx * ny * nz
    m = 40
    Vo, Ho, ko, bo, beta_o = orc.krylov(csr, u[0], m, symmetric=True)
    ctx = P.Context(n_max=n, m_max=100, p_max=2, options={"cluster_lz": cl})
    V, H, k, brk, beta = ctx.krylov(st, to_dev(u[0]), m, symmetric=True)
    ctx.close()
    normA = orc.inf_norm(csr)
    assert k == ko == m and not brk
    assert beta == pytest.approx(beta_o, rel=1e-14)
    assert np.abs(H.cpu().numpy() - Ho).max() <= 1e-9 * normA
    # the Lanczos relation A V_m = V_{m+1} H holds for the GPU basis itself
    import scipy.sparse as sp
    Asp = sp.csr_matrix((csr[2], csr[1], csr[0]), shape=(n, n))
    Vg = V.cpu().numpy()
    Hg = H.cpu().numpy()
    assert np.abs(Asp @ Vg[:, :m] - Vg @ Hg).max() <= 1e-9 * normA


SCASES = [
    # (dim, nx, ny, nz, ninept, t, tol): t large enough that m grows past m_init (relaunch with k0 > 0)
    (2, 256, 256, 1, False, 1e-4, 1e-10),     # c2
    (2, 181, 181, 1, False, 3e-4, 1e-10),
    (2, 150, 140, 1, True, 2e-5, 1e-10),
    (3, 40, 40, 40, False, 1e-3, 1e-10),
    (1, 20001, 1, 1, False, 3e-8, 1e-10),
]


@pytest.mark.parametrize("dim,nx,ny,nz,ninept,t,tol", SCASES)
def test_cluster_solve_parity(orc, dim, nx, ny, nz, ninept, t, tol):
    st, csr, u = laplacian(orc, dim, nx, ny, nz, seed=3 * nx + nz, ninept=ninept)
    wo, so, _ = orc.phipm(t, csr, u, tol, m_init=10, m_max=100, symmetric=True)
    assert so["status"] == 0
    ctx = P.Context(n_max=nx * ny * nz, m_max=100, p_max=4)
    assert ctx.get_option("cluster_lz") == 1
    w, s = ctx.solve_stencil(t, st, [to_dev(x) for x in u], tol=tol, symmetric=True)
    ctx.close()
    assert s.t_reached == t
    assert s.m_peak > 10, s
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol), (s, so)


@pytest.mark.parametrize("modes", [1, 2])
def test_cluster_breakdown(orc, modes):
    # u_0 = a combination of `modes` separable sines (eigenvectors of the 2-D Dirichlet Laplacian): the
    # Krylov space closes at j = modes and the kernel stops at the breakdown (R22) with the halo of
    # v~_{j+1} pushed; the solve must finish (no CTA may exit with a push outstanding) and match the oracle
    nx, ny = 200, 180
    st, csr, _ = laplacian(orc, 2, nx, ny, 1, seed=0)
    n = nx * ny
    gx = np.arange(1, nx + 1) / (nx + 1)
    gy = np.arange(1, ny + 1) / (ny + 1)
    v = np.zeros(n)
    for k in range(1, modes + 1):
        v += 1.0 / k * np.outer(np.sin(k * np.pi * gy), np.sin((k + 2) * np.pi * gx)).ravel()
    t, tol = 1e-4, 1e-10
    wo, so, _ = orc.phipm(t, csr, [v], tol, m_init=10, m_max=100, symmetric=True)
    assert so["status"] == 0
    ctx = P.Context(n_max=n, m_max=100, p_max=2)
    w, s = ctx.solve_stencil(t, st, [to_dev(v)], tol=tol, symmetric=True)
    # and a second solve on the same context (the cluster kernel left no state behind)
    w2, s2 = ctx.solve_stencil(t, st, [to_dev(v)], tol=tol, symmetric=True)
    ctx.close()
    assert s.t_reached == t
    assert s.nspmv <= modes * s.nexpm, s
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(tol), (s, so)
    assert np.array_equal(w.cpu().numpy(), w2.cpu().numpy())


def test_cluster_deterministic_and_matches_grid_kernel():
    # c2 twice with the cluster kernel (bit-identical: fixed reduction order) and once with the grid-wide
    # persistent kernel (cluster_lz = 0): the two differ only in the order of the dot / norm sums
    Pb = W.make("c2")
    u = [to_dev(x) for x in Pb.u]
    S = P.Stencil.of(Pb.stencil)
    res = {}
    for cl in (1, 0):
        ctx = P.Context(n_max=Pb.n, m_max=100, p_max=4, options={"cluster_lz": cl})
        w, s = ctx.solve_stencil(Pb.t, S, u, tol=Pb.tol, symmetric=True)
        if cl:
            w2, _ = ctx.solve_stencil(Pb.t, S, u, tol=Pb.tol, symmetric=True)
            assert np.array_equal(w.cpu().numpy(), w2.cpu().numpy())
        res[cl] = (w.cpu().numpy(), s)
        ctx.close()
    assert relerr(res[1][0], res[0][0]) <= 1e-11, (res[1][1], res[0][1])


@pytest.mark.parametrize("name", ["c1", "c2", "c2_med", "c3_mini", "c5_mini"])
def test_speculative_extension_changes_nothing(name):
    # option spec (default on): the extension to min((4m+2)/3, m_max) runs on a second stream during the
    # exponential.  It splits the basis at the same columns as the unspeculated solve (each m-branch
    # rejection asks for exactly that extension), adds columns beyond m only, and the exponential ignores
    # a breakdown beyond m: w is bit-identical and the stats (the algorithm's SpMV count) are equal
    Pb = W.make(name)
    u = [to_dev(x) for x in Pb.u]
    res = {}
    for spec in (1, 0):
        ctx = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1), options={"spec": spec})
        if Pb.stencil is not None:
            w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric)
        else:
            A = tuple(to_dev(a) for a in Pb.csr)
            w, s = ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric)
        res[spec] = (w.cpu().numpy(), s)
        ctx.close()
    assert np.array_equal(res[1][0], res[0][0])
    assert res[1][1] == res[0][1]


@pytest.mark.parametrize("name", ["c1", "c1_mini", "c2_mini"])
def test_device_solve_matches_host_solve(orc, name):
    # option devsolve (default on): a symmetric problem with n <= 8192 runs as ONE kernel that also
    # executes the controller (solve_small.cuh).  Against the host-driven path on the same inputs: the
    # same trajectory where the two agree to rounding (the first step's attempts; the dot / norm sums
    # are reduced in another order), the solution within the parity bar of both and of the oracle, and
    # the attempt records of the device solve are the ones of that solve (not a stale earlier one)
    Pb = W.make(name)
    u = [to_dev(x) for x in Pb.u]
    out = {}
    for dev in (1, 0):
        ctx = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1), options={"devsolve": dev})
        w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=True)
        out[dev] = (w.cpu().numpy(), s, ctx.attempts())
        ctx.close()
    wo, so, tr = orc.solve(Pb)
    (wd, sd, ad), (wh, sh, ah) = out[1], out[0]
    assert len(ad) == sd.nexpm and len(ah) == sh.nexpm
    first = next(i for i, a in enumerate(ah) if a["accepted"]) + 1
    for a, b in zip(ad[:first], ah[:first]):
        assert (a["m"], a["mu"], a["accepted"], a["branch"]) == (b["m"], b["mu"], b["accepted"], b["branch"])
        assert a["tau"] == pytest.approx(b["tau"], rel=1e-9)
        assert a["beta"] == pytest.approx(b["beta"], rel=1e-10)
    assert sd.t_reached == Pb.t and abs(sd.nsteps - sh.nsteps) <= 2
    assert relerr(wd, wo) <= parity_bound(Pb.tol)
    assert relerr(wd, wh) <= parity_bound(Pb.tol)
    # a following host-path solve on the same context reports its own attempts
    ctx = P.Context(n_max=max(Pb.n, 65536), m_max=100, p_max=4)
    ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=True)
    Q = W.make("c2")
    ctx.solve_stencil(Q.t, P.Stencil.of(Q.stencil), [to_dev(x) for x in Q.u], tol=Q.tol, symmetric=True)
    aq = ctx.attempts()
    ctx.close()
    assert aq[0]["m"] == Q.m_init and len(aq) == 6


def test_device_solve_degenerate():
    # zero input (w = 0), A = 0 (tau = t), a breakdown at the seed: the device solve's special paths
    Pb = W.make("c1_mini")
    S = P.Stencil.of(Pb.stencil)
    ctx = P.Context(n_max=Pb.n, m_max=100, p_max=4)
    z = [to_dev(np.zeros(Pb.n)) for _ in Pb.u]
    w, s = ctx.solve_stencil(Pb.t, S, z, tol=Pb.tol, symmetric=True)
    assert float(w.abs().max()) == 0.0 and s.t_reached == Pb.t
    S0 = P.Stencil(S.dim, S.nx, S.ny, S.nz, (0.0,) * 7)
    u = [to_dev(x) for x in Pb.u]
    w, s = ctx.solve_stencil(Pb.t, S0, u, tol=Pb.tol, symmetric=True)
    # A = 0: w = u_0 + sum_k t^k/k! u_k exactly up to rounding
    import math
    ref = sum(Pb.t ** k / math.factorial(k) * Pb.u[k] for k in range(len(Pb.u)))
    assert relerr(w.cpu().numpy(), ref) <= 1e-14
    ctx.close()
