"""Full phipm parity: the CUDA path (through the C ABI) vs the oracle on the same seeded inputs.

Bar (BASELINE.json north_star): ||w_gpu - w_ref||_2 / ||w_ref||_2 <= max(10 tol, 1e-12).  Only w
is compared; the controller's trajectory may legitimately differ when rounding flips a decision
near a threshold (parity unpinned), so stats are reported, not asserted equal.
"""
import numpy as np
import pytest

import workloads as W
from gpu_common import to_dev, stencil_of, parity_bound, relerr

pytestmark = pytest.mark.gpu


def run_gpu(ctx, Pb, path, **kw):
    u = [to_dev(x) for x in Pb.u]
    kw.setdefault("tol", Pb.tol)
    kw.setdefault("symmetric", Pb.symmetric)
    kw.setdefault("m_init", Pb.m_init)
    if path == "stencil":
        w, s = ctx.solve_stencil(Pb.t, stencil_of(Pb), u, **kw)
    else:
        if Pb.csr is not None:
            A = tuple(to_dev(a) for a in Pb.csr)
        else:
            A = ctx.csr_from_stencil(stencil_of(Pb))     # the product's own CSR builder
        w, s = ctx.solve_csr(Pb.t, A, u, **kw)
    return w.cpu().numpy(), s


def run_oracle(orc, Pb, **kw):
    w, s, _ = orc.solve(Pb, **kw)
    assert s["status"] == 0
    return w, s


CASES = [
    ("c1_mini", "csr"), ("c1_mini", "stencil"),
    ("c2_mini", "stencil"), ("c2_mini", "csr"),
    ("c3_mini", "stencil"), ("c3_mini", "csr"),
    ("c4_mini", "stencil"),
    ("c5_mini", "csr"),
    ("c2_med", "stencil"), ("c3_med", "stencil"), ("c4_med", "stencil"), ("c5_med", "csr"),
]


@pytest.mark.parametrize("name,path", CASES)
def test_solve_parity_small(ctx, orc, name, path):
    Pb = W.make(name)
    wg, sg = run_gpu(ctx, Pb, path)
    wo, so = run_oracle(orc, Pb)
    assert sg.t_reached == Pb.t
    assert relerr(wg, wo) <= parity_bound(Pb.tol), (sg, so)


@pytest.mark.parametrize("name,path", [("c1_mini", "stencil"), ("c3_mini", "stencil"), ("c5_mini", "csr"),
                                       ("c1", "csr"), ("c3_med", "stencil"), ("c5_med", "csr")])
def test_solve_parity_pade13(ctx, orc, name, path):
    # the paper's expm (Pade-13 + pivoted solve) on the GPU: same parity bar as the default Taylor
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    wg, sg = run_gpu(ctx, Pb, path, expm_method=P.EXPM_PADE13)
    wo, so = run_oracle(orc, Pb)
    assert sg.t_reached == Pb.t
    assert relerr(wg, wo) <= parity_bound(Pb.tol), (sg, so)


FULL = [("c1", "csr"), ("c1", "stencil"), ("c2", "csr"), ("c2", "stencil"), ("c3", "stencil"),
        ("c4", "stencil"), ("c5", "csr")]


@pytest.mark.parametrize("name,path", FULL)
def test_solve_parity_full_configs(ctx, orc, name, path):
    """BASELINE.json configs at full size, in the launch configuration bench.py times."""
    Pb = W.make(name)
    wg, sg = run_gpu(ctx, Pb, path)
    wo, so = run_oracle(orc, Pb)
    err = relerr(wg, wo)
    print(f"{name}/{path}: relerr {err:.3e} gpu {sg} oracle {so}")
    assert err <= parity_bound(Pb.tol)


def test_csr_and_stencil_agree(ctx):
    Pb = W.make("c2_med")
    a, sa = run_gpu(ctx, Pb, "stencil")
    b, sb = run_gpu(ctx, Pb, "csr")
    assert relerr(a, b) <= parity_bound(Pb.tol)


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5])
def test_all_p(ctx, orc, p):
    rng = np.random.default_rng(50 + p)
    Pb = W.c5(n=20_011, band=128, seed=300 + p)
    Pb.u = [rng.standard_normal(Pb.n) for _ in range(p + 1)]
    Pb.p = p
    Pb.t = 0.7
    wg, sg = run_gpu(ctx, Pb, "csr")
    wo, so = run_oracle(orc, Pb)
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


def test_multistep_stiff(ctx, orc):
    Pb = W.make("c1")            # t ||A|| = 4008: ~15-30 steps with rejections
    wg, sg = run_gpu(ctx, Pb, "stencil")
    wo, so = run_oracle(orc, Pb)
    assert sg.nsteps > 5
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


def test_cgs2_and_fixed_m(ctx, orc):
    Pb = W.make("c3_med")
    wo, so = run_oracle(orc, Pb)
    wg, sg = run_gpu(ctx, Pb, "stencil", orth=1)
    assert relerr(wg, wo) <= parity_bound(Pb.tol)
    Pb = W.make("c1_mini")
    wo, so = run_oracle(orc, Pb, m_init=30, fixed_m=True)
    wg, sg = run_gpu(ctx, Pb, "csr", m_init=30, fixed_m=True)
    assert sg.m_peak == 30 and sg.m_last == 30
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


@pytest.mark.parametrize("name,path", [("c2_med", "stencil"), ("c3_med", "stencil"), ("c4_med", "stencil"),
                                       ("c5_med", "csr"), ("c1", "csr")])
def test_fixed_m_phip_parity(ctx, orc, name, path):
    # NEXT-1: the paper's phip mode (m fixed, only tau adapts) vs the oracle in the same mode
    Pb = W.make(name)
    wo, so = run_oracle(orc, Pb, m_init=30, fixed_m=True)
    wg, sg = run_gpu(ctx, Pb, path, m_init=30, fixed_m=True)
    assert sg.t_reached == Pb.t
    assert sg.m_peak <= 30
    assert relerr(wg, wo) <= parity_bound(Pb.tol), (sg, so)


def test_eq6_variant(ctx, orc):
    Pb = W.make("c1")
    wo, so = run_oracle(orc, Pb, eq6_variant=True)
    wg, sg = run_gpu(ctx, Pb, "stencil", eq6_variant=True)
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


def test_degenerate_inputs(ctx, orc):
    import torch
    Pb = W.make("c2_mini")
    S = stencil_of(Pb)
    u = [to_dev(x) for x in Pb.u]
    # t = 0 -> u0
    w, s = ctx.solve_stencil(0.0, S, u, tol=1e-8, symmetric=True)
    assert np.array_equal(w.cpu().numpy(), Pb.u[0])
    # all zero -> 0
    z = [torch.zeros_like(x) for x in u]
    w, s = ctx.solve_stencil(Pb.t, S, z, tol=1e-8, symmetric=True)
    assert torch.count_nonzero(w).item() == 0
    # w_p = 0 with u0 != 0 (R23)
    u2 = [u[0], torch.zeros_like(u[0])]
    w, s = ctx.solve_stencil(Pb.t, S, u2, tol=1e-10, symmetric=True)
    wo, so, _ = orc.phipm(Pb.t, orc.operator_csr(Pb), [Pb.u[0], np.zeros(Pb.n)], 1e-10, symmetric=True)
    assert relerr(w.cpu().numpy(), wo) <= 1e-9
    # w may alias u0
    uu = [x.clone() for x in u]
    w, s = ctx.solve_stencil(Pb.t, S, uu, out=uu[0], tol=Pb.tol, symmetric=True)
    wo, so = run_oracle(orc, Pb)
    assert relerr(uu[0].cpu().numpy(), wo) <= parity_bound(Pb.tol)
    # bad arguments -> EINVAL, no crash
    import paper_0907_4631_b200 as P
    with pytest.raises(P.PhipmError) as e:
        ctx.solve_stencil(-1.0, S, u, tol=1e-8)
    assert e.value.status == P.EINVAL
    with pytest.raises(P.PhipmError):
        ctx.solve_stencil(Pb.t, S, u, tol=0.0)
    with pytest.raises(P.PhipmError):
        ctx.solve_stencil(Pb.t, S, u, m_init=0)


def test_a_zero_and_tiny_n(ctx, orc):
    import torch
    # A = 0 (empty CSR): w = sum t^k/k! u_k exactly (phi_l(0) = 1/l!)
    n = 7
    rng = np.random.default_rng(1)
    uu = [rng.standard_normal(n) for _ in range(3)]
    A = (to_dev(np.zeros(n + 1, np.int32)), torch.zeros(0, dtype=torch.int32, device="cuda"),
         torch.zeros(0, dtype=torch.float64, device="cuda"))
    w, s = ctx.solve_csr(1.7, A, [to_dev(x) for x in uu], tol=1e-10)
    ref = uu[0] + 1.7 * uu[1] + 1.7 ** 2 / 2 * uu[2]
    assert np.allclose(w.cpu().numpy(), ref, rtol=1e-15, atol=1e-15)
    # n = 1 and n < m (breakdown inside the Krylov space)
    for n in (1, 5, 33):
        Pb = W.c5(n=max(n, 40), band=16, seed=11) if n >= 40 else None
        Dg = -np.abs(rng.standard_normal(n)) - 0.5
        rp = np.arange(n + 1, dtype=np.int32)
        col = np.arange(n, dtype=np.int32)
        u3 = [rng.standard_normal(n) for _ in range(2)]
        wg, sg = ctx.solve_csr(0.9, (to_dev(rp), to_dev(col), to_dev(Dg)), [to_dev(x) for x in u3], tol=1e-10)
        wo, so, _ = orc.phipm(0.9, (rp, col, Dg), u3, 1e-10)
        assert relerr(wg.cpu().numpy(), wo) <= 1e-9


def test_host_buffers_match_device(ctx):
    Pb = W.make("c3_mini")
    wd, sd = run_gpu(ctx, Pb, "stencil")
    out = np.empty(Pb.n)
    wh, sh = ctx.solve_stencil_host(Pb.t, stencil_of(Pb), Pb.u, out, tol=Pb.tol, symmetric=Pb.symmetric)
    assert np.array_equal(wd, wh)
    Pb = W.make("c5_mini")
    wd, sd = run_gpu(ctx, Pb, "csr")
    out = np.empty(Pb.n)
    wh, sh = ctx.solve_csr_host(Pb.t, Pb.csr, Pb.u, out, tol=Pb.tol, symmetric=False)
    assert np.array_equal(wd, wh)


def test_deterministic(ctx):
    Pb = W.make("c5_med")
    a, sa = run_gpu(ctx, Pb, "csr")
    b, sb = run_gpu(ctx, Pb, "csr")
    assert np.array_equal(a, b) and sa == sb


def test_profile_counts(ctx):
    Pb = W.make("c3_med")
    ctx.reset_profile()
    w, s = run_gpu(ctx, Pb, "stencil", profile=True)
    prof = ctx.profile()
    assert prof["n_expm"] == s.nexpm
    # launches of the SpMV class: one per product (two-kernel path) or one per Krylov extension
    # plus the w-recurrence products (persistent kernel, n <= 2^19)
    assert 0 < prof["n_spmv_dot"] <= s.nspmv
    assert prof["ms_spmv_dot"] > 0 and prof["bytes_spmv_dot"] > 0


@pytest.mark.parametrize("name", ["c3", "c4", "c2_med"])
def test_persistent_kernel_forced(orc, name):
    # option persist = 2 forces the cooperative whole-extension kernel (several tiles per CTA at full
    # size), also for the Arnoldi extension of c3 (n = 1M) that defaults to the two-kernel path
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), options={"persist": 2})
    assert c.get_option("persist") == 2
    w, s = c.solve_stencil(Pb.t, stencil_of(Pb), [to_dev(x) for x in Pb.u], tol=Pb.tol,
                           symmetric=Pb.symmetric, m_init=Pb.m_init)
    wo, so = run_oracle(orc, Pb)
    assert s.t_reached == Pb.t
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(Pb.tol), (s, so)
    c.close()


def test_batch_matches_single_solves():
    # phipm_solve_stencil_batch / _csr_batch: nb independent problems on nb contexts and native
    # threads; each output equals the single solve bit for bit (deterministic kernels per stream)
    import torch
    import paper_0907_4631_b200 as P
    Pb = W.make("c1_mini")
    S = stencil_of(Pb)
    ts = [Pb.t, 0.5 * Pb.t, 2 * Pb.t, Pb.t]
    us = [[to_dev(x) for x in Pb.u], [to_dev(x) for x in Pb.u[:2]], [to_dev(x) for x in Pb.u], [to_dev(Pb.u[0])]]
    ctxs = [P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=4, stream=torch.cuda.Stream()) for _ in ts]
    kw = dict(tol=Pb.tol, symmetric=Pb.symmetric)
    outs, stats = P.solve_batch(ctxs, ts, S, us, **kw)
    torch.cuda.synchronize()
    one = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=4)
    for b in range(len(ts)):
        w, s = one.solve_stencil(ts[b], S, us[b], **kw)
        assert torch.equal(w, outs[b]) and s.nspmv == stats[b].nspmv
    # CSR operands
    A = tuple(to_dev(a) for a in W.make("c5_mini").csr)
    P5 = W.make("c5_mini")
    u5 = [to_dev(x) for x in P5.u]
    ctx5 = [P.Context(n_max=P5.n, m_max=P5.m_max, p_max=4, stream=torch.cuda.Stream()) for _ in range(3)]
    outs5, _ = P.solve_batch(ctx5, P5.t, A, [u5] * 3, tol=P5.tol)
    ref = P.Context(n_max=P5.n, m_max=P5.m_max, p_max=4).solve_csr(P5.t, A, u5, tol=P5.tol)[0]
    for o in outs5:
        assert torch.equal(o, ref)
    # distinct contexts are required
    with pytest.raises(P.PhipmError):
        P.solve_batch([ctxs[0], ctxs[0]], Pb.t, S, [us[0], us[0]], **kw)


@pytest.mark.parametrize("modes", [1, 2, 3])
def test_stencil_arnoldi_early_breakdown(ctx, orc, modes):
    # u0 = a combination of `modes` eigenvectors of the Dirichlet Laplacian (discrete sines): the Krylov
    # space has dimension `modes`, so Arnoldi (symmetric=False on purpose) breaks down at j = modes.
    # n > SMALL_N takes the streaming two-kernel path, whose lagged normalisation detects the
    # breakdown inside the next SpMV's finalize.
    import workloads as W2
    nx = ny = 100
    h2 = float((nx + 1) ** 2)
    coef = (-4.0 * h2, h2, h2, h2, h2, 0.0, 0.0)
    x = np.arange(1, nx + 1) / (nx + 1)
    u0 = np.zeros(nx * ny)
    for k in range(1, modes + 1):
        u0 += (1.0 / k) * np.outer(np.sin(k * np.pi * x), np.sin((k + 1) * np.pi * x)).ravel()
    Pb = W2.Problem(name="bd", n=nx * ny, t=1e-4, tol=1e-10, p=0, symmetric=False, m_init=10, m_max=100,
                    u=[u0], stencil=W2.Stencil(2, nx, ny, 1, coef), csr=None, seed=0)
    wo, so = run_oracle(orc, Pb)
    wg, sg = run_gpu(ctx, Pb, "stencil")
    assert sg.t_reached == Pb.t
    if modes < 3:
        assert sg.nspmv <= modes and so["nspmv"] <= modes   # breakdown: the basis stops at `modes`
    else:
        # three modes: rounding leaves h_{3,2} ~ 6e-6 > n eps ||A||_inf ~ 1.8e-7 (R22), so neither side
        # breaks down; both must still build the same number of vectors
        assert sg.nspmv == so["nspmv"]
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


# ------------------------------------------------------------------------------------------------
# controller trajectory (Alg. 3/4) against the oracle's, attempt by attempt


def _traj_compare(ga, tr, rtol_h=1e-9, rtol_omega=1e-6, rtol_tau=1e-9, rtol_beta=1e-10):
    """Index of the first attempt whose decision differs, or len; asserts everything before it
    (and the decision inputs at it) agree.  rtol_h: ||H_mu||_1 (it only enters the cost model's
    M(.) through ceil(log2(.)), R20)."""
    for i, (g, o) in enumerate(zip(ga, tr)):
        t_k, tau, m, mu, omega, eps, acc, br, nh, beta = o
        assert g["m"] == int(m) and g["mu"] == int(mu), (i, g, o)
        assert g["tau"] == pytest.approx(tau, rel=rtol_tau), (i, g, o)
        assert g["t_k"] == pytest.approx(t_k, rel=max(1e-12, rtol_tau), abs=1e-300), (i, g, o)
        assert g["beta"] == pytest.approx(beta, rel=rtol_beta), (i, g, o)
        assert g["normH1"] == pytest.approx(nh, rel=rtol_h), (i, g, o)
        # eps is the corrector term |h phi_{p+1}[mu]|: relative agreement only where it is well above
        # the rounding of the small exponential (omega >= 1e-6)
        if omega >= 1e-6:
            assert g["omega"] == pytest.approx(omega, rel=rtol_omega), (i, g, o)
        if g["accepted"] != int(acc) or g["branch"] != int(br):
            return i
    return min(len(ga), len(tr))


@pytest.mark.parametrize("name,path", [("c2", "stencil"), ("c2", "csr"), ("c3", "stencil"), ("c4", "stencil"),
                                       ("c5", "csr"), ("c3_med", "stencil"), ("c5_med", "csr")])
def test_controller_trajectory_matches_oracle(ctx, orc, name, path):
    """GPU stats == oracle stats and the same attempt sequence (tau, m, mu, accept, branch), omega to
    1e-6: the host controller (phipm.cu control()) and the oracle's (orc_control) make every decision
    alike on inputs that agree to rounding.  Only an oracle attempt with omega within 1e-6 of delta
    may legitimately flip (none does on these configs)."""
    Pb = W.make(name)
    wg, sg = run_gpu(ctx, Pb, path)
    ga = ctx.attempts()
    wo, so, tr = orc.solve(Pb)
    near = np.abs(tr[:, 4] - 1.2) / 1.2 < 1e-6
    if near.any():
        pytest.skip(f"oracle attempt {int(np.argmax(near))} has omega within 1e-6 of delta")
    assert len(ga) == len(tr) == sg.nexpm, (sg, so)
    assert _traj_compare(ga, tr) == len(tr)
    assert (sg.nsteps, sg.nreject, sg.nspmv, sg.nexpm, sg.m_last, sg.m_peak) == \
        (so["nsteps"], so["nreject"], so["nspmv"], so["nexpm"], so["m_last"], so["m_peak"])


def test_controller_trajectory_c1(ctx, orc):
    """c1 (t||A|| = 4008, 14-15 steps): the first step's attempts agree with the oracle's to rounding
    (tau 1e-9, omega 1e-6, same m / accept / branch).  Later the Lanczos vectors lose orthogonality
    (m ~ 40 with the extreme Ritz values converged) and the T entries of two implementations drift
    apart beyond rounding (measured: ||H||_1 2e-4, omega 7e-4 at attempt 7, 1.3e-2 at attempt 9; tau and
    beta inherit it), so the rest is held to the solution (parity bar) and to the trajectory's size."""
    Pb = W.make("c1")
    wg, sg = run_gpu(ctx, Pb, "stencil")
    ga = ctx.attempts()
    wo, so, tr = orc.solve(Pb)
    first = int(np.argmax(tr[:, 6] == 1)) + 1           # attempts of the first step (through its accept)
    assert _traj_compare(ga[:first], tr[:first]) == first
    print(f"c1: gpu {sg} oracle {so}")
    assert abs(sg.nsteps - so["nsteps"]) <= 2
    assert abs(sg.nspmv - so["nspmv"]) <= 0.1 * so["nspmv"]
    assert relerr(wg, wo) <= parity_bound(Pb.tol)


@pytest.mark.parametrize("name,path,opts", [("c1_mini", "stencil", {}), ("c2_med", "stencil", {}),
                                            ("c3_med", "stencil", {"persist": 0}), ("c3_med", "stencil", {}),
                                            ("c4_tm", "stencil", {}), ("c5_med", "csr", {}),
                                            ("c2_mini", "csr", {}),
                                            ("c4_tm", "stencil", {"brick": 2}),
                                            ("c4_tm", "stencil", {"brick": 2, "brick_halo": 1, "precombine": 1})])
def test_guard_regions_and_inputs_untouched(orc, name, path, opts):
    """Out-of-bounds write check (compute-sanitizer is closed on this GPU pool): w is a view into a
    buffer with 4096-double guard regions of a NaN pattern on both sides, and every input (u_k, the
    CSR arrays) is compared bit for bit after the solve.  Every kernel family runs (single-CTA,
    persistent smem / TMEM Lanczos, cooperative w-recurrence, streaming TMA-halo, CSR x-ring, the brick
    kernels with their tensor-map copies -- c4_tm is 70^3: ragged x segments, ragged last bricks -- and the
    interior-resident brick variant with tensor stores and the guarded combine)."""
    import torch
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), options=opts)
    g = 4096
    buf = torch.full((Pb.n + 2 * g,), float("nan"), dtype=torch.float64, device="cuda")
    w = buf[g:g + Pb.n]
    u = [to_dev(x) for x in Pb.u]
    u_copy = [x.clone() for x in u]
    if path == "stencil":
        c.solve_stencil(Pb.t, stencil_of(Pb), u, out=w, tol=Pb.tol, symmetric=Pb.symmetric)
        A = A_copy = ()
    else:
        A = tuple(to_dev(a) for a in Pb.csr) if Pb.csr is not None else c.csr_from_stencil(stencil_of(Pb))
        A_copy = tuple(a.clone() for a in A)
        c.solve_csr(Pb.t, A, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric)
    torch.cuda.synchronize()
    assert torch.isnan(buf[:g]).all() and torch.isnan(buf[g + Pb.n:]).all()
    for a, b in zip(u + list(A), u_copy + list(A_copy)):
        assert torch.equal(a, b)
    wo, so = run_oracle(orc, Pb)
    assert relerr(w.cpu().numpy(), wo) <= parity_bound(Pb.tol)
    c.close()


@pytest.mark.parametrize("name", ["c5_med", "c5"])
def test_fused_anorm_matches_analysis_pass(orc, name):
    """||A||_inf (a1 setup) from the first w-recurrence SpMV (option fuse_anorm = 1, the default on
    the x-ring CSR path) against the analysis pass that reads val (fuse_anorm = 0, the oracle's
    sequential row sums bit for bit): the row sums differ only in summation order, so tau_0 and the
    whole trajectory agree to rounding, and w to far below the parity bar."""
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    A = tuple(to_dev(a) for a in Pb.csr)
    u = [to_dev(x) for x in Pb.u]
    res = {}
    for f in (1, 0):
        c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), options={"fuse_anorm": f})
        w, s = c.solve_csr(Pb.t, A, u, tol=Pb.tol)
        res[f] = (w.cpu().numpy(), s, c.attempts())
        c.close()
    (w1, s1, a1), (w0, s0, a0) = res[1], res[0]
    assert (s1.nsteps, s1.nreject, s1.nspmv) == (s0.nsteps, s0.nreject, s0.nspmv)
    for x, y in zip(a1, a0):
        assert x["tau"] == pytest.approx(y["tau"], rel=1e-14)
    assert relerr(w1, w0) <= 1e-13


def test_csr_int16_offsets_option(orc):
    """Option csr_off16 = 1 (int16 column offsets written by the analysis pass, streamed by the x-ring
    SpMV; off by default): parity with the oracle and the same trajectory as the int32 columns."""
    import paper_0907_4631_b200 as P
    Pb = W.make("c5_med")
    A = tuple(to_dev(a) for a in Pb.csr)
    u = [to_dev(x) for x in Pb.u]
    out = {}
    for f in (1, 0):
        c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=3, options={"csr_off16": f})
        w, s = c.solve_csr(Pb.t, A, u, tol=Pb.tol)
        out[f] = (w.cpu().numpy(), s)
        c.close()
    wo, so = run_oracle(orc, Pb)
    assert relerr(out[1][0], wo) <= parity_bound(Pb.tol)
    assert np.array_equal(out[1][0], out[0][0]) and out[1][1] == out[0][1]


@pytest.mark.parametrize("name,path", [("c5_med", "csr"), ("c3", "stencil")])
def test_graph_replay_matches_stream_launches(name, path):
    # option graph: the two-kernel extension captured as a CUDA graph and replayed from the context's cache
    # (second solve: every extension is a cache hit) -- the same kernels with the same arguments, so w and
    # the stats are bit-identical with the stream launches
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    res = {}
    for g in (0, 1):
        c = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1), options={"graph": g})
        for rep in range(2):
            w, s = run_gpu(c, Pb, path)
            res[(g, rep)] = (w, s)
        c.close()
    for key in ((1, 0), (1, 1), (0, 1)):
        assert np.array_equal(res[key][0], res[(0, 0)][0]), key
        assert res[key][1] == res[(0, 0)][1], key


@pytest.mark.parametrize("name,path,kw", [("c5_med", "csr", {}), ("c3", "stencil", {}), ("c3_med", "stencil", {"orth": 1}),
                                          ("c2", "csr", {}), ("c3_med", "csr", {})])
def test_deferred_finalize_matches_last_block_finalize(orc, name, path, kw):
    # option defer (default 1): the two-kernel extension's SpMV leaves its partials to the update kernel, whose
    # every CTA reduces them in final_reduce's order and derives H(:, j), g, sigma_j with finalize()'s
    # expressions (Arnoldi CGS, lagged Arnoldi on stencils, Lanczos on CSR, CGS2) -- w and the stats are
    # bit-identical with the SpMV's own last-block finalize, and within parity of the oracle
    import paper_0907_4631_b200 as P
    Pb = W.make(name)
    res = {}
    for d in (1, 0):
        c = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1), options={"defer": d})
        res[d] = run_gpu(c, Pb, path, **kw)
        c.close()
    assert np.array_equal(res[1][0], res[0][0])
    assert res[1][1] == res[0][1]
    wo, so = run_oracle(orc, Pb)             # (the oracle's MGS: CGS and CGS2 agree with it within parity)
    assert relerr(res[1][0], wo) <= parity_bound(Pb.tol)


def test_c5_structure_large_m_cgs_and_cgs2(ctx, orc):
    # R32 at the size where single-pass CGS loses orthogonality: the c5 operator class (random banded CSR,
    # c5_med) with a FIXED m = 45 (phip mode), so every step builds 45 Arnoldi columns.
    #   * CGS2 (orth = 1): the basis is orthonormal to rounding;
    #   * CGS (the default): ||V^T V - I|| is orders of magnitude larger (the loss the survey measured), and
    #     the solve still meets the bar against the MGS oracle in the same fixed-m mode, as does CGS2 --
    #     the error estimate and the step control absorb the loss (a non-orthogonal basis still spans K_m)
    Pb = W.make("c5_med")
    A = tuple(to_dev(a) for a in Pb.csr)
    m = 45
    loss = {}
    for orth in (0, 1):
        V, H, k, brk, beta = ctx.krylov(A, to_dev(Pb.u[-1]), m, symmetric=False, orth=orth)
        assert k == m and not brk
        V = V.cpu().numpy()
        loss[orth] = float(np.abs(V.T @ V - np.eye(m + 1)).max())
    assert loss[1] <= 1e-11, loss
    assert loss[0] >= loss[1], loss
    wo, so = run_oracle(orc, Pb, m_init=m, fixed_m=True)
    for orth in (0, 1):
        wg, sg = run_gpu(ctx, Pb, "csr", m_init=m, fixed_m=True, orth=orth)
        assert sg.m_peak == m and sg.t_reached == Pb.t
        assert relerr(wg, wo) <= parity_bound(Pb.tol), (orth, loss, sg, so)


@pytest.mark.parametrize("name", ["c2_med", "c3_med", "c4_med", "c5_med", "c4"])
def test_precombine_and_side_maxabs_are_bit_identical(name):
    import paper_0907_4631_b200 as P
    # precombine: the exponential's epilogue takes Algorithm 3's acceptance decision (omega <= 1.2, the host's
    # IEEE expression) and a guarded combine is enqueued before the host sees the result; side_maxabs:
    # ||u_0||_inf is reduced on the second stream.  Neither changes any arithmetic: w, the stats and the
    # controller trajectory are identical with both switched off
    import torch
    Pb = W.make(name)
    u = [to_dev(x) for x in Pb.u]
    A = tuple(to_dev(a) for a in Pb.csr) if Pb.csr is not None else None
    out = {}
    for flag in (1, 0):
        c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), options={"precombine": flag, "side_maxabs": flag})
        if A is None:
            w, s = c.solve_stencil(Pb.t, stencil_of(Pb), u, tol=Pb.tol, symmetric=Pb.symmetric)
        else:
            w, s = c.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric)
        out[flag] = (w.clone(), s, c.attempts())
        c.close()
    assert torch.equal(out[1][0], out[0][0])
    assert out[1][1] == out[0][1]
    assert out[1][2] == out[0][2]


def test_precombine_multistep_rejections(orc):
    import paper_0907_4631_b200 as P
    # several steps with rejected attempts in between (2-D Laplacian 181^2, t = 2e-3): every rejected attempt
    # leaves a guarded combine that must not run, every accepted one a combine that ran before the host
    # decided; parity with the oracle and identity with the host-launched combines
    import torch
    from test_gpu_tmem import laplacian
    st, u = laplacian(2, 181, 181, 1, seed=77, p=2)
    t, tol = 2e-3, 1e-9
    Pb = W.Problem(name="pc", n=st.n, p=2, t=t, tol=tol, symmetric=True, u=u, stencil=st, seed=0)
    wo, so, _ = orc.solve(Pb)
    ud = [to_dev(x) for x in u]
    res = {}
    for flag in (1, 0):
        c = P.Context(n_max=st.n, m_max=100, p_max=2, options={"precombine": flag})
        w, s = c.solve_stencil(t, P.Stencil.of(st), ud, tol=tol, symmetric=True)
        res[flag] = (w.clone(), s)
        c.close()
    s1 = res[1][1]
    assert s1.nsteps > 1 and s1.nreject > 0, s1
    assert torch.equal(res[1][0], res[0][0]) and res[1][1] == res[0][1]
    assert relerr(res[1][0].cpu().numpy(), wo) <= parity_bound(tol), (s1, so)
