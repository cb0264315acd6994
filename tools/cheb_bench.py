"""NEXT-2 latency table: phipm_phi_pair on symmetric tridiagonal T (Lanczos-like, spectrum in
[-2s, 0]) with the augmented DMMA Taylor exponential vs the Chebyshev phi-functions, K = mu + p + 1
from 15 to 55.  Per call, including launch and host synchronisation, and device time (CUDA events
around one launch, best of 20)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402

P.build()
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
rng = np.random.default_rng(0)
print(f"{'K':>4} {'mu':>4} {'p':>2} {'tau||T||':>9} | {'taylor us':>10} {'cheb us':>8} | {'taylor dev':>10} {'cheb dev':>9} | speedup")
for mu, p in ((12, 2), (10, 4), (20, 3), (30, 2), (40, 3), (50, 4), (52, 2)):
    for scale in (2.0, 50.0, 120.0):
        a = -scale + scale * rng.uniform(-1, 1, mu)
        b = 0.5 * scale * np.abs(rng.standard_normal(mu - 1))
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        Ht = torch.from_numpy(T).cuda()
        res = {}
        for meth in (P.EXPM_TAYLOR, P.EXPM_CHEBYSHEV):
            ctx.set_expm_method(meth)
            for _ in range(3):
                ctx.phi_pair(Ht, 1.0, p)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            N = 20
            e0.record()
            for _ in range(N):
                ctx.phi_pair(Ht, 1.0, p)
            e1.record()
            torch.cuda.synchronize()
            call = 1e3 * e0.elapsed_time(e1) / N
            best = 1e9
            for _ in range(N):
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record(ctx.stream)
                ctx.phi_pair(Ht, 1.0, p)
                c1.record(ctx.stream)
                torch.cuda.synchronize()
                best = min(best, 1e3 * c0.elapsed_time(c1))
            res[meth] = (call, best)
        nrm = np.abs(T).sum(axis=0).max()
        print(f"{mu + p + 1:4d} {mu:4d} {p:2d} {nrm:9.1f} | {res[0][0]:10.1f} {res[2][0]:8.1f} | "
              f"{res[0][1]:10.1f} {res[2][1]:9.1f} | {res[0][0] / res[2][0]:.2f}x")
ctx.set_expm_method(P.EXPM_TAYLOR)

# ---- in-solve device time per exponential (profile: CUDA events around each launch) and solves/s
import workloads as W  # noqa: E402

print()
print(f"{'config':>8} {'method':>10} | {'us/exp (device)':>15} {'n_exp':>6} | {'solves/s':>9} | stats")
for name in ("c1", "c2", "c4", "c2_med"):
    Pb = W.make(name)
    c2 = P.Context(n_max=Pb.n, m_max=100, p_max=4)
    S = P.Stencil.of(Pb.stencil)
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    for meth, mname in ((P.EXPM_TAYLOR, "taylor"), (P.EXPM_CHEBYSHEV, "chebyshev")):
        kw = dict(tol=Pb.tol, symmetric=True, expm_method=meth)
        for _ in range(3):
            c2.solve_stencil(Pb.t, S, u, **kw)
        c2.reset_profile()
        R = 10
        for _ in range(R):
            _, st = c2.solve_stencil(Pb.t, S, u, profile=1, **kw)
        pr = c2.profile()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c2.stream)
        for _ in range(R):
            c2.solve_stencil(Pb.t, S, u, **kw)
        e1.record(c2.stream)
        torch.cuda.synchronize()
        print(f"{name:>8} {mname:>10} | {1e3 * pr['ms_expm'] / max(pr['n_expm'], 1):15.1f} {pr['n_expm'] // R:6d} | "
              f"{R / (e0.elapsed_time(e1) / 1e3):9.1f} | {st}")
    c2.close()
