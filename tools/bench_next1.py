"""NEXT-1: adaptive phipm vs the fixed-m "phip" mode (m = 30, only tau adapts), the
comparison of the paper's Experiment 2 / Table 2, on the five
synthetic configs.  For each mode: GPU solves/s (device-resident inputs, CUDA events, median of R
solves), the stats (steps, rejections, products, exponentials, m) and the relative difference
from the oracle run in the same mode.

  python tools/bench_next1.py [--configs c1,c2,c3,c4,c5] [--reps 10] [--out gpurun_out/next1.txt]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--m-fixed", type=int, default=30)
ap.add_argument("--out", default="gpurun_out/next1.txt")
a = ap.parse_args()
P.build()
oracle.build()
lines = [f"NEXT-1: adaptive phipm vs fixed-m phip (m = {a.m_fixed}); B200, fp64; relerr vs the oracle in the same mode",
         f"{'config':7s} {'mode':9s} {'solves/s':>9s} {'ms':>8s} {'steps':>5s} {'rej':>4s} {'nSpMV':>6s} "
         f"{'nexpm':>5s} {'m_last':>6s} {'m_peak':>6s} {'relerr':>9s} {'|w_a-w_f|/|w|':>13s}"]
for name in a.configs.split(","):
    Pb = W.make(name)
    ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1))
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None
    res = {}
    for mode, kw in (("adaptive", dict(m_init=Pb.m_init)), ("fixed", dict(m_init=a.m_fixed, fixed_m=True))):
        def solve():
            if Pb.stencil is not None:
                return ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric, **kw)
            return ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric, **kw)
        for _ in range(3):
            w, st = solve()
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            w, st = solve()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        wg = w.cpu().numpy()
        wo, so, _ = oracle.solve(Pb, **kw)
        rel = float(np.linalg.norm(wg - wo) / np.linalg.norm(wo))
        res[mode] = wg
        diff = ""
        if mode == "fixed":
            wa = res["adaptive"]
            diff = f"{np.linalg.norm(wa - wg) / np.linalg.norm(wa):13.2e}"
        lines.append(f"{name:7s} {mode:9s} {1e3 / ms:9.1f} {ms:8.3f} {st.nsteps:5d} {st.nreject:4d} {st.nspmv:6d} "
                     f"{st.nexpm:5d} {st.m_last:6d} {st.m_peak:6d} {rel:9.2e} {diff}")
        print(lines[-1], flush=True)
    ctx.close()
os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
open(a.out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
