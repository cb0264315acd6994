"""A/B of kernel-path options on one config: solves/s (device time, L2 flushed between solves, no
per-kernel events) and the SpMV class's per-launch algorithmic GB/s (profiled solves), interleaved.

    python tools/ab_opts.py --config c5 "csr_prefetch=0" "csr_prefetch=1536" [--rounds 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--solves", type=int, default=10)
ap.add_argument("settings", nargs="+", help="comma-separated name=value lists; 'default' for none")
a = ap.parse_args()
P.build()
Pb = W.make(a.config)
u = [torch.from_numpy(x).cuda() for x in Pb.u]
A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None
S = P.Stencil.of(Pb.stencil) if Pb.stencil is not None else None
w = torch.empty(Pb.n, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ctxs = {}
for st in a.settings:
    opts = {} if st == "default" else {k: int(v) for k, v in (x.split("=") for x in st.split(","))}
    ctxs[st] = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), options=opts)


def solve(c, **kw):
    if S is not None:
        return c.solve_stencil(Pb.t, S, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric, **kw)
    return c.solve_csr(Pb.t, A, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric, **kw)


res = {st: [] for st in a.settings}
for rnd in range(a.rounds):
    for st, c in ctxs.items():
        for _ in range(3):
            solve(c)
        tot = 0.0
        for _ in range(a.solves):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, s = solve(c)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        c.reset_profile()
        for _ in range(3):
            flush.zero_()
            solve(c, profile=1)
        pr = c.profile()
        gbs = pr["bytes_spmv_dot"] / 1e6 / pr["ms_spmv_dot"]
        res[st].append((a.solves / tot * 1e3, gbs, pr["ms_spmv_dot"] / max(pr["n_spmv_dot"], 1) * 1e3))
for st, v in res.items():
    best = max(v)
    print(f"{a.config} {st:30s} solves/s {best[0]:8.1f} (all {[round(x[0], 1) for x in v]})  spmv class "
          f"{max(x[1] for x in v):7.0f} GB/s  {min(x[2] for x in v):7.1f} us/launch  stats {s}")
