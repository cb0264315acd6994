"""A/B of compile-time variants: builds libphipm with each set of -D flags into lib/libphipm_<tag>.so
(here, no GPU needed), then (on the GPU box, --run) times solves of one config with each library in
its own process, interleaved rounds.

    python tools/ab_build.py --build "pipe0:-DPHIPM_RING_PIPE=0" "pipe3:-DPHIPM_RING_PIPE=3"
    python tools/ab_build.py --run --config c5 pipe0 pipe3
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--run", action="store_true")
ap.add_argument("--config", default="c5")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("items", nargs="+")
a = ap.parse_args()
import importlib  # noqa: E402
B = importlib.import_module("paper_0907_4631_b200.build")

if a.build:
    for it in a.items:
        tag, _, flags = it.partition(":")
        out = os.path.join(os.path.dirname(B.LIB), f"libphipm_{tag}.so")
        cmd = ["nvcc", *B.NVCC_FLAGS, *flags.split(), "-I", B.INCLUDE, "-o", out, *B._sources()]
        subprocess.check_call(cmd)
        print("built", out)
RUN = r'''
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_0907_4631_b200 as P, workloads as W
P.LIB = sys.argv[1]
Pb = W.make(sys.argv[2])
u = [torch.from_numpy(x).cuda() for x in Pb.u]
A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None
S = P.Stencil.of(Pb.stencil) if Pb.stencil is not None else None
c = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1))
w = torch.empty(Pb.n, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
def solve(**kw):
    if S is not None:
        return c.solve_stencil(Pb.t, S, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric, **kw)
    return c.solve_csr(Pb.t, A, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric, **kw)
for _ in range(3): solve()
tot = 0.0
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _, s = solve(); e1.record(); torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
c.reset_profile()
for _ in range(3):
    flush.zero_(); solve(profile=1)
pr = c.profile()
print(f"{10 / tot * 1e3:.1f} {pr['ms_spmv_dot'] / max(pr['n_spmv_dot'], 1) * 1e3:.1f} {s}")
'''
if a.run:
    res = {t: [] for t in a.items}
    for r in range(a.rounds):
        for t in a.items:
            lib = os.path.join(os.path.dirname(B.LIB), f"libphipm_{t}.so")
            o = subprocess.run([sys.executable, "-c", RUN, lib, a.config], cwd=ROOT, capture_output=True, text=True)
            res[t].append(o.stdout.strip() or o.stderr[-300:])
    for t, v in res.items():
        print(t, " | ".join(x.split(" Stats")[0] for x in v), "|", v[-1].split(" ", 2)[-1][:90])
