"""Run a few phipm solves of one config (short command for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--orth", type=int, default=0)
ap.add_argument("--option", action="append", default=[], help="kernel-path option name=value (phipm_set_option)")
ap.add_argument("--expm", type=int, default=0, help="expm_method (0 Taylor, 1 Pade-13, 2 Chebyshev)")
ap.add_argument("--profile-last", action="store_true",
                help="wrap only the last solve in cudaProfilerStart/Stop (ncu --profile-from-start off)")
a = ap.parse_args()
Pb = W.make(a.config)
P.build()
ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1),
                options={k: int(v) for k, v in (x.split("=") for x in a.option)})
u = [torch.from_numpy(x).cuda() for x in Pb.u]
for i in range(a.solves):
    if a.profile_last and i == a.solves - 1:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    if Pb.stencil is not None:
        w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric, orth=a.orth,
                                 expm_method=a.expm)
    else:
        A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr)
        w, s = ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric, orth=a.orth,
                                 expm_method=a.expm)
torch.cuda.synchronize()
if a.profile_last:
    torch.cuda.cudart().cudaProfilerStop()
print(a.config, s)
