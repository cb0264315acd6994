import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_0907_4631_b200 as P, workloads as W
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for nx in (64, 48, 96):
    Pb = W.c4(nx=nx)
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    S = P.Stencil.of(Pb.stencil)
    for mode in (1, 0, 1, 0):
        c = P.Context(n_max=Pb.n, m_max=100, p_max=4, options={"brick": mode})
        w = torch.empty(Pb.n, dtype=torch.float64, device="cuda")
        for _ in range(3): c.solve_stencil(Pb.t, S, u, out=w, tol=Pb.tol, symmetric=True)
        tot = 0.0
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); _, s = c.solve_stencil(Pb.t, S, u, out=w, tol=Pb.tol, symmetric=True); e1.record()
            torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
        print(f"c4(nx={nx}) n={Pb.n} brick={mode}: {10 / tot * 1e3:8.1f} solves/s  paths {c.krylov_path()} / {c.wrec_path()}  {s}")
        c.close()
