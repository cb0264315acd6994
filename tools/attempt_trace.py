import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_0907_4631_b200 as P, workloads as W
for name in ["c1", "c2", "c3", "c4", "c5"]:
    Pb = W.make(name)
    ctx = P.Context(n_max=Pb.n, m_max=100, p_max=4)
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    if Pb.stencil is not None:
        w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric)
    else:
        A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr)
        w, s = ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric)
    at = ctx.attempts()
    print(name, s)
    print("   ", [(a["m"], "A" if a["accepted"] else "R", a["branch"]) for a in at] if isinstance(at[0], dict) else at[:3])
    ctx.close()
