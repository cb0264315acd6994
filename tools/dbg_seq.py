import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, paper_0907_4631_b200 as P, workloads as W
def run(ctx, name):
    Pb = W.make(name)
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric, m_init=Pb.m_init)
    at = ctx.attempts()
    return w.cpu().numpy(), s, at
ref = {}
c = P.Context(n_max=70000, m_max=100, p_max=4)
w0, s0, a0 = run(c, "c2"); c.close()
for opts in ({}, {"devsolve": 0}, {"spec": 0}, {"cluster_lz": 0}):
    c = P.Context(n_max=4_194_304, m_max=100, p_max=5, options=opts)
    w1, s1, a1 = run(c, "c1")
    w2, s2, a2 = run(c, "c2")
    print(opts, "c2 after c1", s2, "same as fresh:", np.array_equal(w0, w2), a2[0]["beta"], [(a["m"], a["accepted"]) for a in a2])
    c.close()
