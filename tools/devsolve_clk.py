"""Phase cycles of the device-driven small solve (solve_small.cuh) with PHIPM_EXPM_CLOCKS=1."""
import os
import sys
os.environ["PHIPM_EXPM_CLOCKS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402
import torch  # noqa: E402
import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

for name in sys.argv[1:] or ["c1"]:
    Pb = W.make(name)
    ctx = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1))
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    for _ in range(3):
        w, s = ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=True)
    torch.cuda.synchronize()
    L = P.lib()
    clk = (C.c_longlong * 16)()
    L.phipm_get_clocks(ctx._h, clk)
    names = ["setup", "wrec+seed", "extensions", "exponential", "controller", "combine"]
    tot = sum(clk[i] for i in range(6))
    print(name, s)
    for i, nm in enumerate(names):
        print(f"  {nm:12s} {clk[i]:10d} cycles  {100 * clk[i] / max(tot, 1):5.1f} %   {clk[i] / 1965.0:8.1f} us")
    ctx.close()
