"""Phase cycles of one augmented exponential (expm_kernel, PHIPM_EXPM_CLOCKS=1): Lanczos-like symmetric
tridiagonal T of size mu with tau*||T||_1 ~ scale, p = 2 (phi_pair entry point, mode 2)."""
import os
import sys
os.environ["PHIPM_EXPM_CLOCKS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_0907_4631_b200 as P  # noqa: E402

ctx = P.Context(n_max=1024, m_max=100, p_max=5)
L = P.lib()
rng = np.random.default_rng(0)
for mu, sc in ((38, 50.0), (47, 380.0), (40, 5.0), (10, 2.0), (20, 20.0)):
    d = -2.0 - rng.uniform(0, 0.2, mu)
    e = 1.0 + rng.uniform(0, 0.1, mu - 1)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    T *= sc / np.abs(T).sum(axis=0).max()
    Tt = torch.from_numpy(T).cuda()
    best = None
    for _ in range(5):
        ctx.phi_pair(Tt, 1.0, 2)
        torch.cuda.synchronize()
        clk = (C.c_longlong * 16)()
        L.phipm_get_clocks(ctx._h, clk)
        c = list(clk)
        tot = c[6] - c[0]
        if best is None or tot < best[0]:
            best = (tot, c)
    tot, c = best
    m, s = c[7] >> 16, c[7] & 0xFFFF
    ph = [("build", c[1] - c[0]), ("A2,A3,A4", c[2] - c[1]), ("colsums", c[8] - c[2]), ("barrier", c[9] - c[8]),
          ("log2 est", c[10] - c[9]), ("degree", c[11] - c[10]), ("fold", c[4] - c[11]), ("Horner", c[3] - c[4]),
          ("squarings", c[5] - c[3]), ("epilogue", c[6] - c[5])]
    print(f"mu={mu} tau||T||={sc}: total {tot} cycles ({tot / 1965:.1f} us), Taylor m={m}, s={s}")
    for nm, v in ph:
        print(f"   {nm:10s} {v:7d}  {100 * v / max(tot, 1):5.1f} %")
