"""Per-phase cycles of the Chebyshev phi kernel (PHIPM_EXPM_CLOCKS=1), Lanczos-like T."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_0907_4631_b200 as P
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
ctx.set_expm_method(P.EXPM_CHEBYSHEV)
rng = np.random.default_rng(0)
for mu, p, sc in ((10, 4, 1.0), (38, 3, 25.0), (40, 2, 56.0), (47, 2, 112.0), (60, 2, 400.0)):
    a = -sc + sc * rng.uniform(-1, 1, mu)
    b = 0.5 * sc * np.abs(rng.standard_normal(mu - 1))
    T = torch.from_numpy(np.diag(a) + np.diag(b, 1) + np.diag(b, -1)).cuda()
    for _ in range(2):
        ctx.phi_pair(T, 1.0, p)
    torch.cuda.synchronize()
    print(f"mu={mu} p={p} scale={sc}", flush=True)
    ctx.phi_pair(T, 1.0, p)
    torch.cuda.synchronize()
