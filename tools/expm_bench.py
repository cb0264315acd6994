"""Time the single-CTA augmented exponential (phipm_phi_pair) vs K and ||tau H||."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402

P.build()
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
rng = np.random.default_rng(0)
for mu in (10, 20, 30, 40, 60, 64, 66, 80, 100):
    for scale in (0.01, 100.0):
        H = np.triu(rng.standard_normal((mu, mu)), -1)
        H *= scale / np.abs(H).sum(axis=0).max()
        Ht = torch.from_numpy(H).cuda()
        for _ in range(3):
            ctx.phi_pair(Ht, 1.0, 2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        N = 20
        a.record()
        for _ in range(N):
            ctx.phi_pair(Ht, 1.0, 2)
        b.record()
        torch.cuda.synchronize()
        print(f"mu={mu:3d} K={mu + 3:3d} ||H||_1={scale:7.2f}  {1e3 * a.elapsed_time(b) / N:8.1f} us/call (incl. host sync)")
