"""A few phi_pair calls at one K (short command for ncu on the expm kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402

mu = int(sys.argv[1]) if len(sys.argv) > 1 else 40
P.build()
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
rng = np.random.default_rng(0)
H = np.triu(rng.standard_normal((mu, mu)), -1)
H *= 100.0 / np.abs(H).sum(axis=0).max()
Ht = torch.from_numpy(H).cuda()
for _ in range(3):
    ctx.phi_pair(Ht, 1.0, 2)
torch.cuda.synchronize()
print("ok", mu)
