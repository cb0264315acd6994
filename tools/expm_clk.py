import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_0907_4631_b200 as P
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
rng = np.random.default_rng(0)
for mu, sc in ((40, 5.0), (40, 100.0), (52, 100.0), (52, 1000.0)):
    H = np.triu(rng.standard_normal((mu, mu)), -1)
    H *= sc / np.abs(H).sum(axis=0).max()
    Ht = torch.from_numpy(H).cuda()
    for _ in range(3): ctx.phi_pair(Ht, 1.0, 2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): ctx.phi_pair(Ht, 1.0, 2)
    b.record(); torch.cuda.synchronize()
    print(f"mu={mu} scale={sc}: {1e3*a.elapsed_time(b)/20:.1f} us/call incl host sync", flush=True)
