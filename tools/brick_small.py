import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_0907_4631_b200 as P
m = 20
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for nx, ny, nz in [(64, 64, 64), (48, 48, 48), (96, 64, 32), (128, 32, 32), (64, 64, 32), (32, 32, 32), (40, 40, 40)]:
    n = nx * ny * nz
    h2 = float((nx + 1) ** 2)
    st = P.Stencil(3, nx, ny, nz, (-6 * h2, h2, h2, h2, h2, h2, h2))
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
    res = {}
    for mode in (0, 2):
        for cl in (0, 1):
            c = P.Context(n_max=n, m_max=m + 2, p_max=1, options={"brick": mode, "cluster_lz": cl})
            for _ in range(2):
                c.krylov(st, v, m, symmetric=True, build_only=True)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); c.krylov(st, v, m, symmetric=True, build_only=True); e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / m)
            res[mode, cl] = (min(ts), c.krylov_path())
            c.close()
    print(f"{nx}x{ny}x{nz} n={n}: " + "  ".join(f"brick={k[0]},cl={k[1]}: {v[0]:.2f} us ({v[1]})" for k, v in res.items()))
