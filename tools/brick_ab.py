"""Brick Lanczos kernel vs the contiguous-range TMEM kernel on 3-D grids of several shapes: time of a
Lanczos extension to m columns (phipm_krylov_stencil, build only), L2 flushed, per step.
Usage: python tools/brick_ab.py [m]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 20
P.build()
SHAPES = [(128, 128, 128), (64, 256, 128), (192, 96, 96), (96, 96, 96), (128, 64, 64), (252, 100, 80),
          (64, 64, 128), (160, 160, 80), (128, 128, 40), (128, 200, 150)]
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
print(f"{'grid':>16s} {'n':>9s}  {'tmem us/step':>12s} {'brick us/step':>13s}  path(auto)")
for nx, ny, nz in SHAPES:
    n = nx * ny * nz
    h2 = float((nx + 1) ** 2)
    st = P.Stencil(3, nx, ny, nz, (-6 * h2, h2, h2, h2, h2, h2, h2))
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
    res = {}
    for mode in (0, 2, 1):
        c = P.Context(n_max=n, m_max=m + 2, p_max=1, options={"brick": mode})
        for _ in range(2):
            c.krylov(st, v, m, symmetric=True, build_only=True)
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c.krylov(st, v, m, symmetric=True, build_only=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / m)
        res[mode] = (min(ts), c.krylov_path())
        c.close()
    print(f"{nx:4d}x{ny:4d}x{nz:4d} {n:9d}  {res[0][0]:12.2f} {res[2][0]:13.2f}  {res[1][1]} ({res[0][1]} / {res[2][1]})")
