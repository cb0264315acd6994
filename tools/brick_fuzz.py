"""Randomised cross-check of the brick kernels: random 3-D grid shapes (even nx <= 252), anisotropic
coefficients, p in 0..3, t chosen for a few attempts; solves with brick = 2 (both variants) against brick = 0
(contiguous-range / shared-memory / cluster kernels).  A case passes if the brick path ran, the two brick
variants are bit-identical, the stats equal the reference kernels' and w agrees within the parity bar of the
solve (10 tol: with p = 3 every implementation is ~3e-9 from the oracle, Eq. (step)'s cancellation).  Prints
every case; exits 1 on a disagreement.
Usage: python tools/brick_fuzz.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
P.build()
bad = 0
for ci in range(cases):
    while True:
        nx = 2 * int(rng.integers(2, 127))
        ny, nz = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        n = nx * ny * nz
        if 9000 <= n <= 1_500_000:
            break
    p = int(rng.integers(0, 4))
    cx, cy, cz = rng.uniform(0.3, 2.0, 3)
    h2 = float((nx + 1) ** 2)
    st = P.Stencil(3, nx, ny, nz, (-2 * (cx + cy + cz) * h2, cx * h2, cx * h2, cy * h2, cy * h2, cz * h2, cz * h2))
    u = [torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(p + 1)]
    t = float(rng.uniform(0.5, 6.0)) / (4 * (cx + cy + cz) * h2) * 40
    res = {}
    for key, opts in (("ref", {"brick": 0}), ("planes", {"brick": 2, "cluster_lz": 0}),
                      ("halo", {"brick": 2, "cluster_lz": 0, "brick_halo": 1})):
        c = P.Context(n_max=n, m_max=100, p_max=max(p, 1), options=opts)
        w, s = c.solve_stencil(t, st, u, tol=1e-9, symmetric=True)
        res[key] = (w.clone(), s, c.krylov_path(), c.wrec_path())
        c.close()
    plan = P.brick_plan(nx, ny, nz)
    wr = res["ref"][0]
    e1 = float((res["planes"][0] - wr).norm() / wr.norm())
    same = torch.equal(res["planes"][0], res["halo"][0])
    ok = (plan is None or (res["planes"][2] == "brick" and e1 <= 1e-8 and same and res["planes"][1] == res["ref"][1]))
    bad += 0 if ok else 1
    print(f"{'ok ' if ok else 'BAD'} {nx:3d}x{ny:3d}x{nz:3d} n={n:8d} p={p} plan={'-' if plan is None else (plan['py'], plan['pz'], plan['ylen'], plan['zlen'], plan['ppg'])} "
          f"paths {res['planes'][2]}/{res['planes'][3]} vs {res['ref'][2]}/{res['ref'][3]}  rel diff {e1:.1e}  variants equal {same}  {res['planes'][1]}")
sys.exit(1 if bad else 0)
