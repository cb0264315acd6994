"""Per-launch trace of phipm solves (profile=2): fits time = t0 + bytes/BW per kernel class."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

CLS = ["spmv_dot", "orth", "expm", "combine", "other"]
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c3,c4,c5")
ap.add_argument("--out", default="gpurun_out/trace.json")
a = ap.parse_args()
P.build()
res = {}
for name in a.configs.split(","):
    Pb = W.make(name)
    ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1))
    u = [torch.from_numpy(x).cuda() for x in Pb.u]
    A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None

    def solve(profile):
        if Pb.stencil is not None:
            return ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric,
                                     profile=profile)
        return ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric, profile=profile)

    for _ in range(3):
        solve(0)
    ctx.reset_profile()
    w, st = solve(2)
    tr = ctx.trace()
    out = {"stats": str(st), "launches": tr, "fits": {}}
    print(f"== {name} n={Pb.n} {st}")
    for ci, cn in enumerate(CLS):
        rows = [r for r in tr if r[0] == ci]
        if not rows:
            continue
        us = np.array([r[3] for r in rows])
        by = np.array([r[2] for r in rows])
        tot_us, tot_by = us.sum(), by.sum()
        line = f"  {cn:9s} n={len(rows):3d} total {tot_us:8.1f} us  avg {us.mean():7.1f} us"
        if tot_by > 0:
            line += f"  agg {tot_by / tot_us / 1e3:7.1f} GB/s"
            if len(rows) > 3 and by.std() > 0:
                X = np.stack([np.ones_like(by), by], 1)
                coef, *_ = np.linalg.lstsq(X, us, rcond=None)
                line += f"  fit t0={coef[0]:6.1f} us  BW={1e-3 / coef[1] if coef[1] > 0 else float('inf'):7.1f} GB/s"
                out["fits"][cn] = [float(coef[0]), float(coef[1])]
        print(line)
    for r in tr[:60]:
        print(f"    {CLS[r[0]]:9s} cols={r[1]:3d} {r[2] / 1e6:8.2f} MB {r[3]:8.1f} us "
              f"{(r[2] / r[3] / 1e3) if r[3] > 0 and r[2] > 0 else 0:7.1f} GB/s")
    res[name] = out
    ctx.close()
json.dump(res, open(a.out, "w"))
