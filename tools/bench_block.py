"""NEXT-3 throughput: nb problems with the c5 operator (or another CSR config) as
  (a) nb sequential single solves, (b) phipm_solve_csr_batch (worker pool, nb streams),
  (c) phipm_solve_csr_block (one SpMM pass over A per Krylov step).
Device time with CUDA events, L2 flushed between repetitions; solves/s = nb / time."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--nb", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
P.build()
Pb = W.make(a.config)
A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
rng = np.random.default_rng(9)
NBMAX = max(int(x) for x in a.nb.split(","))
us = [[torch.from_numpy(Pb.u[0] if b == 0 else rng.standard_normal(Pb.n)).cuda()] +
      [torch.from_numpy(Pb.u[k] if b == 0 else rng.uniform(-1, 1, Pb.n)).cuda() for k in range(1, Pb.p + 1)]
      for b in range(NBMAX)]
ctxs = [P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), stream=torch.cuda.Stream()) for _ in range(NBMAX)]
kw = dict(tol=Pb.tol, symmetric=Pb.symmetric, m_init=Pb.m_init)


def timed(fn):
    best = 1e30
    for _ in range(a.reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


print(f"{a.config}: n={Pb.n}, nnz={len(Pb.csr[1])}")
for nb in (int(x) for x in a.nb.split(",")):
    seq = lambda: [ctxs[0].solve_csr(Pb.t, A, us[b], **kw) for b in range(nb)]
    bat = lambda: P.solve_batch(ctxs[:nb], Pb.t, A, us[:nb], **kw)
    blk = lambda: P.solve_block(ctxs[:nb], Pb.t, A, us[:nb], **kw)
    for f in (seq, bat, blk):
        f()
    ts, tb, tk = timed(seq), timed(bat), timed(blk)
    _, st = P.solve_block(ctxs[:nb], Pb.t, A, us[:nb], **kw)
    print(f"nb={nb}: sequential {1e3 * nb / ts:7.1f} | batch {1e3 * nb / tb:7.1f} | block {1e3 * nb / tk:7.1f} solves/s"
          f"   (block stats {st[0].nsteps} steps, {st[0].nexpm} expm, m {st[0].m_peak}, nspmv {st[0].nspmv})", flush=True)
