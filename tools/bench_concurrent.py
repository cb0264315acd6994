"""NEXT-3, first step: throughput of K independent phipm solves running concurrently on
one GPU, one context (workspace + CUDA stream) and one host thread each (the C ABI call releases the
GIL; each context's controller runs on its own thread).  Latency-bound configs (c1: the Krylov
extension is one single-CTA kernel, the exponential another) leave most SMs idle per solve, so
independent solves — e.g. the stages of an exponential integrator, the paper's intended use
 — can share the GPU.  Aggregate solves/s = K * R / wall time (host clock around
synchronised streams; single GPU, so there is no rank maximum).

  python tools/bench_concurrent.py --config c1 --ks 1,2,4,8,16,32 --reps 20
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--ks", default="1,2,4,8,16,32")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=None)
ap.add_argument("--option", action="append", default=[], help="context option name=value")
ap.add_argument("--api", default="threads", choices=["threads", "batch"],
                help="threads: one Python thread per context; batch: one phipm_solve_*_batch call (native threads)")
a = ap.parse_args()
P.build()
Pb = W.make(a.config)
u = [torch.from_numpy(x).cuda() for x in Pb.u]
A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None
torch.cuda.synchronize()
lines = [f"NEXT-3: K concurrent independent solves of {a.config} (n={Pb.n}), one context + stream each; "
         f"api={a.api} ({'one phipm_solve_*_batch call per round, native threads' if a.api == 'batch' else 'one Python thread per context'})"]
base = None
for K in [int(k) for k in a.ks.split(",")]:
    opts = {k: int(v) for k, v in (x.split("=") for x in a.option)}
    ctxs = [P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), stream=torch.cuda.Stream(), options=opts)
            for _ in range(K)]
    outs = [torch.empty(Pb.n, dtype=torch.float64, device="cuda") for _ in range(K)]

    def work(i, reps):
        c = ctxs[i]
        for _ in range(reps):
            if Pb.stencil is not None:
                c.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, out=outs[i], tol=Pb.tol, symmetric=Pb.symmetric)
            else:
                c.solve_csr(Pb.t, A, u, out=outs[i], tol=Pb.tol, symmetric=Pb.symmetric)
        c.stream.synchronize()

    def batch(reps):
        op = P.Stencil.of(Pb.stencil) if Pb.stencil is not None else A
        for _ in range(reps):
            P.solve_batch(ctxs, Pb.t, op, [u] * K, outs=outs, tol=Pb.tol, symmetric=Pb.symmetric)
        for c in ctxs:
            c.stream.synchronize()

    for i in range(K):                                      # warm-up
        work(i, 2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if a.api == "batch":
        batch(a.reps)
    else:
        ths = [threading.Thread(target=work, args=(i, a.reps)) for i in range(K)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rate = K * a.reps / dt
    base = base or rate
    # every stream computed the same problem: check they agree bit for bit (determinism across streams)
    same = all(torch.equal(outs[0], o) for o in outs[1:])
    lines.append(f"  K={K:3d}  {rate:9.1f} solves/s  ({rate / base:5.1f}x K=1)  outputs identical: {same}")
    print(lines[-1], flush=True)
    for c in ctxs:
        c.close()
    del ctxs, outs
    torch.cuda.empty_cache()
if a.out:
    open(a.out, "w").write("\n".join(lines) + "\n")
