"""Per-step latency of the Krylov extension on the small/latency-bound configs.

Times phipm_krylov_* in build-only mode (seed + m steps, no export) for two m and reports the
difference per step, so the fixed cost of the call (seed, host sync) cancels.
Usage: python tools/krylov_lat.py [config[:option=value,...] ...]   (default c1 c2)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def per_call_us(ctx, A, v, m, sym, reps):
    for _ in range(3):
        ctx.krylov(A, v, m, symmetric=sym, build_only=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.krylov(A, v, m, symmetric=sym, build_only=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def main():
    names = sys.argv[1:] or ["c1", "c2"]
    for spec in names:
        name, _, o = spec.partition(":")
        opts = {k: int(v) for k, v in (kv.split("=") for kv in o.split(",") if kv)}
        Pb = W.make(name)
        ctx = P.Context(n_max=Pb.n, m_max=100, p_max=max(Pb.p, 1), options=opts)
        v = torch.from_numpy(Pb.u[0]).cuda()
        A = P.Stencil.of(Pb.stencil) if Pb.stencil is not None else tuple(torch.from_numpy(x).cuda() for x in Pb.csr)
        lo, hi = 10, 50
        t_lo = min(per_call_us(ctx, A, v, lo, Pb.symmetric, 200) for _ in range(3))
        t_hi = min(per_call_us(ctx, A, v, hi, Pb.symmetric, 200) for _ in range(3))
        print(f"{spec}: n={Pb.n} sym={Pb.symmetric}  m={lo}: {t_lo:.1f} us  m={hi}: {t_hi:.1f} us  "
              f"per step {(t_hi - t_lo) / (hi - lo):.3f} us")
        ctx.close()


if __name__ == "__main__":
    main()
