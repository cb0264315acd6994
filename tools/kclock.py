"""In-kernel timeline of one phipm solve from per-CTA %globaltimer stamps (PHIPM_KCLOCKS).

Stamps per CTA (ns): 0 entry, 1 after the PDL wait, 2 first halo tile landed (stencil spmv),
3 end of the streaming body, 4 partials published; last CTA only: 5 grid reduction done,
6 finalize done.  Prints, per launch, where the time between consecutive kernels goes.
Usage: python tools/kclock.py [config]
"""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0907_4631_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
path = os.path.abspath("gpurun_out/kclock_%s.bin" % name)
if os.environ.get("PHIPM_LIB"):
    P.LIB = os.environ["PHIPM_LIB"]          # a variant built by tools/ab_build.py
else:
    P.build()
Pb = W.make(name)
u = [torch.from_numpy(x).cuda() for x in Pb.u]
A = tuple(torch.from_numpy(x).cuda() for x in Pb.csr) if Pb.csr is not None else None


def solve(ctx):
    if Pb.stencil is not None:
        return ctx.solve_stencil(Pb.t, P.Stencil.of(Pb.stencil), u, tol=Pb.tol, symmetric=Pb.symmetric)
    return ctx.solve_csr(Pb.t, A, u, tol=Pb.tol, symmetric=Pb.symmetric)


ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1))
for _ in range(3):
    solve(ctx)
torch.cuda.synchronize()
ctx.close()
os.environ["PHIPM_KCLOCKS"] = path
ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1))
print("stamped solve:", solve(ctx)[1])
torch.cuda.synchronize()
ctx.close()
del os.environ["PHIPM_KCLOCKS"]

recs = []
with open(path, "rb") as f:
    cnt = struct.unpack("i", f.read(4))[0]
    for _ in range(cnt):
        cls, grid, ncols = struct.unpack("iii", f.read(12))
        st = np.frombuffer(f.read(8 * 8 * grid), dtype=np.uint64).reshape(grid, 8).astype(np.int64)
        recs.append((cls, grid, ncols, st))
t00 = min(r[3][:, 0].min() for r in recs)
names = {0: "spmv", 1: "axpy"}
print(f"{name}: {cnt} streaming launches")
print("  kind cols  start  pdl_rel  entry_spread  halo1   body(med/max)  publish  finalred  fin   end   gap_to_next")
prev_end = None
tot = {"gap": 0.0, "pdl": 0.0, "body": 0.0, "tail": 0.0}
for i, (cls, grid, ncols, st) in enumerate(recs):
    s0, s1, s2, s3, s4 = (st[:, k] - t00 for k in range(5))
    last = int(np.argmax(st[:, 6]))
    e = st[last, 6] - t00 if st[last, 6] else s4.max()
    f5 = st[last, 5] - t00 if st[last, 5] else e
    body = (s3 - np.where(s2 > -t00, s2, s1)) / 1e3
    line = (f"  {names[cls]:4s} {ncols:4d} {s0.min() / 1e3:8.1f} {(s1.min() - s0.min()) / 1e3:6.1f} "
            f"{(s0.max() - s0.min()) / 1e3:6.1f} ")
    line += f"{(np.median(s2 - s1) / 1e3) if cls == 0 else 0:6.2f} {np.median(body):6.2f}/{body.max():6.2f} "
    line += f"{(s4.max() - s3.max()) / 1e3:6.2f} {(f5 - s4.max()) / 1e3:6.2f} {(e - f5) / 1e3:5.2f} {e / 1e3:8.1f}"
    if i + 1 < len(recs):
        nxt = recs[i + 1][3][:, 0].min() - t00
        nxt1 = recs[i + 1][3][:, 1].min() - t00
        line += f"  next entry {(nxt - e) / 1e3:+6.1f} pdl-release {(nxt1 - e) / 1e3:+6.1f}"
    print(line)

# persistent Krylov kernel: per phase, body end (max over CTAs) -> flag seen (max over CTAs)
pp = path + ".p"
if os.path.exists(pp):
    with open(pp, "rb") as f:
        cnt = struct.unpack("i", f.read(4))[0]
        for li in range(cnt):
            grid, steps = struct.unpack("ii", f.read(8))
            st = np.frombuffer(f.read(8 * 2 * steps * grid * 2), dtype=np.uint64).astype(np.int64)
            st = st.reshape(2 * steps, grid, 2)
            valid = st[:, :, 1].max(axis=1) > 0
            st = st[valid]
            t0 = st[0, :, 0].min()
            print(f"persistent launch {li}: grid {grid}, {steps} steps, {len(st)} phases")
            print("  phase  body(min/med/max end, us rel. prev release)   sync(max body end -> last release seen)  period")
            prev = None
            for ph in range(len(st)):
                be, rs = st[ph, :, 0], st[ph, :, 1]
                base = prev if prev is not None else be.min()
                print(f"  {ph:3d} {'A' if ph % 2 == 0 else 'B'}  {(be.min() - base) / 1e3:7.2f} {(np.median(be) - base) / 1e3:7.2f} "
                      f"{(be.max() - base) / 1e3:7.2f}   {(rs.max() - be.max()) / 1e3:7.2f}   "
                      f"{(rs.max() - base) / 1e3:7.2f}")
                prev = rs.max()
