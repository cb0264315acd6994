"""Absolute timeline of one solve from the PHIPM_KCLOCKS stamps (run after tools/kclock.py <cfg> wrote
gpurun_out/kclock_<cfg>.bin[.p]): first / last stamp of every stamped launch on one time base."""
import struct
import sys

import numpy as np

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
path = "gpurun_out/kclock_%s.bin" % name
ev = []
with open(path, "rb") as f:
    cnt = struct.unpack("i", f.read(4))[0]
    for _ in range(cnt):
        cls, grid, ncols = struct.unpack("iii", f.read(12))
        st = np.frombuffer(f.read(8 * 8 * grid), dtype=np.uint64).reshape(grid, 8).astype(np.int64)
        v = st[st > 0]
        ev.append((int(v.min()), int(v.max()), f"{'spmv' if cls == 0 else 'axpy'} cols={ncols} grid={grid}"))
with open(path + ".p", "rb") as f:
    cnt = struct.unpack("i", f.read(4))[0]
    for li in range(cnt):
        grid, steps = struct.unpack("ii", f.read(8))
        st = np.frombuffer(f.read(8 * 2 * steps * grid * 2), dtype=np.uint64).astype(np.int64)
        v = st[st > 0]
        ev.append((int(v.min()), int(v.max()), f"persistent launch {li} grid={grid} steps={steps} (first phase end .. last release)"))
ev.sort()
t0 = ev[0][0]
prev = None
for a, b, what in ev:
    gap = f"  (+{(a - prev) / 1e3:6.1f} us after the previous last stamp)" if prev is not None else ""
    print(f"{(a - t0) / 1e3:8.1f} .. {(b - t0) / 1e3:8.1f} us  {what}{gap}")
    prev = b
