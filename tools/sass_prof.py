"""Summaries of an `ncu --page source --csv --print-source sass` export: executed warp instructions by
opcode, the hottest SASS lines by stall samples, and the stall reasons of the whole kernel.
Usage: python tools/sass_prof.py gpurun_out/p4_sass.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ie, isrc, ismp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("# Samples")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = []
for r in rows[2:]:
    try:
        data.append((r[0], r[isrc].strip(), float(r[ie] or 0), float(r[ismp] or 0), [float(r[i] or 0) for i in stalls]))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data)
smp = sum(d[3] for d in data) or 1
print(f"{len(data)} SASS lines, {tot:.0f} warp instructions executed, {smp:.0f} samples")
op = collections.Counter()
for a, s, e, sm, _ in data:
    m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_.]+)", s)
    op[m.group(2).split(".")[0] if m else s[:8]] += e
print("opcode mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in op.most_common(24)))
st = collections.Counter()
for d in data:
    for i, v in zip(stalls, d[4]):
        st[hdr[i]] += v
print("stalls:", ", ".join(f"{k[6:]} {100 * v / smp:.1f}%" for k, v in st.most_common(10)))
print("hottest lines (samples%, executed, address, instruction, top stall):")
for a, s, e, sm, sv in sorted(data, key=lambda d: -d[3])[:top]:
    k = max(range(len(sv)), key=lambda i: sv[i]) if sv else 0
    print(f"{100 * sm / smp:5.1f}%  {e:9.0f}  {a[-5:]}  {s[:70]:70s} {hdr[stalls[k]][6:] if sv else ''}")
