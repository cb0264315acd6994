"""Print the hottest SASS lines (warp-stall samples) of an ncu --page source --csv export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ci, si = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) > max(ci, si):
        try:
            data.append((float(r[si] or 0), r[0], r[ci].strip()))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
for v, a, s in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100 * v / tot:5.1f}%  {a[-5:]}  {s}")
