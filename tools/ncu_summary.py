"""Summarise ncu --set full reports: key metrics and top stall reasons (reads .ncu-rep via ncu -i)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]


def summary(path, ntop=8):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for w in WANT:
            if w in hdr:
                d[w] = (r[hdr.index(w)], units[hdr.index(w)])
        st = [(h, float(r[i])) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and r[i]]
        st = sorted([x for x in st if x[1] > 0], key=lambda x: -x[1])[:ntop]
        tot = sum(float(r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and r[i])
        d["stalls"] = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), round(100 * v / max(tot, 1), 1)) for h, v in st]
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summary(p):
            print("===", p, d["kernel"])
            for w in WANT:
                if w in d:
                    print(f"  {w:62s} {d[w][0]:>14s} {d[w][1]}")
            print("  stalls %:", d["stalls"])
