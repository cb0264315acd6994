"""Turn raw gpurun_out/ ncu outputs into the committed summaries under profiles/<round>/."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summary  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
src = os.path.join(ROOT, "gpurun_out")
# argv[2] (optional): output directory (on the GPU box: a directory under gpurun_out, which is what
# gpurun copies back); profiles/ncu_traffic.json then goes there too
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", rnd)
TRAFFIC = os.path.join(dst, "ncu_traffic.json") if len(sys.argv) > 2 else os.path.join(ROOT, "profiles",
                                                                                        "ncu_traffic.json")
os.makedirs(dst, exist_ok=True)


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    return [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h)]


def short(k):
    for key in ("krylov_brick_tm_kernel", "wrec_brick_kernel", "krylov_cluster_lanczos_kernel", "spmv_stream_kernel", "axpy_stream_kernel", "expm_kernel",
                "maxabs_kernel", "csr_analyze_kernel", "spmv_small_kernel", "axpy_small_kernel",
                "krylov_small_lanczos_kernel", "krylov_small_kernel", "krylov_persist_tm_kernel",
              "krylov_persist_kernel", "wrec_persist_kernel", "phi_cheb_kernel", "spmm_csr_ring_kernel",
              "spmm_csr_kernel"):
        if key in k:
            return key + ("<Stencil>" if "StencilOp" in k else "<Csr>" if "CsrOp" in k else "")
    return k[:40]


# 1) launch list of the bench command: per-kernel share of the step
import glob as _glob
for p in sorted(_glob.glob(os.path.join(src, "pf_launches_*.csv"))):
    lcfg = os.path.basename(p)[len("pf_launches_"):-4]
    d = read_ncu_csv(p)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in d:
        if r["Metric Name"] == "gpu__time_duration.sum":
            k = short(r["Kernel Name"])
            agg[k][0] += 1
            unit = r["Metric Unit"]
            agg[k][1] += float(r["Metric Value"].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
                                                                       "usecond": 1.0, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(dst, f"launches_{lcfg}_summary.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 2 --warmup 3 "
                f"--no-cpu-baseline  (config {lcfg}; cold-cache, serialised launches: compare SHARES)\n")
        f.write(f"{'kernel':34s} {'launches':>8s} {'total us':>10s} {'share':>7s}\n")
        for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k:34s} {n:8d} {us:10.1f} {100 * us / tot:6.1f}%\n")
    os.system(f"cp {p} {dst}/launches_{lcfg}.csv")

# 2) DRAM traffic per launch of each kernel class (exactly one solve: ncu --profile-from-start off)
traffic = {}
for cfg in ("c2", "c3", "c4", "c5"):
    p = os.path.join(src, f"pf_dram_{cfg}.csv")
    if not os.path.exists(p):
        continue
    d = read_ncu_csv(p)
    per = collections.defaultdict(dict)
    for r in d:
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1,
                 "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
        v = float(r["Metric Value"].replace(",", ""))
        per[r["ID"]][r["Metric Name"]] = v * scale
        per[r["ID"]]["kernel"] = short(r["Kernel Name"])
    cls = collections.defaultdict(list)
    for rid, m in per.items():
        cls[m["kernel"]].append((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                                 m.get("gpu__time_duration.sum", 0)))
    with open(os.path.join(dst, f"dram_traffic_{cfg}.txt"), "w") as f:
        f.write(f"ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                f"gpu__time_duration.sum  (exactly one {cfg} solve; cold-cache serialised launches)\n")
        for k, v in sorted(cls.items(), key=lambda x: -sum(t for _, t in x[1])):
            by = [b for b, _ in v]
            us = [t for _, t in v]
            f.write(f"{k:34s} launches {len(v):4d}  avg DRAM bytes/launch {sum(by) / len(by) / 1e6:9.2f} MB"
                    f"  avg {sum(us) / len(us):8.1f} us  total {sum(us):9.1f} us\n")
    # the bench's "spmv_dot" class: SpMV launches plus whole-extension Krylov kernels (persistent /
    # single-CTA), so the per-launch average matches bench.py's algorithmic_bytes_per_launch
    sp = [b for k in cls if k.startswith(("spmv_stream_kernel", "krylov_persist_kernel", "krylov_persist_tm_kernel",
                                                   "krylov_small_kernel", "krylov_small_lanczos_kernel",
                                                   "wrec_persist_kernel", "krylov_cluster_lanczos_kernel", "krylov_brick_tm_kernel",
                                                   "wrec_brick_kernel"))
          for b, _ in cls[k]]
    if sp:
        traffic[cfg] = {"kernel_class": "spmv_dot", "dram_bytes_per_launch": sum(sp) / len(sp),
                        "launches": len(sp), "source": f"profiles/{rnd}/dram_traffic_{cfg}.txt"}
    os.system(f"cp {p} {dst}/dram_{cfg}.csv")
if traffic:
    json.dump(traffic, open(TRAFFIC, "w"), indent=1)

# 3) --set full summaries of the top kernels
for name in ("pf_full_c3_spmv", "pf_full_c3_axpy", "pf_full_c4_persist", "pf_full_c5_spmv",
             "pf_full_c3_expm", "pf_full_c1_small", "pf_full_c5_axpy", "pf_full_c5_analyze", "pf_full_c1_cheb",
             "pf_full_c2_cluster", "pf_full_c2_expm", "pf_full_c4_brick", "pf_full_c4_wrec_brick"):
    p = os.path.join(src, name + ".ncu-rep")
    if os.path.exists(p):
        with open(os.path.join(dst, name.replace("pf_", "") + ".txt"), "w") as f:
            for d in summary(p):
                f.write(f"=== {d['kernel']}\n")
                for k, v in d.items():
                    if k not in ("kernel", "stalls"):
                        f.write(f"  {k:62s} {v[0]:>16s} {v[1]}\n")
                f.write(f"  warp stall samples (%): {d['stalls']}\n")
# 4) bench lines and in-kernel timelines
for cfg in ("c1", "c2", "c3", "c4", "c5"):
    p = os.path.join(src, f"pf_bench_{cfg}.json.log")
    if os.path.exists(p):
        lines = [x for x in open(p) if x.startswith("{")]
        if lines:
            open(os.path.join(dst, f"bench_{cfg}.json"), "w").write(lines[-1])
    p = os.path.join(src, f"kclock_{cfg}.txt")
    if os.path.exists(p):
        os.system(f"cp {p} {dst}/")
for extra in ("stream_roof.txt", "q_trace.txt", "rpt.txt"):
    p = os.path.join(src, extra)
    if os.path.exists(p):
        os.system(f"cp {p} {dst}/")
print("wrote", dst)
