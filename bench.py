#!/usr/bin/env python
"""Benchmark: phipm solves/s on one BASELINE.json config, with the Arnoldi-step roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

A "step" is one full phipm solve (all SURVEY §8(a) rows: ||A||, w-recurrence, Krylov steps,
augmented expm, controller, assembly) of the named config, inputs resident in HBM.  Default
workload: c5 (random banded CSR, n = 4,194,304, 16 nnz/row, Arnoldi, p=3, t=0.5, tol=1e-8), the
largest BASELINE.json config (BASELINE.json quotes its metric on no single config).
Prints ONE JSON line (rank 0).  Under torchrun (N > 1) every rank solves its own replica
(independent problem, seed + rank): weak scaling, no collective on the data path.

--impl reference times the ORACLE (plain single-threaded C, oracle/) on this host on a bounded
sample of the same workload — the one other place bench.py runs oracle/ code.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "phipm solves/s and Arnoldi-step achieved HBM GB/s (SpMV+orthog) vs ~8 TB/s"

DESCR = {
    "c1": "c1: 1-D heat n=1000, Lanczos, p=2, t=1e-3, tol=1e-10",
    "c2": "c2: 2-D Laplacian 256^2, Lanczos, p=3, t=1e-4, tol=1e-10",
    "c3": "c3: 2-D advection-diffusion 1024^2 (n=1,048,576), Arnoldi, p=2, t=1e-3, tol=1e-8",
    "c4": "c4: 3-D Laplacian 128^3 (n=2,097,152), Lanczos, p=4, t=1e-5, tol=1e-10",
    "c5": "c5: random banded CSR n=4,194,304, 16 nnz/row, Arnoldi, p=3, t=0.5, tol=1e-8",
}


def measured_peak_hbm():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        load = [s for s in sm if s > 300] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def host_cpu():
    """Host CPU model and logical core count (stated next to the oracle timing)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"host_cpu": model, "host_logical_cores": os.cpu_count()}


def config_dict(name, Pb, path, world):
    """The `config` object of both arms (identical keys and values for the same workload)."""
    return {"workload": DESCR[name], "n": Pb.n, "p": Pb.p, "t": Pb.t, "tol": Pb.tol, "path": path,
            "parallelism": f"replicas x{world} (independent problems, no collective)",
            "l2": "flushed between timed steps (256 MiB memset outside the events)", "seed": Pb.seed}


def load_traffic(config):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config)
    except Exception:
        return None


# --------------------------------------------------------------------------------------------
def run_reference(args):
    """The oracle, as it stands, on this host: bounded sample of the same workload."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    oracle.build()
    Pb = W.make(args.config)
    csr = oracle.operator_csr(Pb)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        w, s, _ = oracle.phipm(Pb.t, csr, Pb.u, Pb.tol, m_init=Pb.m_init, m_max=Pb.m_max,
                               symmetric=Pb.symmetric)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
        if i == 0 and args.warmup > 1 and dt * (args.warmup + args.steps) > 240:
            args.warmup = 1                      # keep the run within a few minutes
    tot = sum(times)
    val = len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "solves/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, Pb, "stencil" if Pb.stencil is not None else "csr", args.gpus),
        "cpu_baseline": dict({"value": val, "unit": "solves/s", "cores": 1, "kind": "oracle",
                              "sample": f"{len(times)} full solves of {args.config} (single-threaded C oracle; "
                                        "stencil operators as the oracle's own CSR)"}, **host_cpu()),
        "e2e": {"value": val, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stats": s,
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(Pb, budget_s=15.0):
    import oracle
    oracle.build()
    csr = oracle.operator_csr(Pb)
    n_done, t_tot = 0, 0.0
    while True:
        t0 = time.perf_counter()
        oracle.phipm(Pb.t, csr, Pb.u, Pb.tol, m_init=Pb.m_init, m_max=Pb.m_max, symmetric=Pb.symmetric)
        t_tot += time.perf_counter() - t0
        n_done += 1
        if t_tot >= budget_s or n_done >= 50:
            break
    return dict({"value": n_done / t_tot, "unit": "solves/s", "cores": 1, "kind": "oracle",
                 "sample": f"{n_done} full solve(s) of the same {Pb.name} workload, single thread, {t_tot:.1f} s"},
                **host_cpu())


# ---- multi-rank host logic (replicas only: independent problems, no data-path collective) ----

GENERATORS = {"c1": W.c1, "c2": W.c2, "c3": W.c3, "c4": W.c4, "c5": W.c5}


def replica_problem(config, rank):
    """Rank r solves its own instance of the config: same shapes and distributions, seed + 1000 r."""
    Pb = W.CONFIGS[config]()
    if rank:
        Pb = GENERATORS[config](seed=Pb.seed + 1000 * rank)
    return Pb


def max_over_ranks(x, world, device):
    """The slowest rank's time (all_reduce MAX of one scalar; the only collective the bench uses)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(world, steps, t_ms):
    """Whole-job solves/s: every rank completed `steps` solves within the max-over-ranks time."""
    return world * steps / (t_ms / 1e3)


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_0907_4631_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    P.build()
    dev = torch.device("cuda", local)

    # replica inputs: same shapes/distributions, seed offset by rank (independent problems)
    Pb = replica_problem(args.config, rank)
    u = [torch.from_numpy(x).to(dev) for x in Pb.u]
    stream = torch.cuda.current_stream(dev)
    ctx = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1), stream=stream,
                    options={k: int(v) for k, v in (x.split("=") for x in args.option)})
    if Pb.stencil is not None:
        S = P.Stencil.of(Pb.stencil)
        solve = lambda **kw: ctx.solve_stencil(Pb.t, S, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric,
                                               m_init=Pb.m_init, **kw)
        path = "stencil"
        h2d_A = 0
    else:
        A = tuple(torch.from_numpy(a).to(dev) for a in Pb.csr)
        solve = lambda **kw: ctx.solve_csr(Pb.t, A, u, out=w, tol=Pb.tol, symmetric=Pb.symmetric,
                                           m_init=Pb.m_init, **kw)
        path = "csr"
        h2d_A = sum(a.nbytes for a in Pb.csr)
    w = torch.empty(Pb.n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2

    # the first (cold) solve of a fresh context, reported separately (module load, first launches)
    torch.cuda.synchronize()
    ec0, ec1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ec0.record(stream)
    _, st = solve()
    ec1.record(stream)
    torch.cuda.synchronize()
    cold_ms = ec0.elapsed_time(ec1)
    for _ in range(max(args.warmup, 3)):
        _, st = solve()
    torch.cuda.synchronize()

    def timed(profile):
        """K solves; device time from CUDA events on the solve stream around each solve (L2 flushed
        between steps, outside the events).  Returns (max-over-ranks ms, last stats, clocks)."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        ctx.reset_profile()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                _, st_ = solve(profile=profile)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), world, dev)
        return ms, st_, clk.summary()

    # ---- timed region 1: the headline (no per-kernel instrumentation: kernels chain with PDL)
    t_max, st, clocks = timed(0)
    value = aggregate_rate(world, args.steps, t_max)
    # ---- timed region 2: same steps with per-kernel CUDA events (roofline of the dominant kernel)
    t_prof, st2, clocks2 = timed(1)
    prof = ctx.profile()

    # ---- end to end through the host-buffer C-ABI entry point (pinned host memory)
    hu = [torch.from_numpy(x).pin_memory().numpy() for x in Pb.u]
    hw = torch.empty(Pb.n, dtype=torch.float64).pin_memory().numpy()
    if path == "csr":
        hA = tuple(torch.from_numpy(a).pin_memory().numpy() for a in Pb.csr)
        ctx.reserve_host_csr(len(Pb.csr[1]))
        e2e_solve = lambda: ctx.solve_csr_host(Pb.t, hA, hu, hw, tol=Pb.tol, symmetric=Pb.symmetric, m_init=Pb.m_init)
    else:
        e2e_solve = lambda: ctx.solve_stencil_host(Pb.t, S, hu, hw, tol=Pb.tol, symmetric=Pb.symmetric,
                                                   m_init=Pb.m_init)
    e2e_solve()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = 0.0
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_solve()
        b.record(stream)
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    e2e_ms = max_over_ranks(e2e_ms, world, dev)
    e2e_val = aggregate_rate(world, args.steps, e2e_ms)
    h2d = sum(x.nbytes for x in Pb.u) + h2d_A
    d2h = Pb.n * 8

    # ---- roofline of the dominant kernel class
    peak, peak_src = measured_peak_hbm()
    classes = {"spmv_dot": ("ms_spmv_dot", "bytes_spmv_dot", "n_spmv_dot"),
               "orth_update": ("ms_orth", "bytes_orth", "n_orth"),
               "combine": ("ms_combine", "bytes_combine", "n_combine")}
    dom = max(classes, key=lambda k: prof[classes[k][0]])
    ms_k, by_k, n_k = (prof[x] for x in classes[dom])
    achieved = (by_k / 1e9) / (ms_k / 1e3) if ms_k > 0 else 0.0
    krylov_ms = prof["ms_spmv_dot"] + prof["ms_orth"]
    krylov_bytes = prof["bytes_spmv_dot"] + prof["bytes_orth"]
    arnoldi_gbs = (krylov_bytes / 1e9) / (krylov_ms / 1e3) if krylov_ms > 0 else 0.0
    solve_bytes = (prof["bytes_spmv_dot"] + prof["bytes_orth"] + prof["bytes_combine"] + prof["bytes_other"]) / args.steps
    tr = load_traffic(args.config)
    traffic = None
    if tr and tr.get("kernel_class") == dom:
        traffic = tr.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom,
                "algorithmic_bytes_per_launch": by_k / max(n_k, 1), "avg_launch_us": 1e3 * ms_k / max(n_k, 1),
                "peak_source": peak_src}

    # ---- Arnoldi/Lanczos-step microbenchmark: normalised seed u0, extend to m = 30
    #      in the context workspace (no export, no exponential, no controller); algorithmic bytes
    #      sum_j B_SpMV + 8n(2j+3) (Arnoldi) or B_SpMV + 32n (Lanczos) over CUDA-event time
    mb = None
    if rank == 0:
        mk = min(30, Pb.m_max)
        op = S if path == "stencil" else A
        for _ in range(2):
            ctx.krylov(op, u[0], mk, symmetric=Pb.symmetric, build_only=True)
        times = []
        for _ in range(5):
            flush.zero_()
            a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            _, _, kb, _, _ = ctx.krylov(op, u[0], mk, symmetric=Pb.symmetric, build_only=True)
            b0.record(stream)
            torch.cuda.synchronize()
            times.append(a0.elapsed_time(b0))
        ms_mb = statistics.median(times)
        n = Pb.n
        b_spmv = 16.0 * n if path == "stencil" else 12.0 * len(Pb.csr[1]) + 4.0 * (n + 1) + 16.0 * n
        by = sum(b_spmv + 8.0 * n * (4.0 if Pb.symmetric else 2.0 * j + 3.0) for j in range(kb))
        mb = {"m": kb, "ms": ms_mb, "algorithmic_gb": by / 1e9, "achieved_gbs": by / 1e6 / ms_mb,
              "frac_of_measured": by / 1e6 / ms_mb / peak, "frac_of_8000": by / 1e6 / ms_mb / 8000.0,
              "note": "seed u0, one extension k = 0 -> m in one call (plus the seed normalisation"
                      + ("; CSR: + the analysis pass" if path == "csr" else "") + "), L2 flushed before each"}

    if rank == 0:
        cpu = cpu_baseline(Pb) if not args.no_cpu_baseline else None
        launches_total = prof["launches"]
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, Pb, path, world),
            "e2e": {"value": e2e_val, "unit": "solves/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_total,
            "roofline": roofline,
            # whole solve: algorithmic bytes of every n-sized pass of one solve (the profiled region's
            # per-class byte counts) over the UN-instrumented ms_per_step
            "solve_algorithmic_gbs": solve_bytes / 1e6 / (t_max / args.steps),
            "solve_frac_of_measured": solve_bytes / 1e6 / (t_max / args.steps) / peak,
            "arnoldi_step": {"achieved_gbs": arnoldi_gbs, "frac_of_8000": arnoldi_gbs / 8000.0,
                             "frac_of_measured": arnoldi_gbs / peak,
                             "ms_per_solve": krylov_ms / args.steps},
            "arnoldi_microbench": mb,
            "cold_solve_ms": cold_ms,
            "profiled_region": {"ms_per_step": t_prof / args.steps, "value": aggregate_rate(world, args.steps, t_prof),
                                "note": "second timed region with CUDA events around every kernel "
                                        "(source of roofline / arnoldi_step / profile_ms_per_solve)",
                                "clocks": clocks2},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "stats": {"nsteps": st.nsteps, "nreject": st.nreject, "nspmv": st.nspmv, "nexpm": st.nexpm,
                      "m_last": st.m_last, "m_peak": st.m_peak},
            "profile_ms_per_solve": {k: prof[k] / args.steps for k in
                                     ("ms_spmv_dot", "ms_orth", "ms_expm", "ms_combine", "ms_other")},
        }
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(DESCR))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--option", action="append", default=[],
                    help="kernel-path option name=value (phipm_set_option; A/B measurements, default: none)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
