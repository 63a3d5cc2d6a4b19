#!/usr/bin/env python3
"""Benchmark: seconds to nev converged eigenpairs on one B200 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] — 3D 7-point Dirichlet Laplacian 64^3
(n = 262,144), LOBPCG for the 64 smallest eigenpairs with the Jacobi (diagonal)
preconditioner, X0 ~ N(0,1) seed 1, tol 1e-8, shrink-and-expand strategy `fix`
at the reference defaults n_ex = 96 / n_es = 69.
One step = one complete solve through the drop-in C ABI (beig_solve_ex).

  value  device-timed seconds per solve with the matrix already resident
         (handle warmed: full CSR uploaded, norm estimate cached); CUDA events
         on the host-synchronous ABI call.
  e2e    the same solve from HOST buffers: beig_matrix_from_csr + beig_solve_ex
         (x0 from host) + value/vector copy-out, wall clock, every step.
  roofline  the dominant kernel class over the timed region, from the
         library's live CUDA-event per-kernel statistics (ext->profile = 1).
  cpu_baseline  the CPU oracle (a port of the reference's algorithm) on a
         bounded sample (first 1 and 2 iterations), extrapolated to the solve.

--impl reference times that oracle alone (all host threads) on the same
workload and prints the same metric (the reference itself cannot be built
here: Eigen3 is absent).  N > 1: replicas only (the path does
not shard), max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2409_05572_b200 import blockeig as B  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402

METRIC = "s to nev converged eigenpairs (1 B200); SpMM GB/s & Gram TFLOP/s vs roofline"
UNIT = "s"
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liborc_blockeig.so")
# iteration count of the full CPU-oracle run of this workload (tests/golden/oracle_*.json);
# used only to extrapolate the bounded CPU sample to a time-to-solution
FALLBACK_ITERS = 217


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp64_peak():
    """Measured FP64 DMMA/cuBLAS DGEMM peak (profiles/r01_fp64_peaks.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")) as f:
            return float(json.load(f)["dgemm_tflops_burst"]), "measured cuBLAS DGEMM 8192^3 (profiles/r01_fp64_peaks.json)"
    except (OSError, KeyError):
        return 35.5, "fallback 35.5 TF/s"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self):
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", os.environ.get("LOCAL_RANK", "0")],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local, dist


def reduce_max(dist, x):
    if dist is None:
        return x
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def count_launches(solve_once):
    """Kernel launches of one solve, counted by CUPTI (torch.profiler) — every
    kernel of libblockeig_b200.so (namespace bk::), not a self-reported count.
    Run once after the timed region (the profiler perturbs timing)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    try:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            solve_once()
            torch.cuda.synchronize()
    except Exception:  # CUPTI unavailable (e.g. under ncu)
        return None, {}
    names = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and "bk::" in e.name:
            short = e.name.split("(")[0].replace("void ", "").replace("bk::(anonymous namespace)::", "")
            names[short] = names.get(short, 0) + 1
    return sum(names.values()), dict(sorted(names.items(), key=lambda kv: -kv[1]))


def ncu_traffic(kernel):
    """DRAM traffic per launch of the dominant kernel class from the committed ncu
    captures (tools/ncu_full_summary.py): the whole-solve per-launch DRAM capture
    (profiles/*_ncu_dram_all.json, same launches as the class statistics) first,
    else the steady-state --set full sample (profiles/*_ncu_full.json)."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_dram_all.json")), reverse=True) + \
        sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full.json")), reverse=True)
    for path in paths:
        try:
            with open(path) as f:
                d = json.load(f)
            k = d.get("classes", {}).get(kernel)
            if k and k.get("dram_bytes_per_launch"):
                return k["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
        except (OSError, ValueError):
            continue
    return None, None


def oracle_sample(w, threads):
    """CPU oracle on the first 1 and 2 iterations; extrapolate to the solve."""
    L = B.Library(ORACLE_SO)
    L.lib.orc_set_threads.argtypes = [B.C.c_int]
    L.lib.orc_set_threads(threads)
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    a.norm_est()
    times = {}
    for iters in (1, 2):
        cfg = dict(w.cfg)
        cfg["max_iters"] = iters
        t0 = time.perf_counter()
        L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, ext=L.solve_ext(**w.ext), **cfg)
        times[iters] = time.perf_counter() - t0
    per_iter = max(times[2] - times[1], 0.0)
    golden = os.path.join(ROOT, "tests", "golden", f"oracle_{w.name}.json")
    iters_total = FALLBACK_ITERS
    if os.path.exists(golden):
        with open(golden) as f:
            iters_total = int(json.load(f)["iterations"])
    est = times[1] + (iters_total - 1) * per_iter
    return est, times, per_iter, iters_total


def run_reference(args, world, rank, dist):
    """--impl reference: the CPU oracle (port of the reference algorithm), all host threads."""
    if rank != 0:
        return
    w = W.config2(args.strategy, n_ex=96, side=args.side)
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        est, times, per_iter, iters_total = oracle_sample(w, threads)
        if i >= args.warmup:
            vals.append(est)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": w.n, "nev": 64, "n_ex": 96, "n_es": 69, "tol": 1e-8,
                   "solver": "lobpcg", "strategy": "fix", "precond": "diagonal"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"oracle LOBPCG first 1 and 2 iterations ({times[1]:.1f}s, {times[2]:.1f}s); "
                                   f"{per_iter:.2f}s/iteration x {iters_total} oracle iterations, extrapolated"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="fix")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    # lattice side of the workload (64 = BASELINE configs[1]); smaller only for tests
    ap.add_argument("--side", type=int, default=64)
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
        if dist is not None:
            dist.destroy_process_group()
        return

    import torch
    from paper_2409_05572_b200 import load
    torch.cuda.set_device(local)
    L = load()
    w = W.config2(args.strategy, n_ex=96, side=args.side)
    cfg = dict(w.cfg)
    strat = L.strategy_config(w.strategy)
    ext = L.solve_ext(device=local, profile=1)
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    a.norm_est()

    def solve_once():
        return L.solve(a, w.solver, strategy=strat, x0=w.x0, ext=ext, **cfg)

    for _ in range(args.warmup):
        res = solve_once()
    # L2 note: every solve streams S/AS blocks of 0.7 GB each (> 126 MB L2)
    sampler = ClockSampler()
    barrier(dist)
    torch.cuda.synchronize()
    sampler.start()
    times, stats, iters = [], [], []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res = solve_once()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        stats.append(res.kernel_stats())
        iters.append(res.iterations)
    barrier(dist)
    clocks = sampler.stop()
    t_step = reduce_max(dist, float(np.mean(times)))
    launches_per_solve, launch_names = count_launches(solve_once)
    vals = res.values
    ref = W.lap3d_eigs(args.side, 64)
    max_rel = float(np.max(np.abs(vals - ref) / ref))

    # ---- e2e through the public API from host buffers
    e2e = []
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a2 = L.from_csr(w.n, w.row_ptr, w.col, w.val)
        r2 = L.solve(a2, w.solver, strategy=strat, x0=w.x0, ext=L.solve_ext(device=local), **cfg)
        _ = r2.values, r2.vectors
        e2e.append(time.perf_counter() - t0)
        del a2, r2
    e2e_t = reduce_max(dist, float(np.mean(e2e)))
    nnz_full = w.nnz_full
    h2d = 4 * (w.n + 1) + 12 * nnz_full + 8 * w.n * cfg["n_ex"]
    d2h = 8 * 64 + 8 * w.n * 64 + 48 * int(np.mean(iters))

    # ---- roofline of the dominant kernel class over the timed region
    agg = {}
    for s in stats:
        for k, v in s.items():
            a_ = agg.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0})
            for f in a_:
                a_[f] += v[f]
    # the dominant roofline-bound class (HBM: spmm / residual; FP64 tensor: gram /
    # gemm); the latency-bound projected eigensolver is reported beside it
    top = max((k for k in ("spmm", "gram", "gemm", "residual") if agg.get(k, {}).get("launches")),
              key=lambda k: agg[k]["ms"])
    total_ms = sum(v["ms"] for v in agg.values())
    peaks = measured_peaks()
    fp64, fp64_src = fp64_peak()
    kernels = {}
    for k, v in agg.items():
        if not v["launches"]:
            continue
        kernels[k] = {"launches_per_solve": v["launches"] / len(stats), "ms_per_solve": v["ms"] / len(stats),
                      "share_of_step": v["ms"] / len(stats) / (t_step * 1e3),
                      "gbs": v["bytes"] / v["ms"] / 1e6 if v["ms"] else None,
                      "tflops": v["flops"] / v["ms"] / 1e9 if v["ms"] else None}

    def roof(k):
        v = agg[k]
        if k in ("spmm", "residual"):
            ach = v["bytes"] / v["ms"] / 1e6
            pk = float(peaks.get("hbm_gbs", 6650.0))
            return {"kernel": k, "bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk,
                    "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
        if k in ("gram", "gemm"):
            ach = v["flops"] / v["ms"] / 1e9
            return {"kernel": k, "bound": "tensor", "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
                    "frac": ach / fp64, "traffic": None, "peak_source": fp64_src}
        # latency-bound single-CTA kernels: report time per launch, no roofline fraction
        return {"kernel": k, "bound": "latency", "achieved": v["ms"] / v["launches"], "peak": None,
                "unit": "ms/launch", "frac": None, "traffic": None}

    roofline = roof(top)
    roofline["share_of_step"] = agg[top]["ms"] / len(stats) / (t_step * 1e3)
    traffic, traffic_src = ncu_traffic(top)
    if traffic:
        roofline["traffic"] = traffic
        roofline["traffic_source"] = traffic_src
        roofline["algorithmic_bytes_per_launch"] = agg[top]["bytes"] / agg[top]["launches"]
    roofline["by_kernel"] = {k: roof(k) for k in ("spmm", "gram", "gemm") if agg[k]["launches"]}
    if agg.get("syev", {}).get("launches"):
        roofline["latency_bound"] = dict(roof("syev"), share_of_step=agg["syev"]["ms"] / len(stats) / (t_step * 1e3))

    line = {
        "metric": METRIC, "value": t_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE.json configs[1])",
        "config": {"workload": w.name, "n": w.n, "nnz_full": nnz_full, "nev": 64, "n_ex": 96, "n_es": 69,
                   "tol": 1e-8, "solver": "lobpcg", "strategy": w.strategy, "precond": "diagonal",
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": "inputs > L2 (S/AS blocks 0.7 GB each)"},
        "iterations": int(np.mean(iters)), "max_rel_err_vs_closed_form": max_rel,
        "clocks": clocks,
        "e2e": {"value": e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        # CUPTI-counted launches of this library's kernels over the K timed solves
        "gpu_launches": int(launches_per_solve * args.steps) if launches_per_solve else
        int(round(sum(v["launches"] for v in agg.values()) / len(stats))) * args.steps,
        "gpu_launches_per_solve": launches_per_solve,
        "launches_by_kernel": launch_names,
        "roofline": roofline, "kernels": kernels,
        # small bookkeeping kernels (copies, transposes, K6 finishes, K4 flags) and
        # launch gaps are not bracketed by timing events (to keep profiling cheap)
        "untimed_ms_per_solve": t_step * 1e3 - total_ms / len(stats),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(ORACLE_SO):
        threads = os.cpu_count() or 1
        est, times1, per_iter, iters_total = oracle_sample(w, threads)
        line["cpu_baseline"] = {
            "value": est, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle LOBPCG first 1 and 2 iterations ({times1[1]:.1f}s, {times1[2]:.1f}s); "
                      f"{per_iter:.2f}s/iteration x {iters_total} iterations, extrapolated"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
