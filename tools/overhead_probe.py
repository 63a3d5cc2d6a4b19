"""Probe: solve time with and without per-kernel profiling (config 2, short run)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2409_05572_b200 import load, workloads as W

L = load()
w = W.config2("fix")
w.cfg["max_iters"] = int(sys.argv[1]) if len(sys.argv) > 1 else 40
a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
a.norm_est()
for prof in (0, 1, 0, 1):
    t0 = time.perf_counter()
    r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, ext=L.solve_ext(profile=prof), **w.cfg)
    t1 = time.perf_counter()
    ks = r.kernel_stats()
    busy = sum(v["ms"] for v in ks.values())
    print(f"profile={prof} iters={r.iterations} lib_seconds={r.seconds:.3f} wall={t1 - t0:.3f} "
          f"profiled_kernel_ms={busy:.1f} per_iter_ms={1e3 * r.seconds / r.iterations:.2f}", flush=True)
