"""Exploration: one config-2 solve on the GPU with per-kernel stats (not the bench)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_2409_05572_b200 import blockeig as B
from paper_2409_05572_b200 import load, workloads as W

strategy = sys.argv[1] if len(sys.argv) > 1 else "fix"
side = int(sys.argv[2]) if len(sys.argv) > 2 else 64
max_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
L = load()
w = W.config2(strategy, side=side)
w.cfg["max_iters"] = max_iters
a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
t0 = time.time()
print("norm", a.norm_est(), time.time() - t0, flush=True)
ext = L.solve_ext(profile=1)
t0 = time.time()
r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, ext=ext, **w.cfg)
t1 = time.time()
print("status", r.status, "iters", r.iterations, "seconds", r.seconds, "wall", t1 - t0)
ks = r.kernel_stats()
for k, v in ks.items():
    if v["launches"]:
        extra = ""
        if v["flops"] and v["ms"]:
            extra += f" {v['flops'] / v['ms'] / 1e9:.2f} TF/s"
        if v["bytes"] and v["ms"]:
            extra += f" {v['bytes'] / v['ms'] / 1e6:.1f} GB/s"
        print(f"{k:9s} n={v['launches']:6d} ms={v['ms']:9.2f} avg={v['ms'] / v['launches']:.4f}{extra}")
print("diag", r.diagnostics)
vals = r.values
ref = W.lap3d_eigs(side, 64)
print("max rel err vs closed form", np.max(np.abs(vals - ref) / ref))
h = r.history
print("events", [(x["iteration"], x["event"], x["n_now"]) for x in h if x["event"] in (1, 2)][:20])
print("rr_dims", [x["rr_dim"] for x in h[:10]], [x["rr_dim"] for x in h[-5:]])
