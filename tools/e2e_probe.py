"""Where the end-to-end time of one config-2 solve from host buffers goes (tuning tool):
matrix import, norm estimate (first solve on a fresh handle), solve from host X0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05572_b200 import load, workloads as W  # noqa: E402

L = load()
w = W.config2("fix")
for rep in range(3):
    t0 = time.perf_counter()
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    t1 = time.perf_counter()
    nrm = a.norm_est()
    t2 = time.perf_counter()
    r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, **w.cfg)
    t3 = time.perf_counter()
    r2 = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, **w.cfg)
    t4 = time.perf_counter()
    print(f"from_csr {t1 - t0:.4f} s  norm_est {t2 - t1:.4f} s  first solve {t3 - t2:.4f} s  "
          f"warm solve {t4 - t3:.4f} s  ({r.iterations} / {r2.iterations} it)  seconds {r.seconds}")
