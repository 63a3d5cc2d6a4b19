"""Where config 5's end-to-end time goes beyond the device solve: handle creation
from host CSR, the host norm estimate, the device CSR upload, the solve with x0
and result vectors in host memory (BLOCKEIG_TIMING=1 prints the library's own
setup / run / teardown split).  One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_05572_b200 import load  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402

L = load()
w = W.config5()
out = {"threads_host": os.cpu_count()}
t = time.perf_counter()
a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
out["from_csr_s"] = time.perf_counter() - t
t = time.perf_counter()
out["norm_est"] = a.norm_est()
out["norm_est_s"] = time.perf_counter() - t
t = time.perf_counter()
r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, **w.cfg)
out["solve_s"] = time.perf_counter() - t
out["lib_seconds"] = r.seconds
t = time.perf_counter()
v = r.vectors
out["vectors_getter_s"] = time.perf_counter() - t
out["iterations"] = r.iterations
print(json.dumps(out))
