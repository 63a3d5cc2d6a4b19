"""Run the CPU oracle on a full BASELINE configuration and save its trajectory.

Produces tests/golden/oracle_<name>.json: iteration count, status, eigenvalues
and the per-iteration history (r_overall, n_now, event, lock, rr_dim), used as
the reference trajectory for the GPU parity tests at full config size and as
the iteration count for the CPU-baseline extrapolation in bench.py.
Test infrastructure only (oracle), run here on the CPU (hours for config 2).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_05572_b200 import blockeig as B  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--strategy", default="fix")
    ap.add_argument("--n_ex", type=int, default=96)
    ap.add_argument("--max_iters", type=int, default=0)
    args = ap.parse_args()
    if args.config == "1":
        w = W.config1()
    else:
        w = W.config2(args.strategy, n_ex=args.n_ex)
    if args.max_iters:
        w.cfg["max_iters"] = args.max_iters
    lib = B.Library(os.path.join(ROOT, "oracle", "_build", "liborc_blockeig.so"))
    a = lib.from_csr(w.n, w.row_ptr, w.col, w.val)
    ext = lib.solve_ext(**w.ext)
    t0 = time.time()
    r = lib.solve(a, w.solver, strategy=lib.strategy_config(w.strategy), x0=w.x0, ext=ext, **w.cfg)
    secs = time.time() - t0
    out = {
        "workload": w.name, "status": r.status, "iterations": r.iterations, "seconds": secs,
        "threads": os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())),
        "values": list(map(float, r.values)),
        "matrix_sha256": W.sha256(w.row_ptr, w.col, w.val), "x0_sha256": W.sha256(w.x0),
        "history": [{k: h[k] for k in ("iteration", "r_overall", "n_now", "event", "lock_count", "rr_dim",
                                        "spmv_cols", "ortho_flops")} for h in r.history],
    }
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{w.name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(path, r.status, r.iterations, f"{secs:.1f}s")


if __name__ == "__main__":
    main()
