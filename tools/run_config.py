"""Run one BASELINE configuration through the product (GPU) or the oracle (CPU).

    python tools/run_config.py --config 3 --solver lobpcg --impl product --max_iters 200
    python tools/run_config.py --config 4 --impl oracle --max_iters 3 --save

Prints one JSON summary (status, iterations, seconds, values head, n_now
trajectory run-length encoding, kernel stats for the product).  With --save
the oracle's history is written to tests/golden/oracle_<name>[_it<N>].json,
the trajectory fixture the GPU parity tests compare against.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2409_05572_b200 import blockeig as B  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402


def workload(args):
    c = args.config
    if c == "1":
        w = W.config1()
    elif c == "2":
        w = W.config2(args.strategy, n_ex=args.n_ex or 96)
    elif c == "3":
        w = W.config3(args.solver or "lobpcg", n=args.n or 1_000_000)
    elif c == "4":
        w = W.config4(side=args.side or 96)
    elif c == "5":
        side = args.side or 1024
        if args.nev:  # reduced lattice runs (tests): nev and n_ex given
            w = W.config5(side=side, nev=args.nev, n_ex=args.n_ex or (3 * args.nev) // 2)
        else:
            w = W.config5(side=side)
    else:
        raise SystemExit(f"unknown config {c}")
    if args.strategy and c != "2":
        w.strategy = args.strategy
    if args.max_iters:
        w.cfg["max_iters"] = args.max_iters
    return w


def rle(seq):
    out = []
    for x in seq:
        if out and out[-1][0] == x:
            out[-1][1] += 1
        else:
            out.append([x, 1])
    return out


def history_rows(r):
    return [{k: h[k] for k in ("iteration", "r_overall", "n_now", "event", "lock_count", "rr_dim",
                               "spmv_cols", "ortho_flops")} for h in r.history]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--solver", default=None)
    ap.add_argument("--strategy", default=None)
    ap.add_argument("--impl", default="product", choices=["product", "oracle"])
    ap.add_argument("--n_ex", type=int, default=0)
    ap.add_argument("--nev", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--side", type=int, default=0)
    ap.add_argument("--max_iters", type=int, default=0)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--save", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.strategy is None and args.config == "2":
        args.strategy = "fix"
    t0 = time.time()
    w = workload(args)
    tgen = time.time() - t0
    if args.impl == "product":
        from paper_2409_05572_b200 import LIB_PATH
        lib = B.Library(LIB_PATH)
    else:
        lib = B.Library(os.path.join(ROOT, "oracle", "_build", "liborc_blockeig.so"))
    a = lib.from_csr(w.n, w.row_ptr, w.col, w.val)
    ext = lib.solve_ext(**w.ext, profile=1 if args.profile else 0) if args.impl == "product" \
        else lib.solve_ext(**w.ext)
    t0 = time.time()
    r = lib.solve(a, w.solver, strategy=lib.strategy_config(w.strategy), x0=w.x0, ext=ext, **w.cfg)
    secs = time.time() - t0
    vals = np.asarray(r.values)
    out = {
        "workload": w.name, "impl": args.impl, "n": w.n, "nnz_full": w.nnz_full,
        "status": r.status, "iterations": r.iterations, "seconds": secs, "gen_seconds": tgen,
        "threads": os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())),
        "values_head": list(map(float, vals[:4])), "values_tail": list(map(float, vals[-4:])),
        "n_now_rle": rle([h["n_now"] for h in r.history]),
        "final_r": r.history[-1]["r_overall"] if r.history else None,
        "matrix_sha256": W.sha256(w.row_ptr, w.col, w.val),
        "x0_sha256": W.sha256(w.x0) if w.x0 is not None else None,
    }
    if args.impl == "product":
        try:
            out["lib_seconds"] = r.seconds
            out["kernel_stats"] = {k: [s["launches"], round(s["ms"], 3), s["bytes"], s["flops"]]
                                   for k, s in r.kernel_stats().items()}
        except Exception as e:  # profile off
            out["kernel_stats_error"] = str(e)
    print(json.dumps(out))
    if args.save or args.out:
        mg = r.margins
        full = dict(out, values=list(map(float, vals)), history=history_rows(r),
                    margins=[[None if np.isnan(x) else float(x) for x in row] for row in mg])
        suffix = f"_it{args.max_iters}" if args.max_iters else ""
        path = args.out or os.path.join(ROOT, "tests", "golden", f"oracle_{w.name}{suffix}.json")
        with open(path, "w") as f:
            json.dump(full, f, indent=0)
        print(path)


if __name__ == "__main__":
    main()
