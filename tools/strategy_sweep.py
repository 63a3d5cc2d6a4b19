"""Config 2 strategy comparison (BASELINE configs[1]: "each of the reference's
adaptive block-size strategies run in turn and compared with the fixed-width
run"; strategy none at the stated width 64, all four at the
reference default n_ex = 96 / n_es = 69) — the reference CLI's `compare`
(proj/tools/blockeig_cli.cpp:314-400) on the B200.

    python tools/strategy_sweep.py [out.md]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_05572_b200 import load, workloads as W  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    L = load()
    rows = []
    base = None
    for strat, n_ex in (("none", 64), ("none", 96), ("fix", 96), ("slope", 96), ("slopek", 96)):
        w = W.config2(strat, n_ex=n_ex)
        a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
        a.norm_est()
        L.solve(a, w.solver, strategy=L.strategy_config(strat), x0=w.x0, **dict(w.cfg, max_iters=3))  # warm
        t0 = time.perf_counter()
        r = L.solve(a, w.solver, strategy=L.strategy_config(strat), x0=w.x0, **w.cfg)
        secs = time.perf_counter() - t0
        ref = W.lap3d_eigs(64, 64)
        err = float(np.max(np.abs(np.asarray(r.values) - ref) / ref))
        wk = r.work
        fx = os.path.join(GOLDEN, f"oracle_{w.name}.json")
        oracle_it = json.load(open(fx))["iterations"] if os.path.exists(fx) else None
        row = {"strategy": strat, "n_ex": n_ex, "status": r.status, "iterations": r.iterations,
               "oracle_iterations": oracle_it, "seconds": secs, "spmv_cols": wk.spmv_cols,
               "ortho_flops": wk.ortho_flops, "rr_flops": wk.rr_flops, "combined_work": wk.combined,
               "max_rel_err": err,
               "shrinks": sum(1 for h in r.history if h["event"] == 2),
               "expands": sum(1 for h in r.history if h["event"] == 1)}
        if strat == "none" and n_ex == 96:
            base = row
        rows.append(row)
        print(json.dumps(row), flush=True)
    lines = ["| strategy | n_ex | status | iterations (oracle) | s | SpMV cols | ortho flops | RR flops | "
             "work vs none@96 | shrink / expand | max rel err |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        rel = r["combined_work"] / base["combined_work"] if base and base["combined_work"] else float("nan")
        lines.append(f"| {r['strategy']} | {r['n_ex']} | {r['status']} | {r['iterations']} "
                     f"({r['oracle_iterations'] if r['oracle_iterations'] is not None else '-'}) | "
                     f"{r['seconds']:.2f} | {r['spmv_cols']} | {r['ortho_flops']:.3g} | {r['rr_flops']:.3g} | "
                     f"{rel:.3f} | {r['shrinks']} / {r['expands']} | {r['max_rel_err']:.1e} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if out:
        with open(out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
