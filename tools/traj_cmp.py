"""Compare a product run's trajectory with an oracle fixture (tests/golden):
prints the (iteration, n_now, event, r_overall) rows where they differ."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05572_b200 import LIB_PATH, blockeig as B, workloads as W  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    w = W.config1() if cfg == "1" else W.config2("fix")
    ref = json.load(open(os.path.join("tests", "golden", f"oracle_{w.name}.json")))
    L = B.Library(LIB_PATH)
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0,
                ext=L.solve_ext(**w.ext) if w.ext else None, **w.cfg)
    g, o = r.history, ref["history"]
    print("iterations", r.iterations, ref["iterations"])
    for i in range(max(len(g), len(o))):
        a_ = g[i] if i < len(g) else None
        b_ = o[i] if i < len(o) else None
        same = a_ and b_ and (a_["n_now"], a_["event"]) == (b_["n_now"], b_["event"])
        if not same or i % 40 == 0:
            fa = f"{a_['n_now']:4d} {a_['event']} {a_['lock_count']:3d} {a_['r_overall']:.6e}" if a_ else "-"
            fb = f"{b_['n_now']:4d} {b_['event']} {b_['lock_count']:3d} {b_['r_overall']:.6e}" if b_ else "-"
            print(i + 1, "  " if same else "**", fa, "|", fb)


if __name__ == "__main__":
    main()
