"""Debug: SD on laplacian1d:100 (test_solvers.cpp scenario) with and without
speculative tails; prints iteration counts and the first trajectory divergence."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05572_b200 import LIB_PATH, blockeig as B  # noqa: E402
from tests.helpers import laplacian_1d  # noqa: E402

L = B.Library(LIB_PATH)
O = B.Library(os.path.join(os.path.dirname(LIB_PATH), "..", "oracle", "_build", "liborc_blockeig.so"))
rp, col, val = laplacian_1d(100)
strat = sys.argv[1] if len(sys.argv) > 1 else "none"
runs = {}
for name, lib in (("product", L), ("oracle", O)):
    a = lib.from_csr(100, rp, col, val)
    r = lib.solve(a, "sd", strategy=lib.strategy_config(strat), n_ev=4, seed=11)
    runs[name] = r
    print(name, os.environ.get("BLOCKEIG_NO_SPEC", "spec"), r.status, r.iterations, r.diagnostics)
g, o = runs["product"].history, runs["oracle"].history
for i in range(min(len(g), len(o))):
    if (g[i]["n_now"], g[i]["event"]) != (o[i]["n_now"], o[i]["event"]) or abs(g[i]["r_overall"] / o[i]["r_overall"] - 1) > 1e-6:
        print("first divergence at", i + 1, g[i], o[i])
        break
