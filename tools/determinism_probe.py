"""Reproducibility probe: the config-5 reduced-lattice solve (side 256, nev 32)
repeated in one process, before and after other solves, with the device's last
convergence record compared against the host recomputation of the returned pairs.
Prints one JSON line per run; all runs must be bit-identical."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_05572_b200 import load  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402

L = load()
w5 = W.config5(side=256, nev=32, n_ex=48)
full = W.full_from_lower(w5.n, w5.row_ptr, w5.col, w5.val)


def run5(tag):
    a = L.from_csr(w5.n, w5.row_ptr, w5.col, w5.val)
    r = L.solve(a, "lobpcg", strategy=L.strategy_config("fix"), x0=w5.x0, n_ev=32, n_ex=48, tol=1e-8, max_iters=400)
    v, lam = r.vectors, np.asarray(r.values)
    na = a.norm_est()
    crit = np.linalg.norm(full @ v - v * lam, axis=0) / (na * np.linalg.norm(v, axis=0) * (1 + np.abs(lam) / na))
    h = hashlib.sha256(np.asarray(r.values).tobytes() + np.asarray([x["r_overall"] for x in r.history]).tobytes())
    print(json.dumps({"tag": tag, "status": r.status, "iters": r.iterations, "hash": h.hexdigest()[:16],
                      "dev_r_last": r.history[-1]["r_overall"], "host_max": float(crit.max()),
                      "argmax": int(crit.argmax()), "spec": os.environ.get("BLOCKEIG_NO_SPEC", "")}), flush=True)


run5("first")
run5("second")
w2 = W.config2("fix")
a2 = L.from_csr(w2.n, w2.row_ptr, w2.col, w2.val)
r2 = L.solve(a2, "lobpcg", strategy=L.strategy_config("fix"), x0=w2.x0, **w2.cfg)
print(json.dumps({"tag": "config2", "iters": r2.iterations}), flush=True)
run5("after config 2")
w1 = W.config5(side=128, nev=16, n_ex=24)
L.solve(L.from_csr(w1.n, w1.row_ptr, w1.col, w1.val), "lobpcg", strategy=L.strategy_config("fix"), x0=w1.x0,
        n_ev=16, n_ex=24, tol=1e-8, max_iters=400)
run5("after side 128")
run5("last")
