"""Device residual criterion vs the host recomputation on the returned pairs
(config 5 reduced lattice): the last record's r_overall is the device's max over
the n_ev pairs of ||A v - lam v|| / ((||A|| + |lam|) ||v||); the host recomputes
it from the returned vectors with scipy CSR."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_05572_b200 import blockeig as B  # noqa: E402
from paper_2409_05572_b200 import load  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402

side = int(os.environ.get("SIDE", 256))
L = load()
w = W.config5(side=side, nev=32, n_ex=48)
a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
res = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, n_ev=32, n_ex=48, tol=1e-8, max_iters=400)
full = W.full_from_lower(w.n, w.row_ptr, w.col, w.val)
v, lam = res.vectors, np.asarray(res.values)
na = a.norm_est()
rn = np.linalg.norm(full @ v - v * lam, axis=0)
vn = np.linalg.norm(v, axis=0)
crit = rn / (na * vn + vn * np.abs(lam))
print(json.dumps({"z3m": os.environ.get("BK_Z3M", "1"), "status": res.status, "iters": res.iterations,
                  "device_r_overall_last": res.history[-1]["r_overall"], "host_max": float(crit.max()),
                  "host_argmax": int(crit.argmax()), "norm_est": na,
                  "orth": float(np.abs(v.conj().T @ v - np.eye(32)).max()),
                  "vals_spread": float(lam.max() - lam.min()), "host_crit": [float(x) for x in crit]}))
