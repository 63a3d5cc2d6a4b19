"""Full-size run report of one BASELINE configuration on the product, with an
independent a-posteriori check of every returned pair (SURVEY.md §8c plan item 3).

    python tools/check_config.py --config 4 --out profiles/r02_check_cfg4.json

The check recomputes A v - lam v on the host with scipy CSR (the generator's
matrix, not the library's copy) and reports, per pair, the reference criterion
||r|| / ((||A|| + |lam|) ||v||) (proj/src/rr.cpp:29-33) and the north star's
||A v - lam v|| / ||A|| (||v|| = 1), plus the block's orthonormality and, where a
closed form exists, the eigenvalue error.  Config 4 (A^2 operator) also reports
lambda = v^T A v per vector, the eigenvalues of A the A^2 pairs stand for.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402


def make(cfg, solver):
    if cfg == "1":
        return W.config1(), W.lap2d_eigs(100, 100, 20)
    if cfg == "2":
        return W.config2("fix"), W.lap3d_eigs(64, 64)
    if cfg == "3":
        return W.config3(solver or "lobpcg"), None
    if cfg == "4":
        return W.config4(), None
    if cfg == "5":
        return W.config5(), W.magnetic_eigs(1024, 1 / 64, 256)
    raise SystemExit(f"unknown config {cfg}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--solver", default=None)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    w, exact = make(args.config, args.solver)
    L = load()
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    na = a.norm_est()
    ext = L.solve_ext(**w.ext, profile=1)
    t0 = time.time()
    r = L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, ext=ext, **w.cfg)
    secs = time.time() - t0
    lam = np.asarray(r.values)
    v = r.vectors
    full = W.full_from_lower(w.n, w.row_ptr, w.col, w.val)
    t1 = time.time()
    res = full @ v - v * lam[None, :]
    rn = np.linalg.norm(res, axis=0)
    vn = np.linalg.norm(v, axis=0)
    ref_crit = rn / ((na + np.abs(lam)) * vn)
    ns_crit = rn / (na * vn)
    g = v.conj().T @ v
    tol = w.cfg["tol"]
    hist = r.history
    out = {
        "workload": w.name, "n": w.n, "nnz_full": w.nnz_full, "solver": w.solver, "strategy": w.strategy,
        "status": ["converged", "max_iters", "stagnated"][r.status], "iterations": r.iterations,
        "seconds_wall": secs, "seconds_lib": r.seconds, "norm_est": na, "tol": tol,
        "check_seconds": time.time() - t1,
        "ref_criterion": {"max": float(ref_crit.max()), "pairs_above_tol": int((ref_crit > tol).sum())},
        "north_star_criterion": {"max": float(ns_crit.max()), "pairs_above_tol": int((ns_crit > tol).sum()),
                                 "pairs_above_2tol": int((ns_crit > 2 * tol).sum())},
        "orthonormality_max": float(np.abs(g - np.eye(len(lam))).max()),
        "values_head": list(map(float, lam[:4])), "values_tail": list(map(float, lam[-4:])),
        "n_now_events": [[h["iteration"], h["n_now"], h["event"]] for h in hist if h["event"] in (1, 2)][:40],
        "final_r": hist[-1]["r_overall"] if hist else None,
        "kernel_stats": {k: [s["launches"], round(s["ms"], 3)] for k, s in r.kernel_stats().items()},
    }
    if exact is not None:
        out["max_rel_err_vs_closed_form"] = float(np.max(np.abs(lam - exact) / np.abs(exact)))
    if args.config == "4":  # eigenvalues of A behind the A^2 pairs: lambda = v^T A v
        from paper_2409_05572_b200.workloads import anderson, full_from_lower
        rp, c, vals = anderson(96)
        a1 = full_from_lower(w.n, rp, c, vals)
        ray = np.einsum("ij,ij->j", v, a1 @ v) / vn ** 2
        out["rayleigh_A"] = {"min": float(ray.min()), "max": float(ray.max()),
                             "max_abs": float(np.abs(ray).max()),
                             "sq_vs_mu_max_abs_diff": float(np.max(np.abs(ray ** 2 - lam)))}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("workload", "status", "iterations", "seconds_lib", "ref_criterion",
                                          "north_star_criterion", "orthonormality_max")}))


if __name__ == "__main__":
    main()
