"""Full-size BASELINE configurations on the B200 against the oracle's recorded
trajectories (tests/golden/oracle_<workload>[_itN].json, written by
tools/run_config.py --impl oracle --save on the CPU; the oracle is test
infrastructure and is not run here).

Bar (BASELINE.json north_star): eigenvalues within 1e-9 relative of the
oracle's, every returned residual below tolerance, block-size trajectory and
iteration count equal except where rounding flips a threshold decision.
Size-independent checks back this up where the oracle cannot finish (configs
3-5): orthonormality, the residual criterion, and closed-form spectra.
"""
import json
import os

import numpy as np
import pytest

from paper_2409_05572_b200 import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture(name):
    path = os.path.join(GOLDEN, f"oracle_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"no oracle fixture {path}")
    with open(path) as f:
        return json.load(f)


def run(product, w, **over):
    a = product.from_csr(w.n, w.row_ptr, w.col, w.val)
    cfg = dict(w.cfg, **over)
    ext = product.solve_ext(**w.ext) if w.ext else None
    return a, product.solve(a, w.solver, strategy=product.strategy_config(w.strategy), x0=w.x0, ext=ext, **cfg)


def events(hist):
    return [(h["n_now"], h["event"]) for h in hist]


def trajectory_report(got, ref):
    """positions where the block width n_now differs, and the largest lock-count
    difference.  Lock events (soft locking of converged pairs) are threshold
    decisions on per-pair residuals (rr.cpp:29-36) and flip with rounding once a
    pair sits at tol; each flip is reported and bounded by the callers."""
    n = min(len(got), len(ref))
    width = [i for i in range(n) if got[i]["n_now"] != ref[i]["n_now"]]
    dlock = max((abs(got[i]["lock_count"] - ref[i]["lock_count"]) for i in range(n)), default=0)
    return width, dlock


def check_block(product, a, w, res, tol_mult=1.0):
    """residual criterion of the reference (rr.cpp:29-33) on the returned pairs,
    recomputed on the host in fp64, plus orthonormality"""
    from scipy.sparse import csr_matrix  # noqa: F401 (scipy present in the image)
    full = W.full_from_lower(w.n, w.row_ptr, w.col, w.val)
    v, lam = res.vectors, np.asarray(res.values)
    sgn = -1.0 if w.ext.get("which") == 1 else 1.0
    na = a.norm_est()
    r = full @ v - v * lam
    rn = np.linalg.norm(r, axis=0)
    vn = np.linalg.norm(v, axis=0)
    crit = rn / (na * vn + vn * np.abs(sgn * lam))
    assert crit.max() <= tol_mult * w.cfg["tol"], crit.max()
    g = v.conj().T @ v
    assert np.abs(g - np.eye(len(lam))).max() < 1e-10
    return crit


def test_config1_matches_oracle_trajectory(product):
    w = W.config1()
    ref = fixture(w.name)
    assert ref["matrix_sha256"] == W.sha256(w.row_ptr, w.col, w.val)
    assert ref["x0_sha256"] == W.sha256(w.x0)
    a, res = run(product, w)
    assert res.status == ref["status"] == 0
    np.testing.assert_allclose(res.values, ref["values"], rtol=1e-9)
    np.testing.assert_allclose(res.values, W.lap2d_eigs(100, 100, 20), rtol=1e-9)
    flips, dlock = trajectory_report(res.history, ref["history"])
    assert abs(res.iterations - ref["iterations"]) <= max(2, ref["iterations"] // 100), \
        (res.iterations, ref["iterations"], flips[:5])
    assert len(flips) <= 0.02 * ref["iterations"], flips[:10]
    assert dlock <= 2
    check_block(product, a, w, res)


@pytest.mark.parametrize("strategy,n_ex", [("fix", 96), ("slope", 96), ("slopek", 96), ("none", 96), ("none", 64)])
def test_config2_matches_oracle_trajectory(product, strategy, n_ex):
    # BASELINE configs[1]: each strategy run in turn against the fixed width
    # (none also at the stated width 64); fixtures are full oracle runs
    w = W.config2(strategy, n_ex=n_ex)
    ref = fixture(w.name)
    assert ref["matrix_sha256"] == W.sha256(w.row_ptr, w.col, w.val)
    assert ref["x0_sha256"] == W.sha256(w.x0)
    a, res = run(product, w)
    assert res.status == ref["status"] == 0
    np.testing.assert_allclose(res.values, ref["values"], rtol=1e-9)
    np.testing.assert_allclose(res.values, W.lap3d_eigs(64, 64), rtol=1e-9 if n_ex > 64 else 1e-8)
    flips, dlock = trajectory_report(res.history, ref["history"])
    # the last pairs cross tol with residual histories that differ at the 1e-4
    # relative level late in the run (FP64 summation order in every contraction),
    # so the final converged-prefix decisions land within a few iterations
    # (observed 215-220 across kernel revisions vs the oracle's 219)
    assert abs(res.iterations - ref["iterations"]) <= max(3, ref["iterations"] // 40), \
        (res.iterations, ref["iterations"], flips[:5])
    assert len(flips) <= 0.05 * ref["iterations"], flips[:10]
    assert dlock <= 5, dlock
    check_block(product, a, w, res)


@pytest.mark.parametrize("name,make", [
    ("cfg3_clustered_1000000_lobpcg_it3", lambda: W.config3("lobpcg")),
    ("cfg3_clustered_1000000_si_it3", lambda: W.config3("si")),
    ("cfg4_anderson_96_lobpcg_it3", lambda: W.config4()),
])
def test_large_configs_prefix_match_oracle(product, name, make):
    """configs 3/4: the oracle needs minutes per iteration at these sizes, so its
    first 3 iterations are the fixture: same inputs (hashes), same trajectory,
    same residual history and Ritz values to rounding"""
    ref = fixture(name)
    w = make()
    assert ref["matrix_sha256"] == W.sha256(w.row_ptr, w.col, w.val)
    assert ref["x0_sha256"] == W.sha256(w.x0)
    _, res = run(product, w, max_iters=3)
    assert res.status == ref["status"]
    assert events(res.history) == events(ref["history"])
    got_r = np.array([h["r_overall"] for h in res.history])
    ref_r = np.array([h["r_overall"] for h in ref["history"]])
    np.testing.assert_allclose(got_r, ref_r, rtol=1e-6)
    np.testing.assert_allclose(res.values, ref["values"], rtol=1e-9)


def test_config5_band_and_residuals(product):
    """config 5's operator on a reduced lattice (side 256, same flux 1/64, so the
    same lowest Landau band: degenerate to ~6e-14 at 0.0969748)
    for test run time: every returned value must sit in the band.  The full
    1024^2 / nev 256 run is measured by tools/run_config.py --config 5
    (profiles/)."""
    w = W.config5(side=256, nev=32, n_ex=48)
    a, res = run(product, w, max_iters=400)
    assert res.status == 0, res.status
    np.testing.assert_allclose(res.values, 0.0969748, atol=2e-7)
    check_block(product, a, w, res)
