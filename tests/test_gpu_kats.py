"""The reference's own known answers run on the PRODUCT (not only on the oracle):
CGS2 keep/drop counts through K4, HL-trick properties, record-for-record
determinism, the acceptance criteria, speculative vs synchronous iterations,
and the work counters (the history contract) against the oracle.

Every call goes through the C ABI (beig_harness_* for K4 / the HL step, the
solver entry points otherwise); the same calls drive the oracle where a
comparison is made.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2409_05572_b200 import blockeig as B
from tests.helpers import laplacian_1d

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def random_block(oracle, rows, cols, seed):
    """the reference's random_block (mt19937_64 + normal_distribution, column-major)"""
    out = np.empty(rows * cols)
    oracle.lib.orc_random_block.argtypes = [B.C.c_int, B.C.c_int, B.C.c_uint64, B.C.POINTER(B.C.c_double)]
    oracle.lib.orc_random_block(rows, cols, seed, out.ctypes.data_as(B.C.POINTER(B.C.c_double)))
    return out.reshape((rows, cols), order="F")


# ---------------------------------------------------------------- K4 (test_kernel.cpp:91-112)
def test_orthonormalize_drops_dependent_columns(product, oracle):
    x = random_block(oracle, 15, 3, 12)
    xx = np.column_stack([x, 2.0 * x[:, 0], x[:, 1] - x[:, 2]])
    for L in (product, oracle):
        q, kept = L.project_orthonormalize(xx)
        assert kept == 3 and q.shape == (15, 3)
        assert np.abs(q.T @ q - np.eye(3)).max() < 1e-12
        # the kept basis spans the original columns
        assert np.abs(q @ (q.T @ xx) - xx).max() < 1e-10


def test_project_orthonormalize_external_block(product, oracle):
    qo, kq = oracle.project_orthonormalize(random_block(oracle, 25, 5, 13))
    assert kq == 5
    w = random_block(oracle, 25, 4, 14)
    for L in (product, oracle):
        q, _ = L.project_orthonormalize(qo)  # the product's own basis of the same span
        o, kept = L.project_orthonormalize(w, q)
        assert kept == 4
        assert np.abs(q.T @ o).max() < 1e-12
        assert np.abs(o.T @ o - np.eye(4)).max() < 1e-12
        # a column already inside span(q) is dropped entirely
        inside = (q[:, 0] + 1e-12 * q[:, 1])[:, None]
        assert L.project_orthonormalize(inside, q)[1] == 0


@pytest.mark.parametrize("n,a,m,dep", [(400, 24, 48, 3), (5000, 69, 138, 5), (20000, 96, 192, 0)])
def test_k4_keep_counts_match_oracle(product, oracle, n, a, m, dep):
    """keep/drop decisions of K4 (block projection + CholQR drop rule + CGS2
    fallback) equal the oracle's column CGS2 on blocks with exactly dependent
    columns, at solver-like shapes"""
    rng = np.random.default_rng(n + a)
    q, _ = oracle.project_orthonormalize(rng.standard_normal((n, m)))
    w = rng.standard_normal((n, a))
    for j in range(dep):  # dependent on earlier columns / on q
        w[:, a - 1 - j] = w[:, j] * 0.5 - 2.0 * w[:, j + 1] + q[:, j]
    got, kg = product.project_orthonormalize(w, q)
    ref, ko = oracle.project_orthonormalize(w, q)
    assert kg == ko == a - dep
    assert np.abs(q.T @ got).max() < 1e-12
    assert np.abs(got.T @ got - np.eye(kg)).max() < 1e-12
    # same subspace as the oracle's basis
    assert np.abs(got - ref @ (ref.T @ got)).max() < 1e-9


# ---------------------------------------------------------------- HL trick (test_solvers.cpp:307-341)
@pytest.fixture(scope="module")
def hl_inputs(oracle):
    s, ks = oracle.project_orthonormalize(random_block(oracle, 20, 12, 5))
    z, kz = oracle.project_orthonormalize(random_block(oracle, 12, 12, 6))
    assert ks == kz == 12
    return s, z


def test_hl_trick_unlocked(product, oracle, hl_inputs):
    s, z = hl_inputs
    n_now = 5
    for L in (product, oracle):
        x, p = L.hl_trick(s, z, n_now)
        assert x.shape[1] == n_now and p.shape[1] == n_now
        assert np.linalg.norm(x - s @ z[:, :n_now]) < 1e-13
        xp = np.column_stack([x, p])
        assert np.linalg.norm(xp.T @ xp - np.eye(2 * n_now)) < 1e-12
        assert np.linalg.norm(xp - s @ (s.T @ xp)) < 1e-12


def test_hl_trick_locked(product, oracle, hl_inputs):
    s, z = hl_inputs
    for L in (product, oracle):
        x, p = L.hl_trick(s, z, 5, 2)
        assert x.shape[1] == 5 and p.shape[1] <= 3
        assert np.linalg.norm(x.T @ p) < 1e-12
    # the same P subspace as the oracle's
    _, pg = product.hl_trick(s, z, 5, 2)
    _, po = oracle.hl_trick(s, z, 5, 2)
    assert pg.shape == po.shape
    assert np.linalg.norm(pg - po @ (po.T @ pg)) < 1e-12


def test_hl_trick_bad_n_now(product, oracle, hl_inputs):
    s, z = hl_inputs
    for L in (product, oracle):
        for bad in (0, 13):
            with pytest.raises(B.BlockeigError) as e:
                L.hl_trick(s, z, bad)
            assert e.value.code == B.ERR_INVALID


# ---------------------------------------------------------------- determinism (test_solvers.cpp:165-185)
def _records(r):
    return [(h["r_overall"], h["n_now"], h["event"], h["lock_count"], h["spmv_cols"], h["ortho_flops"],
             h["rr_dim"]) for h in r.history]


def test_identical_runs_reproduce_record_for_record(product):
    a = product.gen("diag-geom:200,1.05")
    runs = []
    for i in range(2):
        runs.append(product.solve(a, "lobpcg", n_ev=6, seed=7, strategy=product.strategy_config("slopek")))
        if i == 0:  # a different solve in between: device block cache, pooled events
            product.solve(product.gen("laplacian1d:300"), "sd", n_ev=3, seed=2)
    one, two = runs
    assert one.status == two.status
    assert _records(one) == _records(two)  # bit-equal r_overall
    assert np.array_equal(one.values, two.values)
    assert one.work.rr_flops == two.work.rr_flops
    assert np.array_equal(one.vectors, two.vectors)


SPEC_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
from paper_2409_05572_b200 import load
from tests.helpers import laplacian_1d
L = load()
out = {{}}
for solver, strat, spec in [("lobpcg", "fix", "laplacian1d:100"), ("sd", "slopek", "laplacian1d:100"),
                            ("si", "fix", "laplacian1d:100"), ("lobpcg", "slope", "diag-geom:300,1.03"),
                            ("sd", "none", "laplacian1d:100")]:
    a = L.gen(spec)
    r = L.solve(a, solver, n_ev=4, seed=11, strategy=L.strategy_config(strat))
    out[solver + "/" + strat + "/" + spec] = dict(
        status=r.status, values=list(map(float, r.values)),
        hist=[[h["r_overall"], h["n_now"], h["event"], h["lock_count"], h["spmv_cols"], h["ortho_flops"],
               h["rr_dim"]] for h in r.history])
print(json.dumps(out))
"""


def test_speculative_equals_synchronous(product):
    """The default speculative iterations (one host readback per iteration, redone
    from a snapshot when a K4 call drops a column) give the same history and
    values, bit for bit, as BLOCKEIG_NO_SPEC=1 (every K4 decision read back)."""
    outs = []
    for env in ({}, {"BLOCKEIG_NO_SPEC": "1"}):
        r = subprocess.run([sys.executable, "-c", SPEC_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                           env=dict(os.environ, **env), timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    spec, sync = outs
    assert spec.keys() == sync.keys()
    for k in spec:
        assert spec[k] == sync[k], k


WIN_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2409_05572_b200 import load
from paper_2409_05572_b200 import workloads as W
L = load()
side = 42  # 74088 rows: above the 65536-row threshold of the window plan
rp, col, val = W.grid_laplacian((side,) * 3)
n = side ** 3
out = {{}}
for solver, kw in (("lobpcg", dict(n_ev=12, n_ex=20, max_iters=40, precond=1)), ("sd", dict(n_ev=6, n_ex=10, max_iters=25)),
                   ("tracemin", dict(n_ev=6, n_ex=10, max_iters=6))):
    a = L.from_csr(n, rp, col, val)
    r = L.solve(a, solver, seed=5, tol=1e-9, strategy=L.strategy_config("fix"), **kw)
    out[solver] = dict(status=r.status, values=list(map(float, r.values)), windowed=r.diagnostics["spmm_windowed"],
                       hist=[[h["r_overall"], h["n_now"], h["event"], h["lock_count"], h["spmv_cols"]] for h in r.history],
                       vec_sum=float(np.abs(r.vectors).sum()))
print(json.dumps(out))
"""


def test_windowed_spmm_equals_plain_in_solves(product):
    """Solves whose SpMM runs as the window-staged K1w (BLOCKEIG_SPMM_WIN=2: the plan
    is awaited, every launch of >= 8 columns windowed) give the same history, values
    and vectors, bit for bit, as solves on the plain K1 (BLOCKEIG_SPMM_WIN=0)."""
    outs = []
    for mode in ("2", "0"):
        r = subprocess.run([sys.executable, "-c", WIN_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                           env=dict(os.environ, BLOCKEIG_SPMM_WIN=mode), timeout=900, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    win, plain = outs
    for k in win:
        assert win[k]["windowed"] > 0 and plain[k]["windowed"] == 0, (k, win[k]["windowed"], plain[k]["windowed"])
        for f in ("status", "values", "hist", "vec_sum"):
            assert win[k][f] == plain[k][f], (k, f)


# ---------------------------------------------------------------- acceptance (acceptance_test.cpp)
def test_acceptance_solver_oracle(product):
    """acceptance_test.cpp:135-187: laplacian1d:400, n_ev 10, every solver x
    strategy converges (tol 1e-10, TraceMIN 1e-6, seed 1), values within 1e-8 of
    the closed form (TraceMIN: at most 1 % beyond 1e-6)"""
    n, n_ev = 400, 10
    exact = 2 - 2 * np.cos(np.arange(1, n_ev + 1) * np.pi / (n + 1))
    a = product.gen(f"laplacian1d:{n}")
    converged, tm_values, tm_bad = 0, 0, 0
    for solver in ("si", "sd", "lobpcg", "tracemin"):
        for strat in ("none", "fix", "slope", "slopek"):
            tm = solver == "tracemin"
            r = product.solve(a, solver, n_ev=n_ev, tol=1e-6 if tm else 1e-10, seed=1,
                              strategy=product.strategy_config(strat))
            if r.status != B.STATUS_CONVERGED:
                continue
            converged += 1
            rel = np.abs(r.values - exact) / exact
            if tm:
                tm_values += n_ev
                tm_bad += int((rel > 1e-6).sum())
            else:
                assert rel.max() <= 1e-8, (solver, strat, rel.max())
    assert converged == 16
    assert tm_bad <= tm_values // 100


@pytest.mark.parametrize("spec,max_iters", [("diag-geom:500,1.02", 6000), ("laplacian1d:400", 2000)])
def test_acceptance_sizing_saves_work(product, spec, max_iters):
    """acceptance_test.cpp:189-226: LOBPCG n_ev 10, n_ex 20, n_es 15: fix needs at
    most 1.3x the iterations of none, less ortho+RR work, and fix or slopek
    saves >= 10 % of the combined work"""
    a = product.gen(spec)
    res = {}
    for strat in ("none", "fix", "slopek"):
        r = product.solve(a, "lobpcg", n_ev=10, n_ex=20, n_es=15, max_iters=max_iters, seed=1,
                          strategy=product.strategy_config(strat))
        assert r.status == B.STATUS_CONVERGED, (strat, r.status)
        res[strat] = r
    w = {k: v.work for k, v in res.items()}
    assert res["fix"].iterations / res["none"].iterations <= 1.3
    assert w["fix"].ortho_flops + w["fix"].rr_flops < w["none"].ortho_flops + w["none"].rr_flops
    save = max(1 - w["fix"].combined / w["none"].combined, 1 - w["slopek"].combined / w["none"].combined)
    assert save >= 0.10, save


# ---------------------------------------------------------------- work counters = the history contract
def _prefix_equal(g, o):
    """records up to (excluding) the first (n_now, event, lock, rr_dim)
    difference — rr_dim changes when a K4 drop decision flips (SD)"""
    n = 0
    key = ("n_now", "event", "lock_count", "rr_dim")
    for a, b in zip(g, o):
        if tuple(a[k] for k in key) != tuple(b[k] for k in key):
            break
        n += 1
    return n


@pytest.mark.parametrize("solver", ["si", "sd", "lobpcg", "tracemin"])
@pytest.mark.parametrize("strat", ["none", "fix", "slope", "slopek"])
def test_work_counters_match_oracle(product, oracle, solver, strat):
    """spmv_cols, solve_cols, ortho_flops and rr_dim of every history record equal
    the oracle's (solvers.cpp:26-60 formulas) wherever the trajectories agree;
    rr_flops and the combined work too when the whole run agrees"""
    n = 100
    rp, col, val = laplacian_1d(n)
    out = []
    for L in (product, oracle):
        a = L.from_csr(n, rp, col, val)
        out.append(L.solve(a, solver, n_ev=4, seed=11, strategy=L.strategy_config(strat)))
    g, o = out
    hg, ho = g.history, o.history
    k = _prefix_equal(hg, ho)
    assert k >= min(len(hg), len(ho)) // 2, (k, len(hg), len(ho))
    for i in range(k):
        for f in ("iteration", "spmv_cols", "solve_cols", "ortho_flops", "rr_dim", "n_now", "event", "lock_count"):
            assert hg[i][f] == ho[i][f], (i, f, hg[i][f], ho[i][f])
    if k == len(hg) == len(ho):
        assert g.work.spmv_cols == o.work.spmv_cols and g.work.ortho_flops == o.work.ortho_flops
        assert g.work.rr_flops == o.work.rr_flops
        assert g.work.combined == o.work.combined


# ---------------------------------------------------------------- Matrix Market ingest (matio.cpp:89-214)
@pytest.mark.parametrize("kind", ["real", "complex"])
def test_solve_from_matrix_market_equals_csr(product, oracle, tmp_path, kind):
    """a matrix written to Matrix Market (complex: the 'complex hermitian'
    extension) and read back solves to the same history and values, bit for bit,
    as the in-memory CSR"""
    from paper_2409_05572_b200 import workloads as W
    if kind == "real":
        rp, col, val = W.grid_laplacian((24, 24))
        solver, kw = "lobpcg", dict(n_ev=8, seed=3)
    else:
        rp, col, val = W.magnetic(32)
        solver, kw = "lobpcg", dict(n_ev=8, seed=3)
    n = len(rp) - 1
    a = product.from_csr(n, rp, col, val)
    path = tmp_path / "m.mtx"
    a.write(path)
    b = product.read(path)
    assert b.is_complex == (kind == "complex") and b.nnz_lower == a.nnz_lower
    ra = product.solve(a, solver, strategy=product.strategy_config("fix"), **kw)
    rb = product.solve(b, solver, strategy=product.strategy_config("fix"), **kw)
    assert ra.status == rb.status == 0
    assert _records(ra) == _records(rb)
    assert np.array_equal(ra.values, rb.values)
    # the oracle (fed the same CSR; it has no Matrix Market reader) agrees to rounding
    ro = oracle.solve(oracle.from_csr(n, rp, col, val), solver, strategy=oracle.strategy_config("fix"), **kw)
    np.testing.assert_allclose(rb.values, ro.values, rtol=1e-9)
