"""CPU: pin the oracle (CPU restatement of the reference) against the reference's
own known-answer tests (tests/golden/reference_known_answers.json, each entry
citing proj/tests/*.cpp), so that it can serve as the parity checker."""
import json
import os

import numpy as np
import pytest

from paper_2409_05572_b200 import blockeig as B
from tests.helpers import dense_from_lower, laplacian_1d, random_sym_lower
from tests.oracle_api import OracleKernels

KA = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_known_answers.json")))


@pytest.fixture(scope="module")
def ok(oracle):
    return OracleKernels(oracle)


def lap_eig(n, k):
    return 2 - 2 * np.cos(np.arange(1, k + 1) * np.pi / (n + 1))


def sign_normalise(v):
    v = v.copy()
    for c in range(v.shape[1]):
        i = np.argmax(np.abs(v[:, c]))
        v[:, c] *= np.sign(v[i, c])
    return v


def test_si_3x3_golden(oracle):
    g = KA["si_3x3_step"]
    a = oracle.gen(g["matrix"])
    r = oracle.solve(a, "si", x0=np.array(g["x0_rows"], float), **g["cfg"])
    assert r.status == B.STATUS_MAX_ITERS and r.iterations == 1
    got = sign_normalise(r.vectors).T.ravel()
    want = np.array(g["x1_colmajor_sign_normalised"])
    assert np.all(np.abs(got - want) <= g["rel_tol"] * np.abs(want) + g["abs_tol"])


@pytest.mark.parametrize("solver", ["si", "sd", "lobpcg", "tracemin"])
@pytest.mark.parametrize("strat", ["none", "fix", "slope", "slopek"])
def test_laplacian_all_solvers(oracle, solver, strat):
    g = KA["laplacian1d_solvers"]
    n = g["n"]
    rp, col, val = laplacian_1d(n)
    a = oracle.from_csr(n, rp, col, val)
    r = oracle.solve(a, solver, n_ev=g["n_ev"], seed=g["seed"], strategy=oracle.strategy_config(strat))
    assert r.status == B.STATUS_CONVERGED
    np.testing.assert_allclose(r.values, lap_eig(n, g["n_ev"]), rtol=g["value_rel_tol"])
    A = dense_from_lower(rp, col, val, n)
    v = r.vectors
    na = a.norm_est()
    res = A @ v - v * r.values
    for i in range(g["n_ev"]):
        assert np.linalg.norm(res[:, i]) <= g["residual_factor"] * g["tol"] * (na + abs(r.values[i])) * np.linalg.norm(v[:, i])
    assert np.linalg.norm(v.T @ v - np.eye(g["n_ev"])) < g["orthonormality_tol"]
    # history shape (test_solvers.cpp:35-63)
    h = r.history
    assert [x["iteration"] for x in h] == list(range(1, len(h) + 1))
    assert all(h[i]["spmv_cols"] <= h[i + 1]["spmv_cols"] for i in range(len(h) - 1))
    assert all(h[i]["ortho_flops"] <= h[i + 1]["ortho_flops"] for i in range(len(h) - 1))
    assert h[-1]["spmv_cols"] == r.work.spmv_cols


def test_se_cycles(oracle):
    g = KA["se_cycles"]
    a = oracle.gen(g["matrix"])
    r = oracle.solve(a, g["solver"], n_ev=g["n_ev"], seed=g["seed"], strategy=oracle.strategy_config(g["strategy"]))
    assert r.status == B.STATUS_CONVERGED
    ev = [x["event"] for x in r.history]
    s, e = ev.count(B.EVENT_SHRINK), ev.count(B.EVENT_EXPAND)
    assert s >= g["min_shrinks"] and e >= g["min_expands"] and abs(s - e) <= g["max_shrink_expand_gap"]


def test_determinism(oracle):
    g = KA["determinism"]
    a = oracle.gen(g["matrix"])
    runs = [oracle.solve(a, g["solver"], n_ev=g["n_ev"], seed=g["seed"],
                         strategy=oracle.strategy_config(g["strategy"])) for _ in range(2)]
    assert runs[0].history == runs[1].history
    assert np.array_equal(runs[0].values, runs[1].values)


def test_stagnation(oracle):
    g = KA["stagnation"]
    a = oracle.gen(g["matrix"])
    r = oracle.solve(a, g["solver"], n_ev=g["n_ev"], tol=g["tol"])
    assert r.status == B.STATUS_STAGNATED and r.iterations < 2000


def test_resolve_defaults_and_rejections(oracle, ok):
    for c in KA["resolve_defaults"]["cases"]:
        cfg = oracle.solver_config(n_ev=c["n_ev"], n_ex=c.get("n_ex_in", 0))
        n_ex, n_es = ok.resolve(cfg, B.SOLVERS[c["solver"]], oracle.strategy_config("none"), c["n"])
        if "n_ex" in c:
            assert n_ex == c["n_ex"]
        if "n_es" in c:
            assert n_es == c["n_es"]
    for c in KA["resolve_rejections"]["cases"]:
        kw = {k: v for k, v in c.items() if k not in ("n", "solver", "strategy")}
        cfg = oracle.solver_config(**kw)
        with pytest.raises(B.BlockeigError) as e:
            ok.resolve(cfg, B.SOLVERS[c.get("solver", "si")], oracle.strategy_config(c.get("strategy", "none")), c["n"])
        assert e.value.code == B.ERR_INVALID
    for c in KA["resolve_rejections"]["accepted"]:
        kw = {k: v for k, v in c.items() if k not in ("n", "solver", "strategy", "n_es_out")}
        n_ex, n_es = ok.resolve(oracle.solver_config(**kw), B.SOLVERS[c.get("solver", "si")],
                                oracle.strategy_config(c.get("strategy", "none")), c["n"])
        if "n_es_out" in c:
            assert n_es == c["n_es_out"]


def test_sd_precond_and_shift_and_capi(oracle):
    g = KA["sd_diagonal_precond"]
    r = oracle.solve(oracle.gen(g["matrix"]), "sd", n_ev=g["n_ev"], precond=1)
    np.testing.assert_allclose(r.values, 1.06 ** np.arange(g["n_ev"]), rtol=g["value_rel_tol"])
    g = KA["indefinite_shift"]
    d = g["diag_start"] + g["diag_step"] * np.arange(g["n"])
    a = oracle.gen("diag:" + ",".join(repr(float(x)) for x in d))
    r = oracle.solve(a, "si", n_ev=g["n_ev"], shift=1.05 * g["shift_lambda1"])
    np.testing.assert_allclose(r.values, g["values"], rtol=g["value_rel_tol"])
    g = KA["capi_lobpcg_fix"]
    r = oracle.solve(oracle.gen(g["matrix"]), "lobpcg", n_ev=g["n_ev"], seed=g["seed"],
                     strategy=oracle.strategy_config("fix"))
    np.testing.assert_allclose(r.values, 1.05 ** np.arange(g["n_ev"]), rtol=g["value_rel_tol"])
    g = KA["capi_round_trip"]
    m80 = oracle.gen(g["matrix"])
    r = oracle.solve(m80, "si", n_ev=g["n_ev"])
    np.testing.assert_allclose(r.values, lap_eig(80, 3), rtol=g["value_rel_tol"])
    w = r.work
    assert w.combined == pytest.approx(
        (w.spmv_cols + w.solve_cols) * 2.0 * m80.nnz_lower + w.ortho_flops + w.rr_flops, rel=1e-15)


def test_defaults_and_intro(oracle):
    g = KA["capi_defaults"]
    c = oracle.solver_config()
    for k, v in g["solver"].items():
        assert getattr(c, k) == v
    s = oracle.strategy_config()
    for k, v in g["strategy"].items():
        assert getattr(s, k) == v
    m = oracle.gen("laplacian1d:50")
    intro = KA["capi_matrix_intro"]["laplacian1d_50"]
    assert m.rows == intro["rows"] and m.nnz_lower == intro["nnz_lower"]
    assert intro["norm_lo"] < m.norm_est() <= intro["norm_hi"]


def test_norm_estimate_from_below(oracle):
    g = KA["norm_estimate"]
    a = oracle.gen(g["matrix"])
    est = a.norm_est()
    exact = lap_eig(60, 60)[-1]
    assert abs(est - exact) <= g["rel_tol"] * exact and est <= exact * (1 + 1e-12)
    assert a.norm_est() == est


def test_spmv_matches_dense(oracle, ok):
    for seed in (1, 2, 3):
        rp, col, val = random_sym_lower(23, seed)
        a = oracle.from_csr(23, rp, col, val)
        x = np.random.default_rng(seed + 100).standard_normal((23, 4))
        y = ok.spmv_block(a, x)
        np.testing.assert_allclose(y, dense_from_lower(rp, col, val, 23) @ x, rtol=1e-13, atol=1e-13)


def test_cgs2_counts(ok):
    g = KA["cgs2_counts"]
    rng = np.random.default_rng(11)
    q, kept = ok.project_orthonormalize(rng.standard_normal((20, 6)))
    assert kept == 6 and np.abs(q.T @ q - np.eye(6)).max() < g["orthonormality_tol"]
    x = rng.standard_normal((15, 3))
    xx = np.c_[x, 2 * x[:, 0], x[:, 1] - x[:, 2]]
    assert ok.project_orthonormalize(xx)[1] == g["dependent_kept"]
    qb, _ = ok.project_orthonormalize(rng.standard_normal((25, 5)))
    w = rng.standard_normal((25, 4))
    o, kept = ok.project_orthonormalize(w, qb)
    assert kept == 4 and np.abs(qb.T @ o).max() < 1e-12
    inside = (qb[:, 0] + 1e-12 * qb[:, 1])[:, None]
    assert ok.project_orthonormalize(inside, qb)[1] == g["inside_span_kept"]


def test_eig_vs_numpy(ok):
    g = KA["eig_vs_jacobi"]
    rp, col, val = random_sym_lower(g["n"], 21)
    h = dense_from_lower(rp, col, val, g["n"])
    vals, vecs = ok.sym_eig(h)
    np.testing.assert_allclose(vals, np.linalg.eigvalsh(h), rtol=g["value_rel_tol"], atol=1e-13)
    assert np.linalg.norm(h @ vecs - vecs * vals, axis=0).max() < g["residual_tol"]
    # larger / clustered cases
    rng = np.random.default_rng(5)
    for d in (40, 97):
        qm, _ = np.linalg.qr(rng.standard_normal((d, d)))
        lam = np.sort(np.r_[np.full(3, 0.5), rng.uniform(-3, 3, d - 3)])
        hh = (qm * lam) @ qm.T
        v2, z2 = ok.sym_eig(hh)
        np.testing.assert_allclose(v2, lam, atol=1e-12)
        assert np.abs(z2.T @ z2 - np.eye(d)).max() < 1e-12


def test_rr_full_space(oracle, ok):
    g = KA["rr_full_space"]
    a = oracle.gen(g["matrix"])
    rng = np.random.default_rng(1)
    s, _ = ok.project_orthonormalize(rng.standard_normal((14, 14)))
    vals, vecs, _ = ok.rayleigh_ritz(a, s)
    np.testing.assert_allclose(vals, lap_eig(14, 14), rtol=g["value_rel_tol"])
    assert np.abs(vecs.T @ vecs - np.eye(14)).max() < g["orthonormality_tol"]


def test_hl_trick_properties(ok):
    rng = np.random.default_rng(5)
    s, _ = ok.project_orthonormalize(rng.standard_normal((20, 12)))
    z, _ = ok.project_orthonormalize(rng.standard_normal((12, 12)))
    x, p = ok.hl_trick(s, z, 5)
    assert x.shape[1] == 5 and p.shape[1] == 5
    assert np.linalg.norm(x - s @ z[:, :5]) < 1e-13
    xp = np.c_[x, p]
    assert np.linalg.norm(xp.T @ xp - np.eye(10)) < 1e-12
    assert np.linalg.norm(xp - s @ (s.T @ xp)) < 1e-12
    x2, p2 = ok.hl_trick(s, z, 5, 2)
    assert p2.shape[1] <= 3 and np.linalg.norm(x2.T @ p2) < 1e-12


def test_random_block_reproducible(ok):
    a = ok.random_block(9, 3, 77)
    assert np.array_equal(a, ok.random_block(9, 3, 77))
    assert not np.array_equal(a, ok.random_block(9, 3, 78))


def test_oracle_sparse_shift_invert_band_path(oracle):
    """kernel.cpp:109-134 (n > 2000, SimplicialLLT) restated as a band Cholesky:
    SI with shift-and-invert on a 2D Laplacian of n = 3600 reaches the closed
    form, and an indefinite A - zeta I is refused like the reference"""
    import numpy as np
    from paper_2409_05572_b200 import workloads as W
    from paper_2409_05572_b200.blockeig import BlockeigError
    rp, c, v = W.grid_laplacian((60, 60))
    r = oracle.solve(oracle.from_csr(3600, rp, c, v), "si", n_ev=8, tol=1e-10, max_iters=500, seed=5, shift=0.0,
                     strategy=oracle.strategy_config("fix"))
    assert r.status == 0
    np.testing.assert_allclose(r.values, W.lap2d_eigs(60, 60, 8), rtol=1e-9)
    try:
        oracle.solve(oracle.from_csr(3600, rp, c, v), "si", n_ev=4, shift=0.5, max_iters=5)
        raise AssertionError("indefinite factor accepted")
    except BlockeigError as e:
        assert e.code == 4 and "not positive definite" in e.msg
