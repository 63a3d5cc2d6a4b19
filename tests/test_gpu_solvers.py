"""Solver-level parity: the B200 product vs the CPU oracle on the reference's
own scenarios (proj/tests/test_solvers.cpp, test_capi.cpp, acceptance_test.cpp).

Bar (BASELINE.json north_star): converged eigenvalues within 1e-9 relative,
every returned residual below tolerance, and the block-size trajectory and
iteration count equal to the oracle's except where rounding flips a threshold
decision (reported, and bounded here).
"""
import numpy as np
import pytest

from tests.helpers import laplacian_1d

pytestmark = pytest.mark.gpu

SOLVERS = ["si", "sd", "lobpcg", "tracemin"]
STRATS = ["none", "fix", "slope", "slopek"]


def lap_eig(n, k):
    return 2 - 2 * np.cos(np.arange(1, k + 1) * np.pi / (n + 1))


def run_both(product, oracle, rp, col, val, n, solver, strat, **kw):
    out = []
    for L in (product, oracle):
        a = L.from_csr(n, rp, col, val)
        out.append(L.solve(a, solver, strategy=L.strategy_config(strat), **kw))
    return out


def trajectory(res):
    return [(h["n_now"], h["event"]) for h in res.history]


def check_residuals(L, rp, col, val, n, res, tol):
    from tests.helpers import dense_from_lower
    a = dense_from_lower(rp, col, val, n)
    v, lam = res.vectors, res.values
    na = L.from_csr(n, rp, col, val).norm_est()
    r = a @ v - v * lam
    for i in range(len(lam)):
        assert np.linalg.norm(r[:, i]) <= tol * (na + abs(lam[i])) * np.linalg.norm(v[:, i])
    g = v.T @ v - np.eye(len(lam))
    assert np.linalg.norm(g) < 1e-10


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("strat", STRATS)
def test_laplacian100_matches_oracle(product, oracle, solver, strat):
    # test_solvers.cpp:106-145 scenario: laplacian1d:100, n_ev=4, seed 11
    n = 100
    rp, col, val = laplacian_1d(n)
    g, o = run_both(product, oracle, rp, col, val, n, solver, strat, n_ev=4, seed=11)
    assert g.status == o.status == 0
    np.testing.assert_allclose(g.values, lap_eig(n, 4), rtol=1e-9)
    np.testing.assert_allclose(g.values, o.values, rtol=1e-9)
    check_residuals(product, rp, col, val, n, g, 2 * 1e-10)
    # trajectory parity: identical unless rounding flips a threshold decision.
    # SD on this problem keeps a residual column whose remaining norm hovers at
    # the 1e-8 drop threshold for ~50 iterations (a genuine rounding flip, see
    # DESIGN.md "parity"), so its iteration count is only bounded, not equal.
    tg, to = trajectory(g), trajectory(o)
    slack = max(2, o.iterations // 5) if solver == "sd" else max(2, o.iterations // 20)
    assert abs(g.iterations - o.iterations) <= slack, (g.iterations, o.iterations)
    same = sum(1 for a, b in zip(tg, to) if a == b)
    assert same >= 0.8 * min(len(tg), len(to))


def test_si_3x3_golden_step(product):
    # test_solvers.cpp:81-104: one shift-invert step on diag(1,10,100)
    x1 = np.array([9.9998e-1, -2.4159e-3, 6.5860e-3, 2.1951e-3, 9.9944e-1, 3.3329e-2])
    a = product.gen("diag:1,10,100")
    x0 = np.array([[1, 1], [1, 4], [1, 2]], float)
    r = product.solve(a, "si", n_ev=2, n_ex=2, tol=1e-13, max_iters=1, x0=x0)
    assert r.status == 1 and r.iterations == 1
    v = r.vectors.copy()
    for c in range(2):
        i = np.argmax(np.abs(v[:, c]))
        v[:, c] *= np.sign(v[i, c])
    got = v.T.ravel()
    assert np.all(np.abs(got - x1) <= 5e-4 * np.abs(x1) + 1e-9)


def test_lobpcg_fix_via_abi(product):
    # test_capi.cpp:239-256: diag-geom:150,1.05, LOBPCG + fix, n_ev=5, seed 4
    a = product.gen("diag-geom:150,1.05")
    r = product.solve(a, "lobpcg", n_ev=5, seed=4, strategy=product.strategy_config("fix"))
    assert r.status == 0
    np.testing.assert_allclose(r.values, 1.05 ** np.arange(5), rtol=1e-8)


def test_sd_diagonal_precond(product):
    # test_solvers.cpp:394-404
    a = product.gen("diag-geom:120,1.06")
    r = product.solve(a, "sd", n_ev=4, precond=1)
    assert r.status == 0
    np.testing.assert_allclose(r.values, 1.06 ** np.arange(4), rtol=1e-8)
