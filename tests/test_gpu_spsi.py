"""Shift-and-invert subspace iteration beyond the dense threshold (n > 2000):
the reference factors A - zeta I with Eigen's SimplicialLLT (AMD ordering,
proj/src/kernel.cpp:109-134; used by SI at solvers.cpp:207,234).  The product
runs the symbolic analysis on the host and the numeric factorisation and every
solve on the device (host/spchol.cpp, bk_spchol.cu); the oracle restates the
sparse factor as a band Cholesky in the natural order (oracle/orc_kernel.cpp).
Both factor the same matrix (up to a symmetric permutation), so the solves,
and with them the SI iterates, agree to rounding."""
import numpy as np
import pytest

from paper_2409_05572_b200 import workloads as W
from paper_2409_05572_b200.blockeig import BlockeigError
from tests.helpers import explain_divergence, first_divergence

pytestmark = pytest.mark.gpu


def lap2d(nx, ny):
    rp, c, v = W.grid_laplacian((nx, ny))
    return nx * ny, rp, c, v


@pytest.mark.parametrize("shape,shift,strat", [((60, 60), 0.0, "fix"), ((60, 60), -0.5, "none"),
                                               ((48, 50), 0.001, "slope")])
def test_sparse_shift_invert_matches_oracle(product, oracle, shape, shift, strat):
    n, rp, col, val = lap2d(*shape)
    assert n > 2000
    kw = dict(n_ev=8, tol=1e-10, max_iters=500, seed=5, shift=shift)
    out = []
    for L in (product, oracle):
        a = L.from_csr(n, rp, col, val)
        out.append(L.solve(a, "si", strategy=L.strategy_config(strat), **kw))
    g, o = out
    assert g.status == o.status == 0
    exact = W.lap2d_eigs(shape[0], shape[1], 8)
    np.testing.assert_allclose(g.values, exact, rtol=1e-9)
    np.testing.assert_allclose(g.values, o.values, rtol=1e-9)
    i = first_divergence(g.history, o.history)
    if i is None:
        assert g.iterations == o.iterations
    else:
        why = explain_divergence(g.history, o.history, g.margins, o.margins, i, kw["tol"], values=exact)
        assert why is not None, (i, g.history[i], o.history[i])
    full = W.full_from_lower(n, rp, col, val)
    v = g.vectors
    r = np.linalg.norm(full @ v - v * g.values, axis=0)
    na = product.from_csr(n, rp, col, val).norm_est()
    assert (r <= 2 * kw["tol"] * (na + np.abs(g.values)) * np.linalg.norm(v, axis=0)).all()
    # the history's solve count: every SI iteration applies the factor to the block
    assert g.history[-1]["spmv_cols"] == o.history[-1]["spmv_cols"] or i is not None


def test_sparse_shift_invert_3d(product, oracle):
    rp, col, val = W.grid_laplacian((16, 16, 16))
    n = 4096
    kw = dict(n_ev=6, tol=1e-10, max_iters=500, seed=2, shift=0.0)
    g = product.solve(product.from_csr(n, rp, col, val), "si", strategy=product.strategy_config("fix"), **kw)
    o = oracle.solve(oracle.from_csr(n, rp, col, val), "si", strategy=oracle.strategy_config("fix"), **kw)
    assert g.status == o.status == 0
    np.testing.assert_allclose(g.values, W.lap3d_eigs(16, 6), rtol=1e-9)
    np.testing.assert_allclose(g.values, o.values, rtol=1e-9)


def test_sparse_shift_invert_not_spd(product, oracle):
    # zeta above the smallest eigenvalue: A - zeta I is indefinite; both refuse
    # with the reference's message (kernel.cpp:132-133) as BEIG_ERR_NUMERIC
    n, rp, col, val = lap2d(60, 60)
    for L in (product, oracle):
        with pytest.raises(BlockeigError) as e:
            L.solve(L.from_csr(n, rp, col, val), "si", n_ev=4, shift=0.5, max_iters=5)
        assert e.value.code == 4 and "not positive definite" in str(e.value)
