"""The seeded workload generators (paper_2409_05572_b200/workloads.py): exact
reproducibility against the oracle fixtures' input hashes, and the structural
facts SURVEY.md Appendix A/B fixes for each configuration."""
import json
import os

import numpy as np
import pytest

from paper_2409_05572_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(name):
    path = os.path.join(GOLDEN, f"oracle_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"no fixture {path}")
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("make", [W.config1, lambda: W.config2("fix")])
def test_inputs_reproduce_fixture_hashes(make):
    w = make()
    ref = _fixture(w.name)
    assert ref["matrix_sha256"] == W.sha256(w.row_ptr, w.col, w.val)
    assert ref["x0_sha256"] == W.sha256(w.x0)


def _full(w):
    return W.full_from_lower(w.n, w.row_ptr, w.col, w.val)


def test_config1_and_2_shapes():
    w1 = W.config1()
    assert (w1.n, w1.nnz_full, w1.nnz_lower) == (10000, 49600, 29800)
    assert w1.x0.shape == (10000, 40) and w1.x0.min() >= -1 and w1.x0.max() <= 1
    # the first 20 columns of the 40-column draw are the 20-column draw (B1)
    np.testing.assert_array_equal(W.x0_columns(10000, 20, 0, "uniform"), w1.x0[:, :20])
    w2 = W.config2("fix", x0=False)
    assert (w2.n, w2.nnz_full, w2.nnz_lower) == (262144, 1810432, 1036288)


def test_config3_structure():
    w = W.config3("lobpcg", x0=False)
    assert w.n == 1_000_000
    assert abs(w.nnz_full / w.n - 17.0) < 0.01  # ~17 nnz/row after symmetrisation
    rows = np.repeat(np.arange(w.n), np.diff(w.row_ptr))
    on = w.col == rows
    assert np.count_nonzero(on) == w.n and np.all(w.col <= rows)
    d = w.val[on]
    # 50 clusters of 20000 values, each of width <= 1e-3, centres in [0, 100]
    cl = d.reshape(50, 20000)
    assert (cl.max(axis=1) - cl.min(axis=1)).max() <= 1e-3
    assert cl.min() >= 0.0 and cl.max() <= 100.001
    assert np.abs(w.val[~on]).max() < 0.01 * 8  # 0.01 (S + S^T)/2 with N(0,1) draws


def test_config4_is_anderson_squared():
    side = 12  # same generator as 96^3, small enough to check densely
    rp, col, val = W.anderson(side)
    n = side ** 3
    a = W.full_from_lower(n, rp, col, val).toarray()
    assert np.all(np.abs(np.diag(a)) <= 16.5 / 2)
    assert np.count_nonzero(a - np.diag(np.diag(a))) == 6 * n  # periodic, 6 neighbours
    rp2, col2, val2 = W.squared(n, rp, col, val)
    a2 = W.full_from_lower(n, rp2, col2, val2).toarray()
    np.testing.assert_allclose(a2, a @ a, rtol=0, atol=1e-12)
    assert (2 * rp2[-1] - n) == 25 * n
    w = W.config4(x0=False)
    assert (w.n, w.nnz_full) == (884736, 22118400)


def test_config5_hermitian_and_band():
    rp, col, val = W.magnetic(32, 1.0 / 16)
    n = 32 * 32
    a = W.full_from_lower(n, rp, col, val).toarray()
    np.testing.assert_array_equal(a, a.conj().T)
    assert np.all(np.count_nonzero(a, axis=1) == 5)
    e = np.linalg.eigvalsh(a)
    # lowest Landau band: n * phi = 64 states, nearly degenerate, then a gap
    assert np.ptp(e[:64]) < 1e-3 and e[64] - e[63] > 0.1
    w = W.config5(x0=False)
    assert (w.n, w.nnz_full) == (1048576, 5242880)


def test_magnetic_closed_form_matches_dense():
    """Config 5's Harper-chain closed form (the bench's accuracy check) against a
    dense eigensolve of the same generator at side 64."""
    side = 64
    rp, c, v = W.magnetic(side)
    a = W.full_from_lower(side * side, rp, c, v).toarray()
    exact = np.linalg.eigvalsh(a)[:40]
    np.testing.assert_allclose(W.magnetic_eigs(side, 1 / 64, 40), exact, rtol=0, atol=1e-12)
    # full size: the lowest Landau band is 0.0969748 wide to ~1e-14
    full = W.magnetic_eigs(1024, 1 / 64, 256)
    assert abs(full[0] - 0.0969747894970) < 1e-12 and full[-1] - full[0] < 1e-13
