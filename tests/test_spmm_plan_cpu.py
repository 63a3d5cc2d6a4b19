"""Host plan of the window-staged SpMM (K1w, host/tiling.cpp): invariants that make
the kernel's product equal to the plain CSR product (proj/src/kernel.cpp:8-33) —
checked on the CPU by multiplying through the plan with numpy."""
import ctypes as C

import numpy as np
import pytest

from paper_2409_05572_b200 import LIB_PATH
from paper_2409_05572_b200 import workloads as W
from tests.helpers import spmm_window_plan


@pytest.fixture(scope="module")
def lib():
    return C.CDLL(LIB_PATH)


def full(n, rp, col, val):
    f = W.full_from_lower(n, rp, col, val)
    return f, f.indptr.astype(np.int32), f.indices.astype(np.int32), np.ascontiguousarray(f.data)


def multiply_through_plan(p, n, x):
    """Y = A X the way the kernel walks the plan: per tile, per row, nonzeros in order."""
    y = np.zeros_like(x)
    t_of = np.repeat(np.arange(p["ntiles"]), p["tile"])[:n]
    for i in range(n):
        t = t_of[i]
        w0 = p["wptr"][t]
        row = p["wrow"][w0 + i - t * p["tile"]]
        q0, q1 = p["rp2"][i], p["rp2"][i + 1]
        cols = p["wrow"][w0 + p["code"][q0:q1]]
        y[row] = p["val2"][q0:q1] @ x[cols]
    return y


@pytest.mark.parametrize("dims,tile", [((12, 11, 10), 64), ((40, 37), 32), ((9, 8, 7), 16)])
def test_plan_reproduces_the_product(lib, dims, tile):
    rp, col, val = W.grid_laplacian(dims)
    n = int(np.prod(dims))
    f, frp, fcol, fval = full(n, rp, col, val)
    p = spmm_window_plan(lib, n, frp, fcol, fval, tile=tile, wcap=1 << 20)
    assert p["tile"] == tile and p["ntiles"] == -(-n // tile)
    # the tiles' own rows are a permutation of the matrix rows
    own = np.concatenate([p["wrow"][p["wptr"][t]:p["wptr"][t] + min(tile, n - t * tile)] for t in range(p["ntiles"])])
    assert np.array_equal(np.sort(own), np.arange(n))
    # every slot is inside its tile's window; windows list distinct rows
    sizes = np.diff(p["wptr"])
    assert sizes.max() == p["wmax"]
    for t in range(p["ntiles"]):
        w = p["wrow"][p["wptr"][t]:p["wptr"][t + 1]]
        assert len(np.unique(w)) == len(w)
        q0, q1 = p["rp2"][t * tile], p["rp2"][min(n, (t + 1) * tile)]
        assert q1 - q0 <= p["nzmax"]
        assert p["code"][q0:q1].min() >= 0 and p["code"][q0:q1].max() < len(w)
    x = np.random.default_rng(0).standard_normal((n, 3))
    np.testing.assert_allclose(multiply_through_plan(p, n, x), f @ x, rtol=0, atol=1e-13)
    # each row keeps its nonzeros in CSR order (bit-identity with the plain kernel)
    for i in range(0, n, 97):
        t = i // tile
        row = p["wrow"][p["wptr"][t] + i - t * tile]
        q0, q1 = p["rp2"][i], p["rp2"][i + 1]
        assert np.array_equal(p["wrow"][p["wptr"][t] + p["code"][q0:q1]], fcol[frp[row]:frp[row + 1]])
        assert np.array_equal(p["val2"][q0:q1], fval[frp[row]:frp[row + 1]])


def test_plan_accepts_stencils_and_refuses_random_graphs(lib):
    rp, col, val = W.grid_laplacian((24, 24, 24))
    n = 24 ** 3
    _, frp, fcol, fval = full(n, rp, col, val)
    p = spmm_window_plan(lib, n, frp, fcol, fval)  # defaults: 64-row tiles, shared-memory rule
    assert p["ok"] == 1 and p["tile"] == 64
    assert p["loads_per_row"] < 3.0 and p["wmax"] <= 200  # 4x4x4 blobs: 64 own + 96 halo rows
    # random columns (config 3's structure): as many window rows as nonzeros -> plain kernel
    rng = np.random.default_rng(2)
    m = 4096
    rows = np.repeat(np.arange(m), 8)
    cols = rng.integers(0, m, rows.size)
    lo = rows >= cols
    rp2, c2, v2 = W.lower_csr_from_coo(m, np.r_[rows[lo], np.arange(m)], np.r_[cols[lo], np.arange(m)],
                                        np.r_[rng.standard_normal(lo.sum()), np.full(m, 10.0)])
    _, grp, gcol, gval = full(m, rp2, c2, v2)
    q = spmm_window_plan(lib, m, grp, gcol, gval)
    assert q["ok"] == 0
