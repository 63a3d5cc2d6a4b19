"""Problem generators shared by tests and bench (lower-triangle CSR, numpy).

Seeded synthetic inputs for the BASELINE.json configs and the reference's own
test matrices.  Both the product and the oracle receive the SAME arrays through
beig_matrix_from_csr, so parity is never confounded by input generation.
"""
import numpy as np


def lower_csr_from_coo(n, rows, cols, vals):
    """Sum duplicates, keep the lower triangle (col <= row), sort -> (rp, col, val)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals)
    m = cols <= rows
    rows, cols, vals = rows[m], cols[m], vals[m]
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    summed = np.add.reduceat(vals, start) if len(vals) else vals
    r = (uniq // n).astype(np.int64)
    c = (uniq % n).astype(np.int32)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    return rp, c, summed


def laplacian_1d(n):
    i = np.arange(n)
    rows = np.concatenate([i, i[1:]])
    cols = np.concatenate([i, i[1:] - 1])
    vals = np.concatenate([np.full(n, 2.0), np.full(n - 1, -1.0)])
    return lower_csr_from_coo(n, rows, cols, vals)


def laplacian_grid(dims, periodic=False):
    """Dirichlet (or periodic) 2D/3D Laplacian: diag 2*len(dims), off-diag -1,
    lexicographic ordering with x fastest."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n)
    coords = np.unravel_index(idx, dims[::-1])[::-1]  # x fastest
    rows, cols, vals = [idx], [idx], [np.full(n, 2.0 * len(dims))]
    stride = 1
    for ax, d in enumerate(dims):
        c = coords[ax]
        if periodic:
            nb = idx - stride * c + stride * ((c - 1) % d)
            ok = np.ones(n, bool) if d > 2 else c > 0
        else:
            nb = idx - stride
            ok = c > 0
        rows.append(idx[ok]); cols.append(nb[ok]); vals.append(np.full(ok.sum(), -1.0))
        stride *= d
    return lower_csr_from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def dense_from_lower(rp, col, val, n):
    a = np.zeros((n, n), dtype=np.asarray(val).dtype)
    for r in range(n):
        for p in range(rp[r], rp[r + 1]):
            c = col[p]
            a[r, c] = val[p]
            a[c, r] = np.conj(val[p])
    return a


def random_sym_lower(n, seed, density=0.5):
    rng = np.random.default_rng(seed)
    a = np.tril(rng.standard_normal((n, n)))
    keep = rng.random((n, n)) < density
    np.fill_diagonal(keep, True)
    a = np.where(np.tril(keep), a, 0.0)
    r, c = np.nonzero(a)
    return lower_csr_from_coo(n, r, c, a[r, c])


def x0_normal(n, k, seed):
    return np.random.default_rng(seed).standard_normal((n, k))


def x0_uniform(n, k, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (n, k))
