"""Seeded synthetic inputs for the five BASELINE.json configurations.

Every generator returns the matrix as a LOWER-triangle CSR (int64 row_ptr,
int32 col, values) — the reference's SparseSym layout (proj/src/matio.hpp:31-56)
— plus the solve settings, so the product and the CPU oracle receive identical
bytes through beig_matrix_from_csr.  Resolved parameters and generator choices
follow SURVEY.md Appendix A/B (grid ordering x-fastest; X0 drawn column by
column from numpy's PCG64 so the first k columns of a wider draw equal a
k-column draw).  None of the paper's SuiteSparse matrices are used.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


def lower_csr_from_coo(n, rows, cols, vals):
    """Sum duplicates, keep col <= row, sort by (row, col)."""
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
    r = uniq // n
    c = (uniq % n).astype(np.int32)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), c, summed


def grid_laplacian(dims, periodic=False):
    """2*len(dims) on the diagonal, -1 to each lattice neighbour; x fastest."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    rows, cols, vals = [idx], [idx], [np.full(n, 2.0 * len(dims))]
    stride = 1
    for d in dims:
        c = (idx // stride) % d
        if periodic:
            nb = idx - stride * c + stride * ((c - 1) % d)
            ok = np.ones(n, bool)
        else:
            nb = idx - stride
            ok = c > 0
        rows.append(idx[ok])
        cols.append(nb[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
        stride *= d
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    # store every coupling in the lower triangle
    lo = np.minimum(r, c)
    hi = np.maximum(r, c)
    return lower_csr_from_coo(n, hi, lo, np.concatenate(vals))


def x0_columns(n, k, seed, kind="normal"):
    """X0 drawn column by column (column-major stream order)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        x = rng.uniform(-1.0, 1.0, size=(k, n))
    elif kind == "complex":
        x = rng.standard_normal(size=(k, n)) + 1j * rng.standard_normal(size=(k, n))
    else:
        x = rng.standard_normal(size=(k, n))
    return np.asfortranarray(x.T)


def sha256(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@dataclass
class Workload:
    name: str
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    solver: str
    cfg: dict
    strategy: str = "none"
    ext: dict = field(default_factory=dict)
    x0: np.ndarray | None = None
    notes: str = ""

    @property
    def nnz_lower(self):
        return int(self.row_ptr[-1])

    @property
    def nnz_full(self):
        diag = int(np.count_nonzero(self.col == np.repeat(np.arange(self.n), np.diff(self.row_ptr))))
        return 2 * self.nnz_lower - diag


def config1(x0=True):
    """2D 5-point Dirichlet Laplacian 100x100, SI with the operator 8I - A (Gershgorin
    bound), nev 20, X0 U[-1,1] seed 0 (n x 40), tol 1e-8, strategy fix."""
    rp, c, v = grid_laplacian((100, 100))
    n = 10000
    return Workload("cfg1_lap2d_100_si", n, rp, c, v, "si",
                    dict(n_ev=20, n_ex=40, tol=1e-8, max_iters=30000), "fix",
                    dict(op_mode=1, op_shift=8.0), x0_columns(n, 40, 0, "uniform") if x0 else None)


def config2(strategy="fix", n_ex=96, side=64, x0=True):
    """3D 7-point Dirichlet Laplacian 64^3, LOBPCG nev 64 with the Jacobi (diagonal)
    preconditioner, X0 N(0,1) seed 1, tol 1e-8.  Strategies run at the reference
    default n_ex = 96 / n_es = 69; strategy none also at the stated width 64 (B2)."""
    rp, c, v = grid_laplacian((side, side, side))
    n = side ** 3
    return Workload(f"cfg2_lap3d_{side}_lobpcg_{strategy}_{n_ex}", n, rp, c, v, "lobpcg",
                    dict(n_ev=64, n_ex=n_ex, tol=1e-8, max_iters=5000, precond=1), strategy, {},
                    x0_columns(n, n_ex, 1, "normal") if x0 else None)


def lap2d_eigs(nx, ny, k):
    a = 2 - 2 * np.cos(np.arange(1, nx + 1) * np.pi / (nx + 1))
    b = 2 - 2 * np.cos(np.arange(1, ny + 1) * np.pi / (ny + 1))
    return np.sort((a[:, None] + b[None, :]).ravel())[:k]


def lap3d_eigs(m, k):
    a = 2 - 2 * np.cos(np.arange(1, m + 1) * np.pi / (m + 1))
    s = (a[:, None, None] + a[None, :, None] + a[None, None, :]).ravel()
    return np.sort(s)[:k]
