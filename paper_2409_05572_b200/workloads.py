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


def matrix_rng(seed):
    """Matrix randomness uses its own stream (SeedSequence [seed, 0xA]) so it is
    not the same sequence as the X0 draw of the same config seed."""
    return np.random.default_rng([seed, 0xA])


def clustered(n=1_000_000, clusters=50, width=1e-3, per_row=8, coupling=0.01, seed=2):
    """Config 3 matrix: A = D + coupling (S + S^T)/2.  D: `clusters`
    centres U[0,100], each holding n/clusters values U[c, c+width], cluster-major
    rows; S: per_row draws per row, with replacement, from columns != row, N(0,1)
    values, duplicates summed.  The lower entry (i, j) is coupling * 0.5 * sum of
    the draws landing on (i, j) or (j, i)."""
    rng = matrix_rng(seed)
    centres = rng.uniform(0.0, 100.0, clusters)
    per = n // clusters
    diag = (centres[:, None] + rng.uniform(0.0, width, (clusters, per))).ravel()
    assert diag.size == n
    r = np.repeat(np.arange(n, dtype=np.int64), per_row)
    c = rng.integers(0, n - 1, r.size)
    c = c + (c >= r)  # columns != row
    v = rng.standard_normal(r.size)
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    rp, col, s = lower_csr_from_coo(n, np.concatenate([hi, np.arange(n)]),
                                    np.concatenate([lo, np.arange(n)]),
                                    np.concatenate([v, np.zeros(n)]))
    # s holds the summed off-diagonal draws (0 on the diagonal): scale, add D
    val = (s * 0.5) * coupling
    rows = np.repeat(np.arange(n), np.diff(rp))
    dpos = np.nonzero(col == rows)[0]
    val[dpos] = diag
    return rp, col, val


def anderson(side=96, w=16.5, seed=3):
    """Config 4 base matrix A: 3D periodic lattice, hopping -1 to each neighbour,
    on-site potential U[-w/2, w/2] per site in site order (x fastest)."""
    rp, col, val = grid_laplacian((side, side, side), periodic=True)
    n = side ** 3
    pot = matrix_rng(seed).uniform(-w / 2, w / 2, n)
    rows = np.repeat(np.arange(n), np.diff(rp))
    val = val.copy()
    val[col == rows] = pot
    return rp, col, val


def full_from_lower(n, rp, col, val):
    import scipy.sparse as sp
    rows = np.repeat(np.arange(n), np.diff(rp))
    low = sp.csr_matrix((val, (rows, col)), shape=(n, n))
    d = sp.diags(low.diagonal())
    return (low + low.T.conj() - d).tocsr()


def lower_from_full(m):
    import scipy.sparse as sp
    low = sp.tril(m).tocsr()
    low.sort_indices()
    return low.indptr.astype(np.int64), low.indices.astype(np.int32), low.data.copy()


def squared(n, rp, col, val):
    """A^2 formed once on the host in fp64, returned as lower CSR."""
    a = full_from_lower(n, rp, col, val)
    return lower_from_full(a @ a)


def magnetic(side=1024, phi=1.0 / 64):
    """Config 5: 2D periodic magnetic Laplacian (complex Hermitian).  Diagonal 4,
    x-links -1, and the y-link (x, y) -> (x, y+1) carries -exp(i 2 pi phi x), i.e.
    H[(x, y+1), (x, y)] = -exp(i 2 pi phi x).  Entries are stored in
    the lower triangle (conjugated where the wrap puts them above the diagonal);
    phi*side is an integer, so the wrap is consistent."""
    n = side * side
    idx = np.arange(n, dtype=np.int64)
    x, y = idx % side, idx // side
    up = x + side * ((y + 1) % side)
    hy = -np.exp(2j * np.pi * phi * x)
    right = (x + 1) % side + side * y
    rows = np.concatenate([idx, up, right])
    cols = np.concatenate([idx, idx, idx])
    vals = np.concatenate([np.full(n, 4.0 + 0j), hy, np.full(n, -1.0 + 0j)])
    # entry (r, c) with r < c goes to the lower triangle as conj at (c, r)
    swap = rows < cols
    r2 = np.where(swap, cols, rows)
    c2 = np.where(swap, rows, cols)
    v2 = np.where(swap, np.conj(vals), vals)
    return lower_csr_from_coo(n, r2, c2, v2)


def config3(solver="lobpcg", n=1_000_000, x0=True):
    """Clustered spectrum, n = 1e6: the nev = 100 LARGEST eigenpairs (solved as the
    smallest of M = -A, values negated back).  LOBPCG at n_ex 150 / n_es 105; SI at
    n_ex 200 with the power operator B = -M = A (op_shift 0).  seed 2, tol 1e-8."""
    rp, c, v = clustered(n=n)
    n_ex = 200 if solver == "si" else 150
    ext = dict(which=1)
    if solver == "si":
        ext.update(op_mode=1, op_shift=0.0)
    return Workload(f"cfg3_clustered_{n}_{solver}", n, rp, c, v, solver,
                    dict(n_ev=100, n_ex=n_ex, tol=1e-8, max_iters=3000), "fix", ext,
                    x0_columns(n, n_ex, 2, "normal") if x0 else None)


def config4(side=96, x0=True):
    """Anderson 96^3 (W = 16.5), the nev = 128 eigenpairs nearest 0 via LOBPCG on
    A^2 (explicit), block 128 + 32 guard vectors, tol 1e-7, seed 3."""
    rp, c, v = anderson(side)
    n = side ** 3
    rp2, c2, v2 = squared(n, rp, c, v)
    return Workload(f"cfg4_anderson_{side}_lobpcg", n, rp2, c2, v2, "lobpcg",
                    dict(n_ev=128, n_ex=160, tol=1e-7, max_iters=40000), "fix", {},
                    x0_columns(n, 160, 3, "normal") if x0 else None)


def config5(side=1024, nev=256, n_ex=384, x0=True):
    """Magnetic Laplacian 1024^2, phi = 1/64, complex128, LOBPCG nev 256, width
    up to 384, complex N(0,1) X0 seed 4, tol 1e-8."""
    rp, c, v = magnetic(side)
    n = side * side
    return Workload(f"cfg5_magnetic_{side}_lobpcg", n, rp, c, v, "lobpcg",
                    dict(n_ev=nev, n_ex=n_ex, tol=1e-8, max_iters=5000), "fix", {},
                    x0_columns(n, n_ex, 4, "complex") if x0 else None)


def lap2d_eigs(nx, ny, k):
    a = 2 - 2 * np.cos(np.arange(1, nx + 1) * np.pi / (nx + 1))
    b = 2 - 2 * np.cos(np.arange(1, ny + 1) * np.pi / (ny + 1))
    return np.sort((a[:, None] + b[None, :]).ravel())[:k]


def lap3d_eigs(m, k):
    a = 2 - 2 * np.cos(np.arange(1, m + 1) * np.pi / (m + 1))
    s = (a[:, None, None] + a[None, :, None] + a[None, None, :]).ravel()
    return np.sort(s)[:k]


def magnetic_eigs(side=1024, phi=1.0 / 64, k=256):
    """Closed form for config 5 (SURVEY.md §8c plan item 3, Harper-chain
    reduction).  The y-link phase depends on x only, so a Fourier transform along
    the periodic y direction (momentum q = 2 pi m / side) splits H into `side`
    periodic chains along x with H_q = 4 - (hops to x +- 1) - 2 cos(q + 2 pi phi x).
    Shifting x by one maps q to q + 2 pi phi, i.e. m to m + phi*side, so chains
    whose m differ by a multiple of phi*side are unitarily equivalent: phi*side
    distinct chains are diagonalised, each spectrum counted side/(phi*side) times.
    Checked against a dense eigensolve at side 64 (tests/test_workloads_cpu.py)."""
    step = round(phi * side)  # m -> m + step under x -> x + 1
    if step < 1 or abs(phi * side - step) > 1e-12 or side % step:
        step = side  # no equivalence to use: every chain
    mult = side // step
    x = np.arange(side)
    vals = []
    for m in range(step):
        q = 2 * np.pi * m / side
        h = np.diag(4.0 - 2.0 * np.cos(q + 2 * np.pi * phi * x))
        h[x, (x + 1) % side] -= 1.0
        h[(x + 1) % side, x] -= 1.0
        vals.append(np.repeat(np.linalg.eigvalsh(h)[:k], mult))
    return np.sort(np.concatenate(vals))[:k]
