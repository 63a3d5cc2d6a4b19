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


# ---------------------------------------------------------------- trajectory flips
def first_divergence(hg, ho):
    """index of the first history record whose (n_now, event, lock_count)
    differs, or the shorter length when one run stops earlier; None if equal"""
    for i, (a, b) in enumerate(zip(hg, ho)):
        if (a["n_now"], a["event"], a["lock_count"]) != (b["n_now"], b["event"], b["lock_count"]):
            return i
    return None if len(hg) == len(ho) else min(len(hg), len(ho)) - 1


def rounding_scale(hg, ho, i, window=5):
    """relative product/oracle difference of r_overall over the records up to i:
    how far summation order has moved the two runs apart at that point"""
    lo = max(0, i - window)
    d = [abs(a["r_overall"] - b["r_overall"]) / b["r_overall"] for a, b in zip(hg[lo:i + 1], ho[lo:i + 1])
         if b["r_overall"] > 0]
    return max(d + [1e-13])


def pair_scale(mg, mo, i, window=10):
    """relative difference of the per-pair ratios either side of the converged
    prefix (margins lo / hi) over the records before i: the pairs near tol drift
    apart faster than r_overall, which the slowest pair sets"""
    import math
    d = []
    for k in range(max(0, i - window), i):
        for c in (0, 1):
            a, b = mg[k][c], mo[k][c]
            if a is not None and b is not None and not (math.isnan(a) or math.isnan(b)) and b > 0:
                d.append(abs(a - b) / b)
    return max(d + [0.0])


def degenerate_boundary(hg, ho, i, values, rel=1e-9):
    """The converged-prefix test (rr.cpp:35-36) split inside a degenerate
    eigenvalue cluster: the pairs converged in one run only (indices between
    the two lock counts) each have a neighbour whose eigenvalue agrees to `rel`.
    Within a degenerate eigenspace the individual Ritz vectors are fixed only up
    to a rotation that rounding chooses, so their per-pair residuals — and which
    of them passes tol first — are not determined by the problem (the 3D
    Laplacian's triples and sextets, config 2)."""
    if values is None or i >= min(len(hg), len(ho)):
        return None
    lg, lo = hg[i]["lock_count"], ho[i]["lock_count"]
    if lg == lo:
        return None
    v = np.asarray(values, dtype=float)
    pairs = range(min(lg, lo), max(lg, lo))
    for p in pairs:
        if p >= len(v):
            return None
        near = [q for q in (p - 1, p + 1) if 0 <= q < len(v) and abs(v[q] - v[p]) <= rel * abs(v[p])]
        if not near:
            return None
    return ("degenerate converged-prefix boundary", (lg, lo), float(v[min(lg, lo)]))


def explain_divergence(hg, ho, mg, mo, i, tol, slack=10.0, values=None):
    """Name the threshold decision that flipped at record i, given each run's
    decision margins (beig_result_margins: per record [lo, hi, warm, slope];
    mo may be None for fixtures recorded without margins).  A decision counts as
    a rounding flip when its margin lies within slack x the runs' measured
    difference of its threshold: the r_overall difference for the warm-up and
    termination tests, the per-pair ratio difference (both runs' margins) for the
    converged-prefix test, 100 x the r_overall difference for the slope test
    (differences of log10 residuals).  With `values` (the converged eigenvalues),
    a lock-count split whose boundary pairs are degenerate is explained too
    (degenerate_boundary).  Returns (reason, margin, delta) or None."""
    import math
    deg = degenerate_boundary(hg, ho, i, values)
    if deg is not None:
        return deg
    dr = slack * rounding_scale(hg, ho, i)
    dp = slack * max(rounding_scale(hg, ho, i), pair_scale(mg, mo, i) if mo is not None else 0.0)
    cands = []
    for m, h in ((mg, hg), (mo, ho)):
        if m is None or i >= len(m):
            continue
        lo, hi, warm, slope = (float("nan") if v is None else v for v in m[i])
        r = h[i]["r_overall"] / tol  # the termination test on the first n_ev pairs
        for name, v, d in (("converged-prefix lo", lo, dp), ("converged-prefix hi", hi, dp),
                           ("warm-up r/r_warm", warm, dr), ("termination r/tol", r, dr)):
            if not math.isnan(v) and abs(v - 1.0) <= d:
                cands.append((name, v, d))
        if not math.isnan(slope) and abs(slope) <= 100 * dr:
            cands.append(("slope test", slope, 100 * dr))
    return cands[0] if cands else None


def spmm_window_plan(lib, n, frp, fcol, fval, tile=0, wcap=0):
    """Host plan of the window-staged SpMM (bk_spmm_win_plan, include/bk_kernels.h)
    as numpy arrays: dict(ok, tile, ntiles, wmax, nzmax, loads_per_row, rp2, code,
    val2, wptr, wrow).  `lib` is the ctypes CDLL of libblockeig_b200.so."""
    import ctypes as C
    lib.bk_spmm_win_plan.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                     C.POINTER(C.c_void_p)]
    lib.bk_spmm_win_plan_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5 + [C.POINTER(C.c_double)]
    lib.bk_spmm_win_plan_arrays.argtypes = [C.c_void_p] + [C.POINTER(C.c_void_p)] * 5 + [C.POINTER(C.c_int64)]
    lib.bk_spmm_win_plan_free.argtypes = [C.c_void_p]
    lib.bk_spmm_win_plan_free.restype = None
    frp = np.ascontiguousarray(frp, dtype=np.int32)
    fcol = np.ascontiguousarray(fcol, dtype=np.int32)
    fval = np.ascontiguousarray(fval, dtype=np.float64)
    h = C.c_void_p()
    rc = lib.bk_spmm_win_plan(n, frp.ctypes.data, fcol.ctypes.data, fval.ctypes.data, tile, wcap, C.byref(h))
    assert rc == 0, rc
    ok, t, nt, wmax, nzmax = (C.c_int() for _ in range(5))
    lpr = C.c_double()
    assert lib.bk_spmm_win_plan_info(h, ok, t, nt, wmax, nzmax, lpr) == 0
    ptrs = [C.c_void_p() for _ in range(5)]
    wl = C.c_int64()
    assert lib.bk_spmm_win_plan_arrays(h, *[C.byref(q) for q in ptrs], C.byref(wl)) == 0
    nnz = int(frp[-1])

    def arr(q, ctype, count, dt):
        if count == 0 or not q.value:
            return np.zeros(0, dtype=dt)
        return np.ctypeslib.as_array(C.cast(q, C.POINTER(ctype)), shape=(count,)).astype(dt, copy=True)
    built = nt.value > 0
    out = dict(ok=ok.value, tile=t.value, ntiles=nt.value, wmax=wmax.value, nzmax=nzmax.value,
               loads_per_row=lpr.value,
               rp2=arr(ptrs[0], C.c_int32, n + 1 if built else 0, np.int32),
               code=arr(ptrs[1], C.c_int32, nnz if built else 0, np.int32),
               val2=arr(ptrs[2], C.c_double, nnz if built else 0, np.float64),
               wptr=arr(ptrs[3], C.c_int32, nt.value + 1 if built else 0, np.int32),
               wrow=arr(ptrs[4], C.c_int32, wl.value, np.int32))
    lib.bk_spmm_win_plan_free(h)
    return out
