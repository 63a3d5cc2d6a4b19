"""Kernel-level parity on the B200: every bk_* kernel called through the thin C
ABI on torch-allocated device memory, checked against the CPU oracle (SpMM,
eigensolver) or an fp64 numpy reference (dense contractions).  Tolerances are
written in each test."""
import ctypes as C

import numpy as np
import pytest

from tests.helpers import dense_from_lower, random_sym_lower
from tests.oracle_api import OracleKernels

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

_D = C.c_void_p


@pytest.fixture(scope="module")
def bk(product):
    f = product.lib
    f.bk_spmm_d.argtypes = [C.c_int, _D, _D, _D, _D, C.c_int, C.c_int, _D, C.c_int, _D]
    f.bk_gram_work_bytes.restype = C.c_size_t
    f.bk_gram_work_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
    f.bk_gram_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, _D, _D]
    f.bk_gemm_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, C.c_double, C.c_double, _D,
                            C.c_int, _D]
    f.bk_gram_sym_d.argtypes = [C.c_int, _D, C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, _D, _D]
    f.bk_syev_work_bytes.restype = C.c_size_t
    f.bk_syev_work_bytes.argtypes = [C.c_int]
    f.bk_syev_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, _D, C.c_int, _D, _D, _D]
    f.bk_syev_jacobi_d.argtypes = [C.c_int, _D, C.c_int, _D, _D, C.c_int, _D, _D, _D]
    f.bk_syev_tri_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, _D, C.c_int, _D, _D, _D]
    f.bk_chol_work_bytes.restype = C.c_size_t
    f.bk_chol_work_bytes.argtypes = [C.c_int]
    f.bk_chol_drop_d.argtypes = [C.c_int, _D, C.c_int, _D, C.c_double, _D, C.c_int, _D, _D, _D]
    f.bk_colnorm2_work_bytes.restype = C.c_size_t
    f.bk_colnorm2_work_bytes.argtypes = [C.c_int, C.c_int]
    f.bk_colnorm2_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, _D, _D]
    return f


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def ptr(t):
    return C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def full_csr(rp, col, val, n):
    a = dense_from_lower(rp, col, val, n)
    r, c = np.nonzero(a)
    frp = np.zeros(n + 1, dtype=np.int32)
    np.add.at(frp, r + 1, 1)
    return np.cumsum(frp).astype(np.int32), c.astype(np.int32), a[r, c], a


@pytest.mark.parametrize("k", [1, 7, 32, 50, 96, 150])
def test_spmm_vs_oracle(bk, oracle, k):
    # K1 vs the oracle's reference-order spmv_block: 1e-13 relative (test_kernel.cpp:39-55)
    n = 300
    rp, col, val = random_sym_lower(n, 7, density=0.05)
    frp, fcol, fval, _ = full_csr(rp, col, val, n)
    x = np.random.default_rng(k).standard_normal((n, k))
    ld = k + 3
    xd = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    xd[:, :k] = dev(x)
    yd = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    t_rp, t_c, t_v = dev(frp), dev(fcol), dev(fval)
    assert bk.bk_spmm_d(n, ptr(t_rp), ptr(t_c), ptr(t_v), ptr(xd), ld, k, ptr(yd), ld, stream()) == 0
    torch.cuda.synchronize()
    a = oracle.from_csr(n, rp, col, val)
    want = OracleKernels(oracle).spmv_block(a, x)
    got = yd[:, :k].cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
    # determinism: bit-identical across calls
    y2 = torch.zeros_like(yd)
    bk.bk_spmm_d(n, ptr(t_rp), ptr(t_c), ptr(t_v), ptr(xd), ld, k, ptr(y2), ld, stream())
    torch.cuda.synchronize()
    assert torch.equal(y2[:, :k], yd[:, :k])


@pytest.mark.parametrize("k", [1, 7, 26, 40, 69, 96, 138, 161, 300])
@pytest.mark.parametrize("dims,tile,off", [((12, 11, 10), 64, 0), ((23, 19), 32, 8), ((31, 30, 29), 64, 0),
                                           ((12, 11, 10), 64, 5), ((31, 30, 29), 64, 3)])
def test_spmm_windowed_bit_identical(bk, k, dims, tile, off):
    """Window-staged K1w (X rows of a tile's window staged in shared memory by bulk
    copies, column chunk by column chunk) == plain K1, bit for bit: each row keeps
    its nonzeros in CSR order.  Covers ragged last tiles, odd widths, widths over
    several chunks and X / Y views at an even or odd column offset inside wider blocks
    (odd: the kernel starts one column earlier and never writes that column)."""
    from paper_2409_05572_b200.workloads import grid_laplacian, full_from_lower
    from tests.helpers import spmm_window_plan
    rp, col, val = grid_laplacian(dims)
    n = int(np.prod(dims))
    full = full_from_lower(n, rp, col, val)
    frp, fcol = full.indptr.astype(np.int32), full.indices.astype(np.int32)
    fval = np.random.default_rng(7).standard_normal(full.data.size)  # distinct values: order matters
    p = spmm_window_plan(bk, n, frp, fcol, fval, tile=tile, wcap=1 << 20)
    ld = (k + off + 7) // 8 * 8 + 8
    x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
    y1 = torch.full_like(x, 3.0)
    y2 = torch.full_like(x, 3.0)
    f = bk
    f.bk_spmm_win_d.argtypes = [C.c_int] * 5 + [_D] * 5 + [_D, C.c_int, C.c_int, _D, C.c_int, _D]
    t_rp, t_c, t_v = dev(frp), dev(fcol), dev(fval)
    xo = C.c_void_p(x.data_ptr() + 8 * off)
    assert f.bk_spmm_d(n, ptr(t_rp), ptr(t_c), ptr(t_v), xo, ld, k, C.c_void_p(y1.data_ptr() + 8 * off), ld,
                       stream()) == 0
    d = {name: dev(p[name]) for name in ("rp2", "code", "val2", "wptr", "wrow")}
    assert f.bk_spmm_win_d(n, p["tile"], p["ntiles"], p["wmax"], p["nzmax"], ptr(d["rp2"]), ptr(d["code"]),
                           ptr(d["val2"]), ptr(d["wptr"]), ptr(d["wrow"]), xo, ld, k,
                           C.c_void_p(y2.data_ptr() + 8 * off), ld, stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)  # the columns outside [off, off + k) untouched by both
    want = full_from_lower(n, rp, col, val)
    want.data = fval
    np.testing.assert_allclose(y2[:, off:off + k].cpu().numpy(), want @ x[:, off:off + k].cpu().numpy(),
                               rtol=0, atol=1e-12)


@pytest.mark.parametrize("k", [8, 33, 70])
def test_spmm_windowed_large_windows_and_empty_rows(bk, k):
    """Windows far beyond 8 rows per lane group (a random graph: every tile's halo is
    hundreds of rows, staged by the on-demand row-id loop), rows without nonzeros and
    rows longer than one step group — still bit-identical to K1."""
    from scipy.sparse import random as sprandom, csr_matrix
    from tests.helpers import spmm_window_plan
    n = 1500
    rng = np.random.default_rng(3)
    a = sprandom(n, n, density=0.006, random_state=5, format="csr", data_rvs=rng.standard_normal)
    a = (a + a.T).tolil()
    a[7, :] = 0.0   # empty rows
    a[:, 7] = 0.0
    a[640, :] = 0.0
    a[:, 640] = 0.0
    a[11, 100:160] = rng.standard_normal(60)  # a long row (and its mirror column)
    a[100:160, 11] = a[11, 100:160].T
    a = csr_matrix(a)
    a.eliminate_zeros()
    a.sort_indices()
    frp, fcol, fval = a.indptr.astype(np.int32), a.indices.astype(np.int32), np.ascontiguousarray(a.data)
    p = spmm_window_plan(bk, n, frp, fcol, fval, tile=64, wcap=1 << 20)
    assert p["wmax"] > 300  # beyond 8 rows per lane group
    ld = (k + 7) // 8 * 8
    x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
    y1 = torch.full_like(x, -2.0)
    y2 = torch.full_like(x, -2.0)
    bk.bk_spmm_win_d.argtypes = [C.c_int] * 5 + [_D] * 5 + [_D, C.c_int, C.c_int, _D, C.c_int, _D]
    t_rp, t_c, t_v = dev(frp), dev(fcol), dev(fval)
    assert bk.bk_spmm_d(n, ptr(t_rp), ptr(t_c), ptr(t_v), ptr(x), ld, k, ptr(y1), ld, stream()) == 0
    d = {name: dev(p[name]) for name in ("rp2", "code", "val2", "wptr", "wrow")}
    assert bk.bk_spmm_win_d(n, p["tile"], p["ntiles"], p["wmax"], p["nzmax"], ptr(d["rp2"]), ptr(d["code"]),
                            ptr(d["val2"]), ptr(d["wptr"]), ptr(d["wrow"]), ptr(x), ld, k, ptr(y2), ld,
                            stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert float(y2[7, :k].abs().max()) == 0.0 and float(y2[640, :k].abs().max()) == 0.0
    np.testing.assert_allclose(y2[:, :k].cpu().numpy(), a @ x[:, :k].cpu().numpy(), rtol=0, atol=1e-12)


def test_spmm_windowed_refuses_misaligned_views(bk):
    from paper_2409_05572_b200.workloads import grid_laplacian, full_from_lower
    from tests.helpers import spmm_window_plan
    rp, col, val = grid_laplacian((8, 8, 8))
    full = full_from_lower(512, rp, col, val)
    frp, fcol, fval = full.indptr.astype(np.int32), full.indices.astype(np.int32), full.data
    p = spmm_window_plan(bk, 512, frp, fcol, fval, tile=32, wcap=1 << 20)
    d = {name: dev(p[name]) for name in ("rp2", "code", "val2", "wptr", "wrow")}
    x = torch.randn(512, 16, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    bk.bk_spmm_win_d.argtypes = [C.c_int] * 5 + [_D] * 5 + [_D, C.c_int, C.c_int, _D, C.c_int, _D]
    rc = bk.bk_spmm_win_d(512, p["tile"], p["ntiles"], p["wmax"], p["nzmax"], ptr(d["rp2"]), ptr(d["code"]),
                          ptr(d["val2"]), ptr(d["wptr"]), ptr(d["wrow"]), C.c_void_p(x.data_ptr() + 8), 16, 5,
                          ptr(y), 16, stream())
    assert rc != 0  # odd column offset: not 16-byte aligned, the caller keeps the plain kernel


@pytest.mark.parametrize("n,a,b", [(1000, 13, 70), (262144, 96, 96), (5000, 288, 288), (77, 1, 1),
                                   (100000, 95, 1), (207, 69, 69), (512, 138, 69), (262144, 138, 69)])
def test_gram_vs_numpy(bk, n, a, b):
    rng = np.random.default_rng(n + a)
    x, y = rng.standard_normal((n, a)), rng.standard_normal((n, b))
    xd, yd = dev(x), dev(y)
    c = torch.zeros((a, b), dtype=torch.float64, device="cuda")
    ws = torch.empty(bk.bk_gram_work_bytes(n, a, b) // 8 + 1, dtype=torch.float64, device="cuda")
    assert bk.bk_gram_d(n, ptr(xd), a, a, ptr(yd), b, b, ptr(c), b, ptr(ws), stream()) == 0
    torch.cuda.synchronize()
    want = x.T @ y
    # fp64: |err| <= 1e-13 * n-scaled magnitude
    assert np.abs(c.cpu().numpy() - want).max() <= 1e-13 * np.sqrt(n) * np.abs(want).max() + 1e-12


@pytest.mark.parametrize("n,d,k,beta", [(1000, 40, 40, 0.0), (262144, 288, 96, 0.0), (5000, 96, 7, 1.0), (33, 5, 3, -1.0),
                                        (100000, 70, 1, 1.0), (207, 207, 138, 0.0), (288, 96, 69, 1.0),
                                        (262144, 138, 69, 1.0), (262144, 69, 69, 0.0)])
def test_gemm_vs_numpy(bk, n, d, k, beta):
    rng = np.random.default_rng(d + k)
    x, cm, y0 = rng.standard_normal((n, d)), rng.standard_normal((d, k)), rng.standard_normal((n, k))
    xd, cd, yd = dev(x), dev(cm), dev(y0)
    assert bk.bk_gemm_d(n, ptr(xd), d, d, ptr(cd), k, k, -1.0, beta, ptr(yd), k, stream()) == 0
    torch.cuda.synchronize()
    want = -x @ cm + beta * y0
    assert np.abs(yd.cpu().numpy() - want).max() <= 1e-13 * d * np.abs(want).max()


@pytest.mark.parametrize("n,d,same", [(207, 69, True), (207, 207, False), (262144, 69, True), (262144, 207, False)])
def test_gram_sym_vs_numpy(bk, n, d, same):
    """Symmetric Gram (upper tiles computed, the strict lower triangle mirrored)."""
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d))
    a = rng.standard_normal((n, n)) if n <= 512 else None
    y = x if same else ((a + a.T) @ x if a is not None else x * rng.uniform(0.5, 2.0, (n, 1)))
    xd = dev(x)
    yd = xd if same else dev(y)
    c = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    ws = torch.empty(bk.bk_gram_work_bytes(n, d, d) // 8 + 1, dtype=torch.float64, device="cuda")
    assert bk.bk_gram_sym_d(n, ptr(xd), d, ptr(yd), d, d, ptr(c), d, ptr(ws), stream()) == 0
    torch.cuda.synchronize()
    got, want = c.cpu().numpy(), x.T @ y
    if n <= 512:  # short-axis kernel: upper triangle computed and mirrored
        assert np.array_equal(got, got.T)
    assert np.abs(got - want).max() <= 1e-13 * np.sqrt(n) * np.abs(want).max() + 1e-12


def clustered_sym(d, seed, cluster=(3, 0.5)):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    nc = min(cluster[0], d - 1)
    lam = np.sort(np.r_[np.full(nc, cluster[1]), rng.uniform(-3, 3, d - nc)])
    return (q * lam) @ q.T, lam


@pytest.mark.parametrize("path", ["jacobi", "tri", "dispatch"])
@pytest.mark.parametrize("d", [2, 5, 40, 97, 207, 218, 219, 288])
def test_syev_vs_reference(bk, oracle, path, d):
    if path == "jacobi" and d > 160:
        pytest.skip("one-CTA Jacobi is used for small d only")
    h, lam = clustered_sym(d, d)
    hd = dev(h)
    vals = torch.zeros(d, dtype=torch.float64, device="cuda")
    z = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    ws = torch.empty(bk.bk_syev_work_bytes(d) // 8 + 1, dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    if path == "jacobi":
        rc = bk.bk_syev_jacobi_d(d, ptr(hd), d, ptr(vals), ptr(z), d, ptr(ws), ptr(info), stream())
    elif path == "tri":
        rc = bk.bk_syev_tri_d(d, ptr(hd), d, d, ptr(vals), ptr(z), d, ptr(ws), ptr(info), stream())
    else:
        rc = bk.bk_syev_d(d, ptr(hd), d, d, ptr(vals), ptr(z), d, ptr(ws), ptr(info), stream())
    torch.cuda.synchronize()
    assert rc == 0 and int(info[1]) == 0
    v, zz = vals.cpu().numpy(), z.cpu().numpy()
    ov, _ = OracleKernels(oracle).sym_eig(h)
    scale = np.abs(lam).max()
    np.testing.assert_allclose(v, ov, atol=1e-13 * scale * max(1, d / 50))
    np.testing.assert_allclose(v, lam, atol=1e-12 * scale)
    assert np.all(np.diff(v) >= 0)
    assert np.abs(zz.T @ zz - np.eye(d)).max() < 1e-12
    assert np.linalg.norm(h @ zz - zz * v, axis=0).max() < 1e-12 * scale * max(1, d / 50)


def test_syev_partial_and_degenerate(bk):
    # n_need < d (the LOBPCG use) and an exact 6-fold multiplet
    d, k = 200, 70
    h, lam = clustered_sym(d, 3, cluster=(6, -1.25))
    hd = dev(h)
    vals = torch.zeros(d, dtype=torch.float64, device="cuda")
    z = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    ws = torch.empty(bk.bk_syev_work_bytes(d) // 8 + 1, dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    assert bk.bk_syev_d(d, ptr(hd), d, k, ptr(vals), ptr(z), d, ptr(ws), ptr(info), stream()) == 0
    torch.cuda.synchronize()
    v = vals.cpu().numpy()[:k]
    zz = z.cpu().numpy()[:, :k]
    np.testing.assert_allclose(v, lam[:k], atol=1e-12 * 3)
    assert np.abs(zz.T @ zz - np.eye(k)).max() < 1e-12
    assert np.linalg.norm(h @ zz - zz * v, axis=0).max() < 1e-12 * 3


def test_syev_many_exact_multiplets(bk):
    """Spectra of lattice operators: many exactly degenerate pairs, triples, sextuples
    (the fused small-cluster path) and one 12-fold multiplet (the general path), over
    many matrices.  Inside a multiplet an inverse-iteration step weights the
    eigenvectors by 1 / (lam_i - shift), differences of rounding size; two unbroken
    steps once left a Ritz vector of norm^2 1 + 5e-6 (config 2 none@64), so every
    returned block is checked to 1e-12."""
    rng = np.random.default_rng(2024)
    d, k = 150, 90
    ws = torch.empty(bk.bk_syev_work_bytes(d) // 8 + 1, dtype=torch.float64, device="cuda")
    worst_orth, worst_res = 0.0, 0.0
    for trial in range(60):
        mult = [2, 3, 6, 3, 2, 3, 6, 2, 3, 3, 12, 2, 3, 6, 8, 3, 2]
        lam = []
        x = 0.01
        for m in mult:
            lam += [x] * m
            x += rng.uniform(0.003, 0.02)
        lam += list(rng.uniform(x + 0.05, 12.0, d - len(lam)))
        lam = np.sort(np.array(lam))
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        # nearly diagonal in the leading block, as H = S^T A S is when X holds Ritz vectors
        h = (q * lam) @ q.T
        h = 0.5 * (h + h.T)
        hd = dev(h)
        vals = torch.zeros(d, dtype=torch.float64, device="cuda")
        z = torch.zeros((d, d), dtype=torch.float64, device="cuda")
        info = torch.zeros(4, dtype=torch.int32, device="cuda")
        assert bk.bk_syev_d(d, ptr(hd), d, k, ptr(vals), ptr(z), d, ptr(ws), ptr(info), stream()) == 0
        torch.cuda.synchronize()
        assert int(info[1]) == 0
        v, zz = vals.cpu().numpy()[:k], z.cpu().numpy()[:, :k]
        np.testing.assert_allclose(v, lam[:k], atol=1e-12 * 12)
        worst_orth = max(worst_orth, np.abs(zz.T @ zz - np.eye(k)).max())
        worst_res = max(worst_res, np.linalg.norm(h @ zz - zz * v, axis=0).max())
    assert worst_orth < 1e-12, worst_orth
    assert worst_res < 1e-12 * 12, worst_res


def _chol(bk, w):
    a = w.shape[1]
    g = w.T @ w
    ref2 = np.sum(w * w, axis=0)
    gd, rd = dev(g), dev(ref2)
    m = torch.zeros((a, a), dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    ws = torch.empty(bk.bk_chol_work_bytes(a) // 8 + 1, dtype=torch.float64, device="cuda")
    assert bk.bk_chol_drop_d(a, ptr(gd), a, ptr(rd), 1e-8, ptr(m), a, ptr(info), ptr(ws), stream()) == 0
    torch.cuda.synchronize()
    return int(info[0]), int(info[1]), m.cpu().numpy()


def test_chol_drop_rule(bk):
    # K4 keep/drop (kernel.cpp:83-85 rule): a certainly independent block is
    # orthonormalised by W*m; an exactly dependent column (and a zero column)
    # is dropped; a column whose remaining norm sits inside the cancellation
    # band is reported as uncertain (the driver then redoes it with exact CGS2)
    rng = np.random.default_rng(12)
    x = rng.standard_normal((15, 3))
    w = np.c_[x, 2 * x[:, 0] + 1e-3 * rng.standard_normal(15), np.zeros(15)]
    kept, unsure, m = _chol(bk, w)
    assert (kept, unsure) == (4, 0)
    q = w @ m[:, :kept]
    assert np.abs(q.T @ q - np.eye(kept)).max() < 1e-9
    w2 = np.c_[x, x[:, 1] - x[:, 2] + 1e-10 * rng.standard_normal(15)]
    kept2, unsure2, _ = _chol(bk, w2)
    assert unsure2 == 1


@pytest.mark.parametrize("a", [150, 200, 520])
def test_chol_large_blocks(bk, a):
    # a > 160 runs the grid-cooperative Cholesky (Schur complement in L2); same
    # drop rule and output layout as the shared-memory kernel
    rng = np.random.default_rng(a)
    n = 4 * a
    w = rng.standard_normal((n, a))
    w[:, 7] = 0.0                     # certain drop
    w[:, 11] = w[:, 3] + 1e-3 * w[:, 11]  # kept (well above the 1e-8 threshold)
    kept, unsure, m = _chol(bk, w)
    assert (kept, unsure) == (a - 1, 0)
    assert np.abs(m[7]).max() == 0.0
    q = w @ m[:, :kept]
    assert np.abs(q.T @ q - np.eye(kept)).max() < 1e-7  # one CholQR pass (NS polish follows in K4)
