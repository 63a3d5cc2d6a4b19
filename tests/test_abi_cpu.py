"""CPU: the drop-in boundary without a GPU.

- libblockeig_b200.so loads and exports every symbol include/*.h declares
  (BEIG_API / BK_API), and the CPU oracle exports the same beig_* set;
- the host-side logic that runs before any device work behaves like the
  reference C ABI (argument checks and their codes, config defaults, generator
  specs, resolve_config rejections, Matrix Market round trip), mirroring
  proj/tests/test_capi.cpp.  No compute call is made.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2409_05572_b200 import blockeig as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header, macro):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(macro + r"\s+[\w\s\*]+?\b(\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def prod(product_path):
    return B.Library(product_path)


def test_exports_every_declared_symbol(product_path):
    lib = C.CDLL(product_path)
    names = declared("blockeig.h", "BEIG_API") + declared("bk_kernels.h", "BK_API")
    assert len(names) >= 28 + 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_reference_symbol_set_complete(product_path, oracle):
    ref = declared("blockeig.h", "BEIG_API")
    for n in B.REFERENCE_SYMBOLS:
        assert n in ref
    assert len(B.REFERENCE_SYMBOLS) == 28
    ol = C.CDLL(oracle.path)
    assert all(hasattr(ol, n) for n in ref)


def test_defaults(prod):
    c = prod.solver_config()
    assert (c.n_ev, c.n_ex, c.n_es, c.tol, c.max_iters, c.shift, c.cg_iters, c.precond, c.expand_mode, c.seed) == \
        (1, 0, 0, 1e-10, 2000, 0.0, 5, 0, 0, 0)
    s = prod.strategy_config()
    assert (s.kind, s.j_e, s.j_s, s.mu, s.j_p, s.j_warm, s.r_warm) == (0, 12, 2, 1.1, 10, 5, 1e-4)
    e = prod.solve_ext()
    assert (e.op_mode, e.op_shift, e.which, e.device, e.profile) == (0, 0.0, 0, 0, 0)


def test_generators_and_errors(prod):
    m = prod.gen("laplacian1d:50")
    assert m.rows == 50 and m.nnz_lower == 99
    assert 3.8 < m.norm_est() <= 4.0
    assert prod.gen("diag:1,2,3").nnz_lower == 3
    assert prod.gen("diag-geom:10,2.0").rows == 10
    with pytest.raises(B.BlockeigError) as e:
        prod.gen("frobnicate:3")
    assert e.value.code == B.ERR_INVALID and prod.last_error()
    h = C.c_void_p()
    assert prod.lib.beig_matrix_gen(None, b"diag:1") == B.ERR_INVALID
    assert prod.lib.beig_matrix_gen(C.byref(h), None) == B.ERR_INVALID
    with pytest.raises(B.BlockeigError) as e:
        prod.read("no_such_file.mtx")
    assert e.value.code == B.ERR_IO


def test_matrix_market_round_trip(prod, tmp_path):
    bad = tmp_path / "garbage.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1.0\n3 3 5.0\n")
    with pytest.raises(B.BlockeigError) as e:
        prod.read(bad)
    assert e.value.code == B.ERR_PARSE
    a = prod.gen("diag-geom:12,1.5")
    p = tmp_path / "rt.mtx"
    a.write(p)
    b = prod.read(p)
    assert (b.rows, b.nnz_lower) == (a.rows, a.nnz_lower)


def test_matrix_market_complex_hermitian(prod, tmp_path):
    """extension of matio.cpp:89-214: 'complex hermitian' (lower triangle, real
    diagonal) and 'complex general' (mirror must be the conjugate), with the
    reference's strictness; export writes 'complex hermitian'"""
    good = tmp_path / "h.mtx"
    good.write_text("%%MatrixMarket matrix coordinate complex hermitian\n3 3 4\n"
                    "1 1 2.0 0.0\n2 1 -1.0 0.5\n2 2 2.0 0.0\n3 3 4.0 0.0\n")
    a = prod.read(good)
    assert a.is_complex and (a.rows, a.nnz_lower) == (3, 4)
    out = tmp_path / "h2.mtx"
    a.write(out)
    text = out.read_text().splitlines()
    assert text[0] == "%%MatrixMarket matrix coordinate complex hermitian"
    assert text[3].split() == ["2", "1", "-1", "0.5"]
    b = prod.read(out)
    assert b.is_complex and (b.rows, b.nnz_lower) == (3, 4)
    gen = tmp_path / "g.mtx"
    gen.write_text("%%MatrixMarket matrix coordinate complex general\n2 2 4\n"
                   "1 1 1.0 0.0\n2 1 0.0 1.0\n1 2 0.0 -1.0\n2 2 1.0 0.0\n")
    assert prod.read(gen).nnz_lower == 3
    bad_cases = [
        "%%MatrixMarket matrix coordinate complex general\n2 2 4\n1 1 1 0\n2 1 0 1\n1 2 0 1\n2 2 1 0\n",
        "%%MatrixMarket matrix coordinate complex hermitian\n2 2 2\n1 1 1 0.5\n2 2 1 0\n",
        "%%MatrixMarket matrix coordinate complex hermitian\n2 2 2\n1 2 1 0\n2 2 1 0\n",
        "%%MatrixMarket matrix coordinate complex hermitian\n2 2 1\n2 1 1\n",
        "%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n2 1 1 0\n",
    ]
    for i, text in enumerate(bad_cases):
        f = tmp_path / f"bad{i}.mtx"
        f.write_text(text)
        with pytest.raises(B.BlockeigError) as e:
            prod.read(f)
        assert e.value.code == B.ERR_PARSE, (i, e.value)


def test_solve_argument_validation_before_device(prod):
    a = prod.gen("diag:1,2,3,4")
    for kw in ({"n_ev": 0}, {"n_ev": 2, "tol": 0.0}):
        with pytest.raises(B.BlockeigError) as e:
            prod.solve(a, "si", **kw)
        assert e.value.code == B.ERR_INVALID
    with pytest.raises(B.BlockeigError):
        prod.solve(a, 9, n_ev=2)
    s = prod.strategy_config()
    s.kind = 17
    with pytest.raises(B.BlockeigError):
        prod.solve(a, "si", n_ev=2, strategy=s)
    cfg = prod.solver_config(n_ev=2)
    r = C.c_void_p()
    assert prod.lib.beig_solve(None, a.h, 0, C.byref(cfg), C.byref(prod.strategy_config()), None, 0) == B.ERR_INVALID
    x = np.zeros(8)
    assert prod.lib.beig_solve(C.byref(r), a.h, 0, C.byref(cfg), C.byref(prod.strategy_config()), None, 2) == B.ERR_INVALID
    assert prod.lib.beig_solve(C.byref(r), a.h, 0, C.byref(cfg), C.byref(prod.strategy_config()),
                               x.ctypes.data_as(C.POINTER(C.c_double)), 0) == B.ERR_INVALID
    # resolve_config rejections surface before any device work
    for kw, solver, st in [({"n_ev": 4, "n_ex": 4}, "si", "fix"), ({"n_ev": 2, "expand_mode": 1}, "sd", "none"),
                           ({"n_ev": 2, "cg_iters": 0}, "tracemin", "none"), ({"n_ev": 5}, "si", "none")]:
        with pytest.raises(B.BlockeigError) as e:
            prod.solve(a, solver, strategy=prod.strategy_config(st), **kw)
        assert e.value.code == B.ERR_INVALID
    with pytest.raises(B.BlockeigError):
        prod.solve(a, "sd", n_ev=2, ext=prod.solve_ext(op_mode=1, op_shift=8.0))


def test_csr_import_invariants(prod):
    with pytest.raises(B.BlockeigError) as e:  # column above the diagonal
        prod.from_csr(2, [0, 1, 2], [1, 1], [1.0, 1.0])
    assert e.value.code == B.ERR_INVALID
    with pytest.raises(B.BlockeigError):  # unsorted columns
        prod.from_csr(2, [0, 1, 3], [0, 1, 0], [1.0, 1.0, 2.0])
    m = prod.from_csr(2, [0, 1, 3], [0, 0, 1], [2.0, -1.0, 2.0])
    assert m.rows == 2 and m.nnz_lower == 3 and not m.is_complex
    z = prod.from_csr(2, [0, 1, 3], [0, 0, 1], np.array([2.0, -1j, 2.0]))
    assert z.is_complex


def test_theory_checks_out_of_scope(prod):
    ex = B.Example3x3()
    assert prod.lib.beig_theory_example3x3(None) == B.ERR_INVALID
    assert prod.lib.beig_theory_example3x3(C.byref(ex)) == B.ERR_INVALID
    assert "scope" in prod.last_error()


@pytest.mark.parametrize("side", [64, 41])
def test_threaded_norm_estimate_bit_identical(prod, oracle, side):
    """The product's host norm estimate splits the full-CSR rows over threads for
    n >= 65536; each row is summed in the reference scatter order, so the value is
    bit-identical to the oracle's serial estimate_norm2 (kernel.cpp:174-196)."""
    from paper_2409_05572_b200.workloads import grid_laplacian
    rp, col, val = grid_laplacian((side, side, side))
    n = side ** 3
    val = val * (1.0 + 0.1 * np.sin(np.arange(val.size)))  # break the stencil's symmetry of values
    assert prod.from_csr(n, rp, col, val).norm_est() == oracle.from_csr(n, rp, col, val).norm_est()
