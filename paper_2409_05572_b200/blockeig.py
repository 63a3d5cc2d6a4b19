"""ctypes mirror of the ``blockeig.h`` C interface.

This is the Python host-side view of the drop-in boundary (reference
``proj/include/blockeig.h``): the same handles, config structs, status codes,
history records and getters, bound with ctypes.  ``Library`` binds any shared
object that exports the ``beig_*`` symbol set, so the same calls drive the
B200 product (``libblockeig_b200.so``) and, in the tests only, the CPU oracle.

Errors map to ``BlockeigError`` carrying the status code and
``beig_last_error()``, mirroring the reference's exception -> code mapping
(``proj/src/capi.cpp:24-49``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

# status / selector values (reference blockeig.h:22-51)
OK, ERR_INVALID, ERR_PARSE, ERR_IO, ERR_NUMERIC, ERR_INTERNAL = range(6)
SI, SD, LOBPCG, TRACEMIN = range(4)
NONE, FIX, SLOPE, SLOPEK = range(4)
PRECOND_IDENTITY, PRECOND_DIAGONAL = range(2)
EXPAND_XDROP, EXPAND_POWERED, EXPAND_RANDOM = range(3)
STATUS_CONVERGED, STATUS_MAX_ITERS, STATUS_STAGNATED = range(3)
EVENT_NONE, EVENT_SHRINK, EVENT_EXPAND, EVENT_LOCK = range(4)
OP_DEFAULT, OP_SHIFTED = range(2)
WHICH_SMALLEST, WHICH_LARGEST = range(2)

SOLVERS = {"si": SI, "sd": SD, "lobpcg": LOBPCG, "tracemin": TRACEMIN}
STRATEGIES = {"none": NONE, "fix": FIX, "slope": SLOPE, "slopek": SLOPEK}


class SolverConfig(C.Structure):
    _fields_ = [("n_ev", C.c_int), ("n_ex", C.c_int), ("n_es", C.c_int), ("tol", C.c_double),
                ("max_iters", C.c_int), ("shift", C.c_double), ("cg_iters", C.c_int),
                ("precond", C.c_int), ("expand_mode", C.c_int), ("seed", C.c_uint64)]


class StrategyConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("j_e", C.c_int), ("j_s", C.c_int), ("mu", C.c_double),
                ("j_p", C.c_int), ("j_warm", C.c_int), ("r_warm", C.c_double)]


class SolveExt(C.Structure):
    _fields_ = [("op_mode", C.c_int), ("op_shift", C.c_double), ("which", C.c_int),
                ("device", C.c_int), ("profile", C.c_int), ("x0_on_device", C.c_int),
                ("vectors_device", C.c_void_p)]


class IterRecord(C.Structure):
    _fields_ = [("iteration", C.c_int), ("r_overall", C.c_double), ("n_now", C.c_int),
                ("event", C.c_int), ("lock_count", C.c_int), ("spmv_cols", C.c_int64),
                ("solve_cols", C.c_int64), ("ortho_flops", C.c_int64), ("rr_dim", C.c_int)]


class WorkSummary(C.Structure):
    _fields_ = [("spmv_cols", C.c_int64), ("solve_cols", C.c_int64), ("ortho_flops", C.c_int64),
                ("rr_flops", C.c_int64), ("combined", C.c_double)]


class KernelStat(C.Structure):
    _fields_ = [("launches", C.c_int64), ("ms", C.c_double), ("bytes", C.c_double),
                ("flops", C.c_double)]


KERNEL_CLASSES = ["spmm", "gram", "gemm", "syev", "chol", "residual", "other"]


class Example3x3(C.Structure):
    _fields_ = [("x1", C.c_double * 6), ("x2", C.c_double * 6), ("rho_x1", C.c_double),
                ("rho_power", C.c_double), ("rho_expanded", C.c_double), ("asymptotic", C.c_double)]


class SuiteOutcome(C.Structure):
    _fields_ = [("trials", C.c_int), ("violations", C.c_int), ("inconclusive", C.c_int)]


class ScalingOutcome(C.Structure):
    _fields_ = [("floor_rate", C.c_double), ("rate_at_zero", C.c_double),
                ("excess_at_zero", C.c_double), ("eps", C.c_double * 3),
                ("excess", C.c_double * 3), ("slope", C.c_double), ("k_fit", C.c_double),
                ("zero_limit_ok", C.c_int), ("slope_ok", C.c_int)]


# every symbol the header declares: name -> (restype, argtypes)
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_DP = C.POINTER(C.c_double)
SYMBOLS = {
    "beig_last_error": (C.c_char_p, []),
    "beig_matrix_read": (C.c_int, [_PP, C.c_char_p]),
    "beig_matrix_gen": (C.c_int, [_PP, C.c_char_p]),
    "beig_matrix_write": (C.c_int, [_P, C.c_char_p]),
    "beig_matrix_destroy": (None, [_P]),
    "beig_matrix_rows": (C.c_int, [_P]),
    "beig_matrix_nnz_lower": (C.c_int64, [_P]),
    "beig_matrix_norm_est": (C.c_int, [_P, _DP]),
    "beig_matrix_lambda_min": (C.c_int, [_P, _DP]),
    "beig_matrix_spd_shift": (C.c_int, [_PP, _P, C.c_double]),
    "beig_solver_config_default": (None, [C.POINTER(SolverConfig)]),
    "beig_strategy_config_default": (None, [C.POINTER(StrategyConfig)]),
    "beig_solve": (C.c_int, [_PP, _P, C.c_int, C.POINTER(SolverConfig),
                             C.POINTER(StrategyConfig), _DP, C.c_int]),
    "beig_result_destroy": (None, [_P]),
    "beig_result_status": (C.c_int, [_P]),
    "beig_result_iterations": (C.c_int, [_P]),
    "beig_result_nev": (C.c_int, [_P]),
    "beig_result_rows": (C.c_int, [_P]),
    "beig_result_values": (C.c_int, [_P, _DP, C.c_int]),
    "beig_result_vectors": (C.c_int64, [_P, _DP, C.c_int64]),
    "beig_result_history_len": (C.c_int, [_P]),
    "beig_result_history": (C.c_int, [_P, C.POINTER(IterRecord), C.c_int]),
    "beig_result_work": (C.c_int, [_P, C.POINTER(WorkSummary)]),
    "beig_theory_example3x3": (C.c_int, [C.POINTER(Example3x3)]),
    "beig_theory_rate_suite": (C.c_int, [C.POINTER(SuiteOutcome), C.c_int, C.c_uint64,
                                         C.c_char_p, C.c_size_t]),
    "beig_theory_decomp_suite": (C.c_int, [C.POINTER(SuiteOutcome), C.c_int, C.c_uint64,
                                           C.c_char_p, C.c_size_t]),
    "beig_theory_perturb_suite": (C.c_int, [C.POINTER(SuiteOutcome), C.c_int, C.c_uint64,
                                            C.c_char_p, C.c_size_t]),
    "beig_theory_scaling": (C.c_int, [C.POINTER(ScalingOutcome), C.c_uint64]),
    # extensions
    "beig_matrix_from_csr": (C.c_int, [_PP, C.c_int, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int32), _DP]),
    "beig_zmatrix_from_csr": (C.c_int, [_PP, C.c_int, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int32), _DP]),
    "beig_matrix_is_complex": (C.c_int, [_P]),
    "beig_solve_ext_default": (None, [C.POINTER(SolveExt)]),
    "beig_solve_ex": (C.c_int, [_PP, _P, C.c_int, C.POINTER(SolverConfig),
                                C.POINTER(StrategyConfig), _DP, C.c_int, C.POINTER(SolveExt)]),
    "beig_result_vectors_z": (C.c_int64, [_P, _DP, C.c_int64]),
    "beig_result_seconds": (C.c_double, [_P]),
    "beig_result_kernel_stats": (C.c_int, [_P, C.c_int, C.POINTER(KernelStat)]),
    "beig_result_diagnostics": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "beig_result_spmm_windowed": (C.c_longlong, [_P]),
    "beig_release_device_cache": (None, []),
    "beig_result_margins": (C.c_int, [_P, _DP, C.c_int]),
    "beig_harness_project_orthonormalize": (C.c_int, [_DP, C.c_int, C.c_int, _DP, C.c_int, C.c_double, _DP,
                                                      C.POINTER(C.c_int)]),
    "beig_harness_hl_trick": (C.c_int, [_DP, C.c_int, C.c_int, _DP, C.c_int, C.c_int, _DP, _DP,
                                        C.POINTER(C.c_int)]),
}
REFERENCE_SYMBOLS = [s for s in SYMBOLS if s not in (
    "beig_matrix_from_csr", "beig_zmatrix_from_csr", "beig_matrix_is_complex",
    "beig_solve_ext_default", "beig_solve_ex", "beig_result_vectors_z", "beig_result_seconds",
    "beig_result_kernel_stats", "beig_result_diagnostics", "beig_result_spmm_windowed",
    "beig_release_device_cache",
    "beig_harness_project_orthonormalize", "beig_harness_hl_trick", "beig_result_margins")]


class BlockeigError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


class Library:
    """Binds the beig_* symbol set of one shared object."""

    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args

    # -- helpers
    def last_error(self) -> str:
        return self.lib.beig_last_error().decode()

    def check(self, code: int):
        if code != OK:
            raise BlockeigError(code, self.last_error())

    def solver_config(self, **kw) -> SolverConfig:
        c = SolverConfig()
        self.lib.beig_solver_config_default(C.byref(c))
        for k, v in kw.items():
            if not hasattr(c, k):
                raise AttributeError(k)
            setattr(c, k, v)
        return c

    def strategy_config(self, kind=NONE, **kw) -> StrategyConfig:
        c = StrategyConfig()
        self.lib.beig_strategy_config_default(C.byref(c))
        c.kind = STRATEGIES[kind] if isinstance(kind, str) else kind
        for k, v in kw.items():
            if not hasattr(c, k):
                raise AttributeError(k)
            setattr(c, k, v)
        return c

    def solve_ext(self, **kw) -> SolveExt:
        e = SolveExt()
        self.lib.beig_solve_ext_default(C.byref(e))
        for k, v in kw.items():
            setattr(e, k, v)
        return e

    # -- test harness (beig_harness_*)
    def project_orthonormalize(self, w: np.ndarray, q: np.ndarray | None = None, drop: float = 1e-8):
        w = np.asfortranarray(w, dtype=np.float64)
        n, a = w.shape
        q = np.zeros((n, 0)) if q is None else np.asfortranarray(q, dtype=np.float64)
        out = np.zeros((n, max(a, 1)), order="F")
        kept = C.c_int()
        self.check(self.lib.beig_harness_project_orthonormalize(_dptr(w), n, a, _dptr(q) if q.size else None,
                                                                q.shape[1], drop, _dptr(out), C.byref(kept)))
        return out[:, :kept.value].copy(), kept.value

    def hl_trick(self, s: np.ndarray, z: np.ndarray, n_now: int, lock: int = 0):
        s = np.asfortranarray(s, dtype=np.float64)
        z = np.asfortranarray(z, dtype=np.float64)
        n, d = s.shape
        x = np.zeros((n, n_now), order="F")
        p = np.zeros((n, n_now), order="F")
        pc = C.c_int()
        self.check(self.lib.beig_harness_hl_trick(_dptr(s), n, d, _dptr(z), n_now, lock, _dptr(x), _dptr(p),
                                                  C.byref(pc)))
        return x, p[:, :pc.value].copy()

    # -- matrices
    def gen(self, spec: str) -> "Matrix":
        h = C.c_void_p()
        self.check(self.lib.beig_matrix_gen(C.byref(h), spec.encode()))
        return Matrix(self, h)

    def read(self, path: str) -> "Matrix":
        h = C.c_void_p()
        self.check(self.lib.beig_matrix_read(C.byref(h), str(path).encode()))
        return Matrix(self, h)

    def from_csr(self, n, row_ptr, col, val) -> "Matrix":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(col, dtype=np.int32)
        h = C.c_void_p()
        if np.iscomplexobj(val):
            vv = np.ascontiguousarray(val, dtype=np.complex128).view(np.float64)
            self.check(self.lib.beig_zmatrix_from_csr(
                C.byref(h), int(n), rp.ctypes.data_as(C.POINTER(C.c_int64)),
                cl.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(vv)))
        else:
            vv = np.ascontiguousarray(val, dtype=np.float64)
            self.check(self.lib.beig_matrix_from_csr(
                C.byref(h), int(n), rp.ctypes.data_as(C.POINTER(C.c_int64)),
                cl.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(vv)))
        return Matrix(self, h)

    # -- solving
    def solve(self, a: "Matrix", solver="lobpcg", cfg: SolverConfig | None = None,
              strategy: StrategyConfig | None = None, x0: np.ndarray | None = None,
              ext: SolveExt | None = None, x0_device: tuple[int, int] | None = None,
              **cfg_kw) -> "Result":
        """x0_device = (device pointer, columns): a device-resident column-major
        block (ext.x0_on_device); ext.vectors_device keeps the result on the device."""
        solver = SOLVERS[solver] if isinstance(solver, str) else solver
        cfg = cfg if cfg is not None else self.solver_config(**cfg_kw)
        strategy = strategy if strategy is not None else self.strategy_config()
        h = C.c_void_p()
        if x0_device is not None:
            if ext is None or not ext.x0_on_device:
                raise ValueError("x0_device needs ext.x0_on_device = 1")
            xp, cols = C.cast(C.c_void_p(int(x0_device[0])), _DP), int(x0_device[1])
        elif x0 is None:
            xp, cols, keep = None, 0, None
        else:
            if np.iscomplexobj(x0):
                keep = np.asfortranarray(x0, dtype=np.complex128)
                cols = keep.shape[1]
                xp = keep.reshape(-1, order="F").view(np.float64).ctypes.data_as(_DP)
            else:
                keep = np.asfortranarray(x0, dtype=np.float64)
                cols = keep.shape[1]
                xp = keep.ctypes.data_as(_DP)
        code = self.lib.beig_solve_ex(C.byref(h), a.h, solver, C.byref(cfg), C.byref(strategy),
                                      xp, cols, C.byref(ext) if ext is not None else None)
        self.check(code)
        return Result(self, h)


class Matrix:
    def __init__(self, lib: Library, h):
        self.L = lib
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.L.lib.beig_matrix_destroy(self.h)
        except Exception:
            pass

    @property
    def rows(self) -> int:
        return self.L.lib.beig_matrix_rows(self.h)

    @property
    def nnz_lower(self) -> int:
        return self.L.lib.beig_matrix_nnz_lower(self.h)

    @property
    def is_complex(self) -> bool:
        return bool(self.L.lib.beig_matrix_is_complex(self.h))

    def norm_est(self) -> float:
        v = C.c_double()
        self.L.check(self.L.lib.beig_matrix_norm_est(self.h, C.byref(v)))
        return v.value

    def lambda_min(self) -> float:
        v = C.c_double()
        self.L.check(self.L.lib.beig_matrix_lambda_min(self.h, C.byref(v)))
        return v.value

    def spd_shift(self, lam: float) -> "Matrix":
        h = C.c_void_p()
        self.L.check(self.L.lib.beig_matrix_spd_shift(C.byref(h), self.h, lam))
        return Matrix(self.L, h)

    def write(self, path: str):
        self.L.check(self.L.lib.beig_matrix_write(self.h, str(path).encode()))


@dataclass
class Work:
    spmv_cols: int
    solve_cols: int
    ortho_flops: int
    rr_flops: int
    combined: float


class Result:
    def __init__(self, lib: Library, h):
        self.L = lib
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.L.lib.beig_result_destroy(self.h)
        except Exception:
            pass

    @property
    def status(self) -> int:
        return self.L.lib.beig_result_status(self.h)

    @property
    def iterations(self) -> int:
        return self.L.lib.beig_result_iterations(self.h)

    @property
    def nev(self) -> int:
        return self.L.lib.beig_result_nev(self.h)

    @property
    def rows(self) -> int:
        return self.L.lib.beig_result_rows(self.h)

    @property
    def seconds(self) -> float:
        return self.L.lib.beig_result_seconds(self.h)

    @property
    def values(self) -> np.ndarray:
        out = np.zeros(self.nev)
        self.L.lib.beig_result_values(self.h, _dptr(out), self.nev)
        return out

    @property
    def vectors(self) -> np.ndarray:
        n, k = self.rows, self.nev
        out = np.empty(n * k)  # every entry is written by the copy-out
        got = self.L.lib.beig_result_vectors(self.h, _dptr(out), n * k)
        if got == n * k:
            return out.reshape((n, k), order="F")
        out = np.empty(n * k * 2)
        got = self.L.lib.beig_result_vectors_z(self.h, _dptr(out), 2 * n * k)
        if got != 2 * n * k:
            raise BlockeigError(ERR_INTERNAL, "vector copy-out failed")
        return out.view(np.complex128).reshape((n, k), order="F")

    @property
    def history(self) -> list[dict]:
        ln = self.L.lib.beig_result_history_len(self.h)
        arr = (IterRecord * max(ln, 1))()
        got = self.L.lib.beig_result_history(self.h, arr, ln)
        return [{f: getattr(arr[i], f) for f, _ in IterRecord._fields_} for i in range(got)]

    @property
    def margins(self) -> np.ndarray:
        """records x 4: [lo, hi, warm, slope] decision margins (beig_result_margins)"""
        ln = self.L.lib.beig_result_history_len(self.h)
        out = np.full(4 * max(ln, 1), np.nan)
        got = self.L.lib.beig_result_margins(self.h, _dptr(out), ln)
        return out[: 4 * got].reshape(got, 4)

    def kernel_stats(self) -> dict:
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            k = KernelStat()
            self.L.check(self.L.lib.beig_result_kernel_stats(self.h, i, C.byref(k)))
            out[name] = {"launches": k.launches, "ms": k.ms, "bytes": k.bytes, "flops": k.flops}
        return out

    @property
    def diagnostics(self) -> dict:
        fb, sw = C.c_int(), C.c_int()
        self.L.check(self.L.lib.beig_result_diagnostics(self.h, C.byref(fb), C.byref(sw)))
        out = {"cgs2_fallbacks": fb.value, "max_jacobi_sweeps": sw.value}
        if hasattr(self.L.lib, "beig_result_spmm_windowed"):
            out["spmm_windowed"] = int(self.L.lib.beig_result_spmm_windowed(self.h))
        return out

    @property
    def work(self) -> Work:
        w = WorkSummary()
        self.L.check(self.L.lib.beig_result_work(self.h, C.byref(w)))
        return Work(w.spmv_cols, w.solve_cols, w.ortho_flops, w.rr_flops, w.combined)
