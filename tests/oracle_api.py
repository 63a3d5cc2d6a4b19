"""ctypes bindings of the oracle's kernel-level orc_* entry points (test infrastructure)."""
import ctypes as C

import numpy as np

from paper_2409_05572_b200 import blockeig as B

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_D)


class OracleKernels:
    def __init__(self, lib: B.Library):
        self.L = lib
        f = lib.lib
        f.orc_set_threads.argtypes = [C.c_int]
        f.orc_spmv_block.argtypes = [C.c_void_p, _D, C.c_int, _D]
        f.orc_project_orthonormalize.argtypes = [_D, C.c_int, C.c_int, _D, C.c_int, C.c_double, _D, _I]
        f.orc_sym_eig.argtypes = [_D, C.c_int, _D, _D]
        f.orc_hl_trick.argtypes = [_D, C.c_int, C.c_int, _D, C.c_int, C.c_int, _D, _D, _I]
        f.orc_rayleigh_ritz.argtypes = [C.c_void_p, _D, C.c_int, _D, _D, _D]
        f.orc_residual_report.argtypes = [C.c_void_p, _D, _D, C.c_int, C.c_int, C.c_double, _D, _D, _D, _I]
        f.orc_decide_sequence.argtypes = [C.POINTER(B.StrategyConfig), _D, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_int, _I, _D]
        f.orc_validate_strategy.argtypes = [C.POINTER(B.StrategyConfig)]
        f.orc_slope.argtypes = [_D, C.c_int, C.c_int, _D]
        f.orc_resolve_config.argtypes = [C.POINTER(B.SolverConfig), C.c_int, C.POINTER(B.StrategyConfig),
                                         C.c_int, C.c_int, _I, _I]
        f.orc_random_block.argtypes = [C.c_int, C.c_int, C.c_uint64, _D]
        self.f = f

    def _chk(self, code):
        if code != 0:
            raise B.BlockeigError(code, self.L.last_error())

    def spmv_block(self, a, x):
        x = np.asfortranarray(x, dtype=np.float64)
        y = np.zeros_like(x, order="F")
        self._chk(self.f.orc_spmv_block(a.h, _d(x), x.shape[1], _d(y)))
        return y

    def project_orthonormalize(self, w, q=None, drop=1e-8):
        w = np.asfortranarray(w, dtype=np.float64)
        n, a = w.shape
        q = np.zeros((n, 0), order="F") if q is None else np.asfortranarray(q, dtype=np.float64)
        out = np.zeros((n, a), order="F")
        kept = C.c_int()
        qq = q if q.size else np.zeros((n, 1), order="F")
        self._chk(self.f.orc_project_orthonormalize(_d(w), n, a, _d(qq), q.shape[1], drop, _d(out), C.byref(kept)))
        return out[:, :kept.value], kept.value

    def sym_eig(self, h):
        h = np.asfortranarray(h, dtype=np.float64)
        d = h.shape[0]
        vals = np.zeros(d)
        vecs = np.zeros((d, d), order="F")
        self._chk(self.f.orc_sym_eig(_d(h), d, _d(vals), _d(vecs)))
        return vals, vecs

    def hl_trick(self, s, z, n_now, lock=0):
        s = np.asfortranarray(s, dtype=np.float64)
        z = np.asfortranarray(z, dtype=np.float64)
        n, d = s.shape
        x = np.zeros((n, n_now), order="F")
        p = np.zeros((n, n_now), order="F")
        pc = C.c_int()
        self._chk(self.f.orc_hl_trick(_d(s), n, d, _d(z), n_now, lock, _d(x), _d(p), C.byref(pc)))
        return x, p[:, :pc.value]

    def rayleigh_ritz(self, a, s):
        s = np.asfortranarray(s, dtype=np.float64)
        n, d = s.shape
        vals = np.zeros(d)
        vecs = np.zeros((n, d), order="F")
        coeffs = np.zeros((d, d), order="F")
        self._chk(self.f.orc_rayleigh_ritz(a.h, _d(s), d, _d(vals), _d(vecs), _d(coeffs)))
        return vals, vecs, coeffs

    def residual_report(self, a, values, vectors, n_ev, tol):
        vectors = np.asfortranarray(vectors, dtype=np.float64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        n, k = vectors.shape
        r = np.zeros((n, k), order="F")
        pp = np.zeros(k)
        ov = C.c_double()
        cv = C.c_int()
        self._chk(self.f.orc_residual_report(a.h, _d(values), _d(vectors), k, n_ev, tol, _d(r), _d(pp),
                                             C.byref(ov), C.byref(cv)))
        return r, pp, ov.value, cv.value

    def decide_sequence(self, strat, r, n_es, n_ex, start_n_now, start_shrunk, apply_changes=True):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(len(r), dtype=np.int32)
        cmax = C.c_double()
        self._chk(self.f.orc_decide_sequence(C.byref(strat), _d(r), len(r), n_es, n_ex, start_n_now,
                                             int(start_shrunk), int(apply_changes),
                                             out.ctypes.data_as(_I), C.byref(cmax)))
        return list(out), cmax.value

    def slope(self, lr, j_p=0):
        lr = np.ascontiguousarray(lr, dtype=np.float64)
        out = C.c_double()
        self._chk(self.f.orc_slope(_d(lr), len(lr), j_p, C.byref(out)))
        return out.value

    def resolve(self, cfg, solver, strat, n, op_shifted=0):
        ne, ns = C.c_int(), C.c_int()
        self._chk(self.f.orc_resolve_config(C.byref(cfg), solver, C.byref(strat), n, op_shifted,
                                            C.byref(ne), C.byref(ns)))
        return ne.value, ns.value

    def random_block(self, rows, cols, seed):
        out = np.zeros((rows, cols), order="F")
        self.f.orc_random_block(rows, cols, seed, _d(out))
        return out
