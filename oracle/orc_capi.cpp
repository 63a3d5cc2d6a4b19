// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp header).
//
// CPU build of the blockeig.h C interface over the oracle restatement
// (reference proj/src/capi.cpp: same validation order, thread-local error,
// exception -> status mapping).  Exported from liborc_blockeig.so so that the
// parity tests drive the oracle and the B200 product through identical calls.
// Also exports orc_* kernel-level entry points (column-major) for kernel
// parity tests.
#include <chrono>
#include <cstring>
#include <string>

#include "../include/blockeig.h"
#include "orc.hpp"

using orc::cd;

struct beig_matrix {
    bool is_complex = false;
    orc::Sparse<double> m;
    orc::Sparse<cd> z;
    int rows() const { return is_complex ? z.n : m.n; }
    int64_t nnz() const { return is_complex ? z.nnz_lower() : m.nnz_lower(); }
};

struct beig_result {
    bool is_complex = false;
    orc::Result<double> r;
    orc::Result<cd> rz;
    int64_t nnz_lower = 0;
    int rows = 0;
    double seconds = 0;
    // common views
    orc::Status status() const { return is_complex ? rz.status : r.status; }
    int iterations() const { return is_complex ? rz.iterations : r.iterations; }
    const std::vector<double>& values() const { return is_complex ? rz.values : r.values; }
    const std::vector<orc::Record>& history() const { return is_complex ? rz.history : r.history; }
    const orc::Work& work() const { return is_complex ? rz.work : r.work; }
    int64_t rr_flops() const { return is_complex ? rz.rr_flops : r.rr_flops; }
};

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return BEIG_OK;
    } catch (const orc::ParseError& e) {
        g_err = e.what();
        return BEIG_ERR_PARSE;
    } catch (const orc::IoError& e) {
        g_err = e.what();
        return BEIG_ERR_IO;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return BEIG_ERR_INVALID;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return BEIG_ERR_NUMERIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BEIG_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return BEIG_ERR_INTERNAL;
    }
}

int invalid(const char* msg) {
    g_err = msg;
    return BEIG_ERR_INVALID;
}

orc::Mat<double> colmajor(const double* p, int n, int k) {
    orc::Mat<double> m(n, k);
    std::memcpy(m.a.data(), p, sizeof(double) * static_cast<size_t>(n) * k);
    return m;
}

orc::Mat<cd> colmajor_z(const double* p, int n, int k) {
    orc::Mat<cd> m(n, k);
    std::memcpy(reinterpret_cast<double*>(m.a.data()), p, sizeof(double) * 2 * static_cast<size_t>(n) * k);
    return m;
}

}  // namespace

extern "C" {

const char* beig_last_error(void) { return g_err.c_str(); }

int beig_matrix_read(beig_matrix** out, const char* path) {
    if (!out || !path) return invalid("beig_matrix_read: null argument");
    return guarded([&] { throw orc::IoError("oracle: Matrix Market input is not restated"); });
}

int beig_matrix_gen(beig_matrix** out, const char* spec) {
    if (!out || !spec) return invalid("beig_matrix_gen: null argument");
    return guarded([&] {
        auto* h = new beig_matrix;
        try {
            h->m = orc::gen_from_spec(spec);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int beig_matrix_write(const beig_matrix* a, const char* path) {
    if (!a || !path) return invalid("beig_matrix_write: null argument");
    return guarded([&] { throw orc::IoError("oracle: Matrix Market output is not restated"); });
}

void beig_matrix_destroy(beig_matrix* a) { delete a; }
int beig_matrix_rows(const beig_matrix* a) { return a ? a->rows() : 0; }
int64_t beig_matrix_nnz_lower(const beig_matrix* a) { return a ? a->nnz() : 0; }

int beig_matrix_norm_est(const beig_matrix* a, double* out) {
    if (!a || !out) return invalid("beig_matrix_norm_est: null argument");
    return guarded([&] { *out = a->is_complex ? orc::estimate_norm2(a->z) : orc::estimate_norm2(a->m); });
}

int beig_matrix_lambda_min(const beig_matrix* a, double* out) {
    if (!a || !out) return invalid("beig_matrix_lambda_min: null argument");
    return guarded([&] {
        if (a->is_complex) throw std::invalid_argument("lambda_min: real matrices only");
        const int n = a->m.n;
        orc::Mat<double> d(n, n);
        for (int r = 0; r < n; ++r)
            for (int64_t p = a->m.rp[r]; p < a->m.rp[r + 1]; ++p) {
                d(r, a->m.col[p]) = a->m.val[p];
                d(a->m.col[p], r) = a->m.val[p];
            }
        *out = orc::sym_eig_small(d).values.at(0);
    });
}

int beig_matrix_spd_shift(beig_matrix** out, const beig_matrix* a, double lambda1) {
    if (!out || !a) return invalid("beig_matrix_spd_shift: null argument");
    return guarded([&] {
        if (a->is_complex) throw std::invalid_argument("spd_shift: real matrices only");
        auto* h = new beig_matrix;
        h->m = orc::apply_spd_shift(a->m, lambda1);
        *out = h;
    });
}

void beig_solver_config_default(beig_solver_config* cfg) {
    if (!cfg) return;
    const orc::SolverCfg d;
    cfg->n_ev = d.n_ev;
    cfg->n_ex = d.n_ex;
    cfg->n_es = d.n_es;
    cfg->tol = d.tol;
    cfg->max_iters = d.max_iters;
    cfg->shift = d.shift;
    cfg->cg_iters = d.cg_iters;
    cfg->precond = BEIG_PRECOND_IDENTITY;
    cfg->expand_mode = BEIG_EXPAND_XDROP;
    cfg->seed = d.seed;
}

void beig_strategy_config_default(beig_strategy_config* cfg) {
    if (!cfg) return;
    const orc::StratCfg d;
    cfg->kind = BEIG_STRATEGY_NONE;
    cfg->j_e = d.j_e;
    cfg->j_s = d.j_s;
    cfg->mu = d.mu;
    cfg->j_p = d.j_p;
    cfg->j_warm = d.j_warm;
    cfg->r_warm = d.r_warm;
}

void beig_solve_ext_default(beig_solve_ext* ext) {
    if (!ext) return;
    ext->op_mode = BEIG_OP_DEFAULT;
    ext->op_shift = 0.0;
    ext->which = BEIG_WHICH_SMALLEST;
    ext->device = 0;
    ext->profile = 0;
    ext->x0_on_device = 0;
    ext->vectors_device = nullptr;
}

int beig_solve_ex(beig_result** out, const beig_matrix* a, int solver, const beig_solver_config* cfg,
                  const beig_strategy_config* strategy, const double* x0, int x0_cols,
                  const beig_solve_ext* ext) {
    if (!out || !a || !cfg || !strategy) return invalid("beig_solve: null argument");
    if (solver < BEIG_SOLVER_SI || solver > BEIG_SOLVER_TRACEMIN) return invalid("beig_solve: unknown solver");
    if (strategy->kind < BEIG_STRATEGY_NONE || strategy->kind > BEIG_STRATEGY_SLOPEK)
        return invalid("beig_solve: unknown strategy");
    if (cfg->precond < BEIG_PRECOND_IDENTITY || cfg->precond > BEIG_PRECOND_DIAGONAL)
        return invalid("beig_solve: unknown preconditioner");
    if (cfg->expand_mode < BEIG_EXPAND_XDROP || cfg->expand_mode > BEIG_EXPAND_RANDOM)
        return invalid("beig_solve: unknown expand mode");
    if ((x0 == nullptr) != (x0_cols == 0)) return invalid("beig_solve: inconsistent x0");
    if (ext && (ext->op_mode < BEIG_OP_DEFAULT || ext->op_mode > BEIG_OP_SHIFTED))
        return invalid("beig_solve_ex: unknown operator mode");
    if (ext && (ext->which < BEIG_WHICH_SMALLEST || ext->which > BEIG_WHICH_LARGEST))
        return invalid("beig_solve_ex: unknown target");
    if (ext && (ext->x0_on_device || ext->vectors_device))
        return invalid("beig_solve_ex: device-resident blocks need the GPU build");
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        orc::SolverCfg sc;
        sc.n_ev = cfg->n_ev;
        sc.n_ex = cfg->n_ex;
        sc.n_es = cfg->n_es;
        sc.tol = cfg->tol;
        sc.max_iters = cfg->max_iters;
        sc.shift = cfg->shift;
        sc.cg_iters = cfg->cg_iters;
        sc.precond = static_cast<orc::Precond>(cfg->precond);
        sc.expand = static_cast<orc::Expand>(cfg->expand_mode);
        sc.seed = cfg->seed;
        if (ext && ext->op_mode == BEIG_OP_SHIFTED) {
            sc.op_shifted = true;
            sc.op_c = ext->op_shift;
        }
        orc::StratCfg st;
        st.kind = static_cast<orc::Kind>(strategy->kind);
        st.j_e = strategy->j_e;
        st.j_s = strategy->j_s;
        st.mu = strategy->mu;
        st.j_p = strategy->j_p;
        st.j_warm = strategy->j_warm;
        st.r_warm = strategy->r_warm;
        const bool largest = ext && ext->which == BEIG_WHICH_LARGEST;
        auto res = std::make_unique<beig_result>();
        res->nnz_lower = a->nnz();
        res->rows = a->rows();
        const auto kind = static_cast<orc::Solver>(solver);
        if (!a->is_complex) {
            orc::Sparse<double> neg;
            const orc::Sparse<double>* mat = &a->m;
            if (largest) {
                neg = orc::Sparse<double>(a->m.n, a->m.rp, a->m.col, a->m.val);
                for (auto& v : neg.val) v = -v;
                mat = &neg;
            }
            orc::Mat<double> xb;
            if (x0) xb = colmajor(x0, a->m.n, x0_cols);
            res->r = orc::solve(kind, *mat, sc, st, x0 ? &xb : nullptr);
            if (largest)
                for (auto& v : res->r.values) v = -v;
        } else {
            res->is_complex = true;
            orc::Sparse<cd> neg;
            const orc::Sparse<cd>* mat = &a->z;
            if (largest) {
                neg = orc::Sparse<cd>(a->z.n, a->z.rp, a->z.col, a->z.val);
                for (auto& v : neg.val) v = -v;
                mat = &neg;
            }
            orc::Mat<cd> xb;
            if (x0) xb = colmajor_z(x0, a->z.n, x0_cols);
            res->rz = orc::solve(kind, *mat, sc, st, x0 ? &xb : nullptr);
            if (largest)
                for (auto& v : res->rz.values) v = -v;
        }
        res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = res.release();
    });
}

int beig_solve(beig_result** out, const beig_matrix* a, int solver, const beig_solver_config* cfg,
               const beig_strategy_config* strategy, const double* x0, int x0_cols) {
    return beig_solve_ex(out, a, solver, cfg, strategy, x0, x0_cols, nullptr);
}

void beig_result_destroy(beig_result* r) { delete r; }
int beig_result_status(const beig_result* r) { return r ? static_cast<int>(r->status()) : BEIG_STATUS_MAX_ITERS; }
int beig_result_iterations(const beig_result* r) { return r ? r->iterations() : 0; }
int beig_result_nev(const beig_result* r) { return r ? static_cast<int>(r->values().size()) : 0; }
int beig_result_rows(const beig_result* r) { return r ? r->rows : 0; }
double beig_result_seconds(const beig_result* r) { return r ? r->seconds : 0.0; }

int beig_result_values(const beig_result* r, double* out, int cap) {
    if (!r || !out || cap < 0) return 0;
    const int n = std::min<int>(cap, static_cast<int>(r->values().size()));
    for (int i = 0; i < n; ++i) out[i] = r->values()[i];
    return n;
}

int64_t beig_result_vectors(const beig_result* r, double* out, int64_t cap) {
    if (!r || !out || cap < 0 || r->is_complex) return 0;
    const int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(r->r.vectors.a.size()));
    std::memcpy(out, r->r.vectors.a.data(), static_cast<size_t>(n) * sizeof(double));
    return n;
}

int64_t beig_result_vectors_z(const beig_result* r, double* out, int64_t cap) {
    if (!r || !out || cap < 0 || !r->is_complex) return 0;
    const int64_t n = std::min<int64_t>(cap, 2 * static_cast<int64_t>(r->rz.vectors.a.size()));
    std::memcpy(out, reinterpret_cast<const double*>(r->rz.vectors.a.data()), static_cast<size_t>(n) * sizeof(double));
    return n;
}

int beig_result_history_len(const beig_result* r) { return r ? static_cast<int>(r->history().size()) : 0; }

int beig_result_history(const beig_result* r, beig_iter_record* out, int cap) {
    if (!r || !out || cap < 0) return 0;
    const auto& h = r->history();
    const int n = std::min<int>(cap, static_cast<int>(h.size()));
    for (int i = 0; i < n; ++i) {
        out[i].iteration = h[i].iteration;
        out[i].r_overall = h[i].r_overall;
        out[i].n_now = h[i].n_now;
        out[i].event = static_cast<int>(h[i].event);
        out[i].lock_count = h[i].lock_count;
        out[i].spmv_cols = h[i].work.spmv_cols;
        out[i].solve_cols = h[i].work.solve_cols;
        out[i].ortho_flops = h[i].work.ortho_flops;
        out[i].rr_dim = h[i].work.rr_dim;
    }
    return n;
}

int beig_result_margins(const beig_result* r, double* out, int cap_records) {
    if (!r || !out || cap_records < 0) return 0;
    const auto& m = r->is_complex ? r->rz.margins : r->r.margins;
    const int n = std::min<int>(cap_records, static_cast<int>(m.size() / 4));
    std::copy(m.begin(), m.begin() + 4 * static_cast<size_t>(n), out);
    return n;
}

int beig_result_work(const beig_result* r, beig_work_summary* out) {
    if (!r || !out) return invalid("beig_result_work: null argument");
    const auto& w = r->work();
    out->spmv_cols = w.spmv_cols;
    out->solve_cols = w.solve_cols;
    out->ortho_flops = w.ortho_flops;
    out->rr_flops = r->rr_flops();
    out->combined = static_cast<double>(w.spmv_cols + w.solve_cols) * 2.0 * static_cast<double>(r->nnz_lower) +
                    static_cast<double>(w.ortho_flops) + static_cast<double>(r->rr_flops());
    return BEIG_OK;
}

int beig_matrix_from_csr(beig_matrix** out, int n, const int64_t* row_ptr, const int32_t* col,
                         const double* val) {
    if (!out || !row_ptr || (n > 0 && (!col || !val)) || n < 0)
        return invalid("beig_matrix_from_csr: bad argument");
    return guarded([&] {
        const int64_t nnz = row_ptr[n];
        auto* h = new beig_matrix;
        try {
            h->m = orc::Sparse<double>(n, std::vector<int64_t>(row_ptr, row_ptr + n + 1),
                                       std::vector<int>(col, col + nnz), std::vector<double>(val, val + nnz));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int beig_zmatrix_from_csr(beig_matrix** out, int n, const int64_t* row_ptr, const int32_t* col,
                          const double* val) {
    if (!out || !row_ptr || (n > 0 && (!col || !val)) || n < 0)
        return invalid("beig_zmatrix_from_csr: bad argument");
    return guarded([&] {
        const int64_t nnz = row_ptr[n];
        std::vector<cd> v(static_cast<size_t>(nnz));
        std::memcpy(reinterpret_cast<double*>(v.data()), val, sizeof(double) * 2 * static_cast<size_t>(nnz));
        auto* h = new beig_matrix;
        h->is_complex = true;
        try {
            h->z = orc::Sparse<cd>(n, std::vector<int64_t>(row_ptr, row_ptr + n + 1),
                                   std::vector<int>(col, col + nnz), std::move(v));
            for (int r = 0; r < n; ++r)
                if (h->z.diagonal(r).imag() != 0.0)
                    throw std::invalid_argument("Hermitian matrix needs a real diagonal");
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int beig_matrix_is_complex(const beig_matrix* a) { return a && a->is_complex ? 1 : 0; }

// CPU oracle: no device kernels, so no per-kernel statistics
int beig_result_kernel_stats(const beig_result* r, int kernel, beig_kernel_stat* out) {
    if (!r || !out) return invalid("beig_result_kernel_stats: null argument");
    if (kernel < 0 || kernel >= BEIG_KERNEL_CLASSES) return invalid("beig_result_kernel_stats: unknown kernel class");
    *out = beig_kernel_stat{0, 0.0, 0.0, 0.0};
    return BEIG_OK;
}

int beig_result_diagnostics(const beig_result* r, int* cgs2_fallbacks, int* max_jacobi_sweeps) {
    if (!r) return invalid("beig_result_diagnostics: null argument");
    if (cgs2_fallbacks) *cgs2_fallbacks = 0;
    if (max_jacobi_sweeps) *max_jacobi_sweeps = 0;
    return BEIG_OK;
}

// the oracle has one SpMV loop (kernel.cpp:8-33 restated); no windowed variant
long long beig_result_spmm_windowed(const beig_result*) { return 0; }

void beig_release_device_cache(void) {}  // no device memory in the oracle

// ---- analysis checks: outside the hot path; not restated by the oracle ----
int beig_theory_example3x3(beig_example3x3* out) {
    if (!out) return invalid("beig_theory_example3x3: null argument");
    return guarded([&] { throw std::invalid_argument("oracle: theory checks are out of scope"); });
}
int beig_theory_rate_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return invalid("beig_theory_rate_suite: bad arguments");
    return invalid("oracle: theory checks are out of scope");
}
int beig_theory_decomp_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return invalid("beig_theory_decomp_suite: bad arguments");
    return invalid("oracle: theory checks are out of scope");
}
int beig_theory_perturb_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return invalid("beig_theory_perturb_suite: bad arguments");
    return invalid("oracle: theory checks are out of scope");
}
int beig_theory_scaling(beig_scaling_outcome* out, uint64_t) {
    if (!out) return invalid("beig_theory_scaling: null argument");
    return invalid("oracle: theory checks are out of scope");
}

// ================================================================ orc_* kernel entry points
// All blocks column-major.  Return 0 on success, a BEIG_ERR_* code otherwise.

BEIG_API void orc_set_threads(int n) { orc::set_threads(n); }

BEIG_API int orc_spmv_block(const beig_matrix* a, const double* x, int k, double* y) {
    return guarded([&] {
        if (a->is_complex) {
            auto yy = orc::spmv_block(a->z, colmajor_z(x, a->z.n, k));
            std::memcpy(y, reinterpret_cast<double*>(yy.a.data()), yy.a.size() * sizeof(cd));
        } else {
            auto yy = orc::spmv_block(a->m, colmajor(x, a->m.n, k));
            std::memcpy(y, yy.a.data(), yy.a.size() * sizeof(double));
        }
    });
}

BEIG_API int orc_project_orthonormalize(const double* w, int n, int a_cols, const double* q, int m,
                                        double drop, double* out, int* kept) {
    return guarded([&] {
        auto o = orc::project_orthonormalize(colmajor(w, n, a_cols), colmajor(q, n, m), drop);
        std::memcpy(out, o.q.a.data(), o.q.a.size() * sizeof(double));
        *kept = o.kept;
    });
}

BEIG_API int beig_harness_project_orthonormalize(const double* w, int n, int a_cols, const double* q, int m,
                                                 double drop, double* out, int* kept) {
    return orc_project_orthonormalize(w, n, a_cols, q, m, drop, out, kept);
}

BEIG_API int orc_sym_eig(const double* h, int d, double* values, double* vectors) {
    return guarded([&] {
        auto e = orc::sym_eig_small(colmajor(h, d, d));
        std::memcpy(values, e.values.data(), d * sizeof(double));
        std::memcpy(vectors, e.vectors.a.data(), e.vectors.a.size() * sizeof(double));
    });
}

BEIG_API int orc_zsym_eig(const double* h, int d, double* values, double* vectors) {
    return guarded([&] {
        auto e = orc::sym_eig_small(colmajor_z(h, d, d));
        std::memcpy(values, e.values.data(), d * sizeof(double));
        std::memcpy(vectors, reinterpret_cast<double*>(e.vectors.a.data()), e.vectors.a.size() * sizeof(cd));
    });
}

BEIG_API int orc_hl_trick(const double* s, int n, int d, const double* z, int n_now, int lock,
                          double* x_out, double* p_out, int* p_cols) {
    return guarded([&] {
        auto xp = orc::hl_trick(colmajor(s, n, d), colmajor(z, d, d), n_now, lock);
        std::memcpy(x_out, xp.first.a.data(), xp.first.a.size() * sizeof(double));
        std::memcpy(p_out, xp.second.a.data(), xp.second.a.size() * sizeof(double));
        *p_cols = xp.second.c;
    });
}

BEIG_API int beig_harness_hl_trick(const double* s, int n, int d, const double* z, int n_now, int lock,
                                   double* x_out, double* p_out, int* p_cols) {
    return orc_hl_trick(s, n, d, z, n_now, lock, x_out, p_out, p_cols);
}

// one RR step: values (d), vectors (n x d), coeffs (d x d)
BEIG_API int orc_rayleigh_ritz(const beig_matrix* a, const double* s, int d, double* values,
                               double* vectors, double* coeffs) {
    return guarded([&] {
        auto rz = orc::rayleigh_ritz(a->m, colmajor(s, a->m.n, d));
        std::memcpy(values, rz.values.data(), d * sizeof(double));
        std::memcpy(vectors, rz.vectors.a.data(), rz.vectors.a.size() * sizeof(double));
        std::memcpy(coeffs, rz.coeffs.a.data(), rz.coeffs.a.size() * sizeof(double));
    });
}

// residual block + convergence report for given Ritz pairs
BEIG_API int orc_residual_report(const beig_matrix* a, const double* values, const double* vectors,
                                 int k, int n_ev, double tol, double* r_out, double* per_pair,
                                 double* overall, int* converged) {
    return guarded([&] {
        orc::Ritz<double> rz;
        rz.values.assign(values, values + k);
        rz.vectors = colmajor(vectors, a->m.n, k);
        auto r = orc::residual_block(a->m, rz);
        auto rep = orc::assess_convergence(orc::estimate_norm2(a->m), rz, r, n_ev, tol);
        if (r_out) std::memcpy(r_out, r.a.data(), r.a.size() * sizeof(double));
        std::memcpy(per_pair, rep.per_pair.data(), k * sizeof(double));
        *overall = rep.overall;
        *converged = rep.converged;
    });
}

// Drives decide() over a residual sequence, mirroring the block-size change a
// solver applies (reference tests/test_strategy.cpp step()).  decisions[i] gets
// 0 hold / 1 shrink / 2 expand.
BEIG_API int orc_decide_sequence(const beig_strategy_config* cfg, const double* r, int count, int n_es,
                                 int n_ex, int start_n_now, int start_shrunk, int apply_changes,
                                 int* decisions, double* c_max_out) {
    return guarded([&] {
        orc::StratCfg c;
        c.kind = static_cast<orc::Kind>(cfg->kind);
        c.j_e = cfg->j_e;
        c.j_s = cfg->j_s;
        c.mu = cfg->mu;
        c.j_p = cfg->j_p;
        c.j_warm = cfg->j_warm;
        c.r_warm = cfg->r_warm;
        orc::StratState st;
        st.n_now = start_n_now;
        st.shrunk_once = start_shrunk != 0;
        for (int i = 0; i < count; ++i) {
            const auto d = orc::decide(st, c, r[i], n_es, n_ex);
            decisions[i] = static_cast<int>(d);
            if (apply_changes) {
                if (d == orc::Decision::expand) st.n_now = n_ex;
                if (d == orc::Decision::shrink) st.n_now = n_es;
            }
        }
        if (c_max_out) *c_max_out = st.c_max;
    });
}

BEIG_API int orc_validate_strategy(const beig_strategy_config* cfg) {
    return guarded([&] {
        orc::StratCfg c;
        c.kind = static_cast<orc::Kind>(cfg->kind);
        c.j_e = cfg->j_e;
        c.j_s = cfg->j_s;
        c.mu = cfg->mu;
        c.j_p = cfg->j_p;
        c.j_warm = cfg->j_warm;
        c.r_warm = cfg->r_warm;
        orc::validate(c);
    });
}

BEIG_API int orc_slope(const double* lr, int count, int j_p, double* out) {
    return guarded([&] {
        std::vector<double> v(lr, lr + count);
        *out = j_p == 0 ? orc::slope(v) : orc::slope_avg(v, j_p);
    });
}

// resolve_config: writes the resolved n_ex / n_es
BEIG_API int orc_resolve_config(const beig_solver_config* cfg, int solver, const beig_strategy_config* s,
                                int n, int op_shifted, int* n_ex, int* n_es) {
    return guarded([&] {
        orc::SolverCfg sc;
        sc.n_ev = cfg->n_ev;
        sc.n_ex = cfg->n_ex;
        sc.n_es = cfg->n_es;
        sc.tol = cfg->tol;
        sc.max_iters = cfg->max_iters;
        sc.cg_iters = cfg->cg_iters;
        sc.expand = static_cast<orc::Expand>(cfg->expand_mode);
        sc.op_shifted = op_shifted != 0;
        orc::StratCfg c;
        c.kind = static_cast<orc::Kind>(s->kind);
        c.j_e = s->j_e;
        c.j_s = s->j_s;
        c.mu = s->mu;
        c.j_p = s->j_p;
        c.j_warm = s->j_warm;
        c.r_warm = s->r_warm;
        auto r = orc::resolve_config(sc, static_cast<orc::Solver>(solver), c, n);
        *n_ex = r.n_ex;
        *n_es = r.n_es;
    });
}

// consecutive random blocks from one engine, a fresh distribution per block
BEIG_API void orc_random_blocks(uint64_t seed, const int* sizes, int nblocks, double* out) {
    std::mt19937_64 rng(seed);
    size_t off = 0;
    for (int b = 0; b < nblocks; ++b) {
        auto m = orc::random_block<double>(sizes[b], 1, rng);
        std::memcpy(out + off, m.a.data(), m.a.size() * sizeof(double));
        off += m.a.size();
    }
}

// std::mt19937_64 + std::normal_distribution block (reference random_block)
BEIG_API void orc_random_block(int rows, int cols, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    auto m = orc::random_block<double>(rows, cols, rng);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
}

}  // extern "C"
