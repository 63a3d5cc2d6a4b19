// Host-side core of libblockeig_b200.so: matrix handle, strategy state
// machine, device workspace and the four solver loops.  The loops restate the
// reference's control flow (proj/src/solvers.cpp) over device-resident blocks;
// every dense / sparse operation is a bk_* CUDA kernel (include/bk_kernels.h).
#pragma once

#include <sys/mman.h>

#include <atomic>
#include <cstdlib>
#include <new>
#include <cstdint>
#include <future>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/bk_kernels.h"

namespace b2 {

// allocator whose value-initialisation is a no-op: resize() without a zero-fill
// pass over GB-sized host result buffers
template <class T>
struct NoInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <class U>
    NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
    // GB-sized results: 2 MB-aligned with transparent huge pages requested, so
    // first-touch page faults (which halved the result copy-out rate) are rare
    T* allocate(std::size_t n) {
        const std::size_t bytes = n * sizeof(T);
        if (bytes < (std::size_t(4) << 20)) return std::allocator<T>::allocate(n);
        void* p = nullptr;
        if (posix_memalign(&p, std::size_t(2) << 20, bytes) != 0) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);
        return static_cast<T*>(p);
    }
    void deallocate(T* p, std::size_t n) {
        if (n * sizeof(T) < (std::size_t(4) << 20)) return std::allocator<T>::deallocate(p, n);
        free(p);
    }
    template <class U>
    void construct(U*) noexcept {}
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};

// ---------------------------------------------------------------- errors
// Mapped by the C ABI exactly like the reference (proj/src/capi.cpp:24-49):
// invalid_argument -> INVALID, runtime_error -> NUMERIC, ParseError -> PARSE,
// IoError -> IO, anything else -> INTERNAL.  A CUDA failure is deliberately
// NOT a runtime_error so that it surfaces as BEIG_ERR_INTERNAL.
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, long line)
        : std::runtime_error("line " + std::to_string(line) + ": " + what) {}
};
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CudaError : public std::exception {
public:
    explicit CudaError(std::string m) : msg_(std::move(m)) {}
    const char* what() const noexcept override { return msg_.c_str(); }

private:
    std::string msg_;
};

void cuda_check(int code, const char* what);  // throws CudaError when code != 0

// ---------------------------------------------------------------- device memory
class DevMem {
public:
    DevMem() = default;
    explicit DevMem(size_t bytes) { alloc(bytes); }
    ~DevMem();
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    DevMem(DevMem&& o) noexcept : p_(o.p_), bytes_(o.bytes_), dev_(o.dev_) { o.p_ = nullptr, o.bytes_ = 0; }
    void alloc(size_t bytes);
    template <class T> T* as() const { return static_cast<T*>(p_); }
    void* p() const { return p_; }
    double* d() const { return static_cast<double*>(p_); }
    size_t bytes() const { return bytes_; }

private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
    int dev_ = 0;
};

// empty the device block cache (see matrix.cpp)
void release_device_cache();

// Host plan of the window-staged SpMM (K1w, host/tiling.cpp): rows regrouped into
// tiles of graph-local rows; window t = wrow[wptr[t] .. wptr[t+1]) lists the X rows
// tile t needs (its own rows first, then the halo); code[p] is the window slot of
// nonzero p (rows in tile order, each row's nonzeros in their original order).
struct WindowPlan {
    bool ok = false;
    int n = 0, tile = 0, ntiles = 0, wmax = 0, nzmax = 0;
    double loads_per_row = 0.0;  // window slots per matrix row (X-row loads from L2)
    std::vector<int32_t> rp2, code, wptr, wrow;
    std::vector<double> val2;
};
double cluster_rows(int n, const int32_t* rp, const int32_t* col, int tile, std::vector<int32_t>& order);
void build_windows(int n, const int32_t* rp, const int32_t* col, const double* val, int per, int tile,
                   const std::vector<int32_t>& order, WindowPlan& w);
bool plan_windows(int n, const int32_t* rp, const int32_t* col, const double* val, int per, int tile_req,
                  int wcap, WindowPlan& w);

// ---------------------------------------------------------------- matrix
// Lower-triangle CSR with the reference invariants (proj/src/matio.cpp:17-35):
// int64 row_ptr, int32 strictly increasing columns <= row.  Immutable after
// construction; the norm estimate and the device copy (full CSR, int32) are
// cached and shared between copies of the handle.
struct DeviceCsr {
    int device = -1;
    int n = 0;
    int64_t nnz_full = 0;
    DevMem row_ptr, col, val;
    bool negated = false;
    // window-staged SpMM (K1w, bk_spmm_win_d): the plan is built and uploaded by a
    // host thread started with the first solve on a real matrix of >= 65536 rows;
    // win_state: 0 not started, 1 building, 2 ready, 3 unsuitable (or failed).
    // K1w is bit-identical to the plain kernel, so a solve switches over as soon
    // as the state reads 2.
    struct Win {
        int tile = 0, ntiles = 0, wmax = 0, nzmax = 0;
        double loads_per_row = 0.0, plan_seconds = 0.0;
        DevMem rp2, code, val2, wptr, wrow;
    };
    mutable std::atomic<int> win_state{0};
    mutable Win win;
    mutable std::future<void> win_job;  // joined by the destructor (std::async future)
};

class SparseSym {
public:
    SparseSym();
    SparseSym(int n, std::vector<int64_t> rp, std::vector<int> col, std::vector<double> val,
              bool complex_values = false);
    int rows() const { return n_; }
    int64_t nnz_lower() const { return static_cast<int64_t>(col_.size()); }
    bool is_complex() const { return complex_; }
    const std::vector<int64_t>& row_ptr() const { return rp_; }
    const std::vector<int>& col() const { return col_; }
    const std::vector<double>& val() const { return val_; }  // interleaved when complex
    double diagonal(int i) const;                             // real part; 0 when absent
    double norm_est() const;                                  // estimate_norm2, cached
    bool norm_cached() const { return norm_cache_->load(std::memory_order_relaxed) >= 0.0; }
    // full (both triangles) CSR on `device`, optionally with negated values (M = -A)
    const DeviceCsr& device_csr(int device, bool negate) const;
    // full (both triangles) CSR: per row the lower entries then the mirrored
    // (conjugated) upper ones, columns ascending; built once per handle and
    // shared by the norm estimate and the device uploads
    struct FullCsr {
        std::vector<int32_t> rp, col;
        std::vector<double> val;  // interleaved when complex
    };
    const FullCsr& full_csr() const;

private:
    int n_;
    bool complex_;
    std::vector<int64_t> rp_;
    std::vector<int> col_;
    std::vector<double> val_;
    std::shared_ptr<std::atomic<double>> norm_cache_;
    struct DevCache {
        std::mutex mu;
        std::vector<std::unique_ptr<DeviceCsr>> entries;
        std::mutex full_mu;
        bool full_ready = false;
        FullCsr full;
        // the window-plan threads of the entries read `full`: join them before any
        // member goes away (members are destroyed last-declared first)
        ~DevCache() {
            for (auto& e : entries)
                if (e && e->win_job.valid()) e->win_job.wait();
        }
    };
    std::shared_ptr<DevCache> dev_;
};

SparseSym gen_from_spec(const std::string& spec);
SparseSym apply_spd_shift(const SparseSym& a, double lambda1);
double spd_shift_value(double lambda1);
SparseSym parse_matrix_market_file(const std::string& path);
void write_matrix_market_file(const SparseSym& a, const std::string& path);

// ---------------------------------------------------------------- sparse shift-and-invert
// Factor of sgn A - shift I for shift-and-invert SI on n > 2000 (reference
// SpdFactor sparse path, proj/src/kernel.cpp:110-134): symbolic analysis on the
// host, numeric factorisation and solves on the device (host/spchol.cpp,
// bk_spchol.cu).  Throws runtime_error when the matrix is not positive definite.
class SpChol {
public:
    SpChol(const SparseSym& a, double sgn, double shift, void* stream);
    // y = (sgn A - shift I)^{-1} x for m columns of row-major blocks (x != y)
    void solve(const double* x, int ldx, int m, double* y, int ldy, void* stream);
    int64_t nnz_l() const { return nnz_l_; }
    int levels() const { return nlev_; }

private:
    int n_ = 0, nlev_ = 0;
    int64_t nnz_l_ = 0;
    std::vector<int> perm_h_, lvlptr_h_;
    DevMem colptr_, rowind_, val_, rptr_, rk_, rpos_, order_, lvlptr_, perm_, fail_, t_;
};

// ---------------------------------------------------------------- strategy
// proj/src/strategy.{hpp,cpp}: same knobs, same decisions.
enum class StrategyKind { none = 0, fix = 1, slope = 2, slopek = 3 };
enum class Decision { hold = 0, shrink = 1, expand = 2 };
struct StrategyConfig {
    StrategyKind kind = StrategyKind::none;
    int j_e = 12, j_s = 2;
    double mu = 1.1;
    int j_p = 10, j_warm = 5;
    double r_warm = 1e-4;
};
class BlockSizer {
public:
    explicit BlockSizer(const StrategyConfig& c) : c_(c) {}
    Decision step(double r_now, int n_now, int n_es, int n_ex);
    double c_max() const { return c_max_; }
    // enter the post-warm-up state (reference tests' shrunken_state(), test_strategy.cpp:15-20)
    void mark_warmed() { warmed_ = true; }
    // decision margins of the last step (NaN when the test did not run):
    // r / r_warm of the warm-up shrink test; (c_max - mu c) / (mu c) for c > 0,
    // else c_max, of the slope test (strategy.cpp:49,85)
    double warm_margin() const { return m_warm_; }
    double slope_margin() const { return m_slope_; }

private:
    double m_warm_ = 0.0, m_slope_ = 0.0;
    StrategyConfig c_;
    int j_ = 0;
    std::vector<double> lg_;
    bool warmed_ = false;
    int last_expand_ = -1;
    bool have_ref_ = false;
    double c_max_ = 0.0;
};
void validate_strategy(const StrategyConfig& c);

// ---------------------------------------------------------------- solver
enum class SolverKind { si = 0, sd = 1, lobpcg = 2, tracemin = 3 };
enum class Precond { identity = 0, diagonal = 1 };
enum class ExpandMode { x_drop = 0, powered = 1, random = 2 };
enum class Status { converged = 0, max_iters = 1, stagnated = 2 };
enum class Event { none = 0, shrink = 1, expand = 2, lock = 3 };

struct SolverConfig {
    int n_ev = 1, n_ex = 0, n_es = 0;
    double tol = 1e-10;
    int max_iters = 2000;
    double shift = 0.0;
    int cg_iters = 5;
    Precond precond = Precond::identity;
    ExpandMode expand = ExpandMode::x_drop;
    uint64_t seed = 0;
    // extensions (beig_solve_ex)
    bool op_shifted = false;
    double op_c = 0.0;
    bool largest = false;
    int device = 0;
    bool profile = false;
    bool x0_on_device = false;        // x0 is a device pointer (column-major)
    double* vectors_device = nullptr;  // result vectors stay on the device (column-major)
};

enum KernelClass { K_SPMM = 0, K_GRAM, K_GEMM, K_SYEV, K_CHOL, K_RESID, K_OTHER, K_CLASSES };
struct KernelStat {
    int64_t launches = 0;
    double ms = 0.0, bytes = 0.0, flops = 0.0;
};

struct Work {
    int64_t spmv_cols = 0, solve_cols = 0, ortho_flops = 0;
    int rr_dim = 0;
};
struct Record {
    int iteration;
    double r_overall;
    int n_now;
    Event event;
    int lock_count;
    Work work;
};
struct SolveOutput {
    Status status = Status::max_iters;
    std::vector<double> values;   // n_ev, ascending (descending for `largest`)
    // n x n_ev column-major (interleaved when complex); no zero-fill on resize
    // (the device copy overwrites every element)
    std::vector<double, NoInitAlloc<double>> vectors;
    bool complex_vectors = false;
    std::vector<Record> history;
    std::vector<double> margins;  // 4 per record (beig_result_margins)
    int iterations = 0;
    Work work;
    int64_t rr_flops = 0;
    double seconds = 0.0;
    // device-side diagnostics (not part of the reference record)
    int cgs2_fallbacks = 0;
    int max_jacobi_sweeps = 0;
    int64_t spmm_windowed = 0;  // K1 launches that ran as the window-staged K1w
    KernelStat kstats[K_CLASSES];
};

SolverConfig resolve_config(SolverConfig cfg, SolverKind kind, const StrategyConfig& s, int n);
SolveOutput solve(SolverKind kind, const SparseSym& a, const SolverConfig& cfg,
                  const StrategyConfig& s, const double* x0_colmajor, int x0_cols);

// test harness (beig_harness_*): one K4 / HL-trick call through the solver code
int harness_project_orthonormalize(const double* w, int n, int a, const double* q, int m, double* out, int device);
int harness_hl_trick(const double* s, int n, int d, const double* z, int n_now, int lock, double* x, double* p,
                     int device);

}  // namespace b2
