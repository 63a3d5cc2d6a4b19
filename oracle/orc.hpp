// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference block-eigensolver library
// (/root/reference/proj/src/{matio,kernel,rr,strategy,solvers}.cpp) used as the
// parity checker for the B200 product.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs load it; the product
// (paper_2409_05572_b200/) never links, imports or calls anything here.
//
// The reference itself cannot be built in this image (Eigen3 and its vendored
// doctest/CLI11/json are absent), so this is a restatement of
// its algorithms in plain C++ with no third-party code.  Dense arithmetic that
// the reference delegates to Eigen 3.x (GEMV/GEMM, SelfAdjointEigenSolver,
// LLT) is restated here from the published algorithms (Householder
// tridiagonalisation + implicit QL for the symmetric eigenproblem, right-looking
// Cholesky).  Summation orders inside those Eigen calls differ from Eigen's
// vectorised kernels, so agreement with the reference is to rounding, pinned by
// the reference's own known-answer tests (tests/golden/reference_known_answers.json).
//
// Everything is templated on the scalar: double (the reference) and
// std::complex<double> (Hermitian extension for config 5 — parity unpinned:
// the reference rejects complex input, proj/src/matio.cpp:102-103).
#pragma once

#include <atomic>
#include <complex>
#include <cstdint>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using cd = std::complex<double>;

inline double conj_(double x) { return x; }
inline cd conj_(cd x) { return std::conj(x); }
inline double re_(double x) { return x; }
inline double re_(cd x) { return x.real(); }
inline double abs2_(double x) { return x * x; }
inline double abs2_(cd x) { return x.real() * x.real() + x.imag() * x.imag(); }

// Column-major dense block (n rows x m columns), like the reference DenseBlock.
template <class T>
struct Mat {
    int r = 0, c = 0;
    std::vector<T> a;
    Mat() = default;
    Mat(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, T(0)) {}
    T& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
    const T& operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
    T* col(int j) { return a.data() + static_cast<size_t>(j) * r; }
    const T* col(int j) const { return a.data() + static_cast<size_t>(j) * r; }
    void resize_cols(int cols) {
        a.resize(static_cast<size_t>(r) * cols);
        c = cols;
    }
};

// Lower-triangle CSR (reference SparseSym, proj/src/matio.hpp:31-56).
template <class T>
struct Sparse {
    int n = 0;
    std::vector<int64_t> rp{0};
    std::vector<int> col;
    std::vector<T> val;
    std::shared_ptr<std::atomic<double>> norm_cache = std::make_shared<std::atomic<double>>(-1.0);

    Sparse() = default;
    Sparse(int n_, std::vector<int64_t> rp_, std::vector<int> col_, std::vector<T> val_);
    int64_t nnz_lower() const { return static_cast<int64_t>(val.size()); }
    T diagonal(int i) const;  // matio.cpp:37-43 (reverse scan)
};

class ParseError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ---- kernels (reference proj/src/kernel.cpp) ----
template <class T> std::vector<T> spmv(const Sparse<T>& a, const T* x);
template <class T> Mat<T> spmv_block(const Sparse<T>& a, const Mat<T>& x);

template <class T>
struct Ortho {
    Mat<T> q;
    int kept = 0;
};
template <class T> Ortho<T> project_orthonormalize(const Mat<T>& w, const Mat<T>& q, double drop = 1e-8);
template <class T> Ortho<T> orthonormalize(const Mat<T>& x, double drop = 1e-8);

template <class T>
struct Eig {
    std::vector<double> values;  // ascending
    Mat<T> vectors;
};
template <class T> Eig<T> sym_eig_small(const Mat<T>& h);

template <class T> Mat<T> random_block(int rows, int cols, std::mt19937_64& rng);
template <class T> double estimate_norm2(const Sparse<T>& a);

// dense helpers (deterministic; OpenMP over independent outputs only)
template <class T> Mat<T> gemm_hn(const Mat<T>& a, const Mat<T>& b);  // a^H b
template <class T> Mat<T> gemm_nn(const Mat<T>& a, const Mat<T>& b);  // a b
template <class T> double nrm2(int n, const T* x);

// ---- Rayleigh-Ritz (reference proj/src/rr.cpp) ----
template <class T>
struct Ritz {
    std::vector<double> values;
    Mat<T> vectors;
    Mat<T> coeffs;
};
template <class T> Ritz<T> rayleigh_ritz(const Sparse<T>& a, const Mat<T>& s);
template <class T> Mat<T> residual_block(const Sparse<T>& a, const Ritz<T>& rz);
struct Report {
    std::vector<double> per_pair;
    double overall = 0;
    int converged = 0;
    // decision margins (diagnostic, not in the reference): per_pair/tol of the
    // last pair inside the converged prefix and of the first pair outside it
    // (NaN when there is none)
    double lo = 0, hi = 0;
};
template <class T>
Report assess_convergence(double norm_a, const Ritz<T>& rz, const Mat<T>& r, int n_ev, double tol);

// ---- strategy (reference proj/src/strategy.cpp) ----
enum class Kind { none = 0, fix = 1, slope = 2, slopek = 3 };
enum class Decision { hold = 0, shrink = 1, expand = 2 };
struct StratCfg {
    Kind kind = Kind::none;
    int j_e = 12, j_s = 2;
    double mu = 1.1;
    int j_p = 10, j_warm = 5;
    double r_warm = 1e-4;
};
struct StratState {
    int j = 0, n_now = 0;
    std::vector<double> log10_r;
    bool shrunk_once = false;
    int last_expand_iter = -1;
    bool have_cmax = false;
    double c_max = 0.0;
    // decision margins of the last decide() (diagnostic; NaN when not evaluated):
    // r_now / r_warm of the warm-up shrink test, and the slope test's
    // (c_max - mu c) / (mu c) (c > 0) or c_max (c <= 0)
    double m_warm = 0, m_slope = 0;
};
double slope(const std::vector<double>& lr);
double slope_avg(const std::vector<double>& lr, int j_p);
void validate(const StratCfg& c);
Decision decide(StratState& st, const StratCfg& c, double r_now, int n_es, int n_ex);

// ---- solvers (reference proj/src/solvers.cpp) ----
enum class Solver { si = 0, sd = 1, lobpcg = 2, tracemin = 3 };
enum class Precond { identity = 0, diagonal = 1 };
enum class Expand { x_drop = 0, powered = 1, random = 2 };
enum class Status { converged = 0, max_iters = 1, stagnated = 2 };
enum class Event { none = 0, shrink = 1, expand = 2, lock = 3 };

struct SolverCfg {
    int n_ev = 1, n_ex = 0, n_es = 0;
    double tol = 1e-10;
    int max_iters = 2000;
    double shift = 0.0;
    int cg_iters = 5;
    Precond precond = Precond::identity;
    Expand expand = Expand::x_drop;
    uint64_t seed = 0;
    // extension: operator-mode SI (y = (c I - M) x) instead of shift-and-invert
    bool op_shifted = false;
    double op_c = 0.0;
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
template <class T>
struct Result {
    Status status = Status::max_iters;
    std::vector<double> values;
    Mat<T> vectors;
    std::vector<Record> history;
    std::vector<double> margins;  // 4 per record: rep.lo, rep.hi, st.m_warm, st.m_slope
    int iterations = 0;
    Work work;
    int64_t rr_flops = 0;
};

SolverCfg resolve_config(SolverCfg cfg, Solver kind, const StratCfg& s, int n);
template <class T>
Result<T> solve(Solver kind, const Sparse<T>& a, const SolverCfg& cfg, const StratCfg& s,
                const Mat<T>* x0);
template <class T>
std::pair<Mat<T>, Mat<T>> hl_trick(const Mat<T>& s, const Mat<T>& z, int n_now, int lock);

// Cholesky of (A - zeta I) for the reference's shift-and-invert SI: dense for
// n <= 2000 (kernel.cpp:103-108), and for n > 2000 the sparse path
// (kernel.cpp:109-134, SimplicialLLT with AMD) restated as a band (envelope)
// Cholesky in the natural order — the factor of the same matrix up to a
// symmetric permutation, so solves agree to rounding
template <class T>
struct DenseLLT {
    int n = 0;
    Mat<T> l;
    int bw = -1;          // band path: lower bandwidth
    std::vector<T> band;  // L(i, j), i - bw <= j <= i, at band[i * (bw + 1) + j - i + bw]
    DenseLLT(const Sparse<T>& a, double zeta);
    Mat<T> solve(const Mat<T>& b) const;
};

// generators (reference proj/src/matio.cpp:216-290)
Sparse<double> gen_diag(const std::vector<double>& v);
Sparse<double> gen_diag_geometric(int n, double ratio);
Sparse<double> gen_laplacian_1d(int n);
Sparse<double> gen_from_spec(const std::string& spec);
double spd_shift_value(double lambda1);
Sparse<double> apply_spd_shift(const Sparse<double>& a, double lambda1);

void set_threads(int n);

}  // namespace orc
