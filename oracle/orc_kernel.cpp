// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp header).
// Restates /root/reference/proj/src/kernel.cpp and matio.cpp:17-69,216-313.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>

#include "orc.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

void set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

// parallelise only when the loop body is large enough to amortise a fork
static inline bool par_ok(double work) { return work > 2e5; }

// ---------------------------------------------------------------- matrices

// invariants of reference matio.cpp:24-34
template <class T>
Sparse<T>::Sparse(int n_, std::vector<int64_t> rp_, std::vector<int> col_, std::vector<T> val_)
    : n(n_), rp(std::move(rp_)), col(std::move(col_)), val(std::move(val_)) {
    if (n < 0 || rp.size() != static_cast<size_t>(n) + 1 || col.size() != val.size() ||
        rp.back() != static_cast<int64_t>(val.size()) || rp.front() != 0)
        throw std::invalid_argument("SparseSym: inconsistent CSR arrays");
    for (int r = 0; r < n; ++r) {
        if (rp[r + 1] < rp[r]) throw std::invalid_argument("SparseSym: inconsistent CSR arrays");
        int prev = -1;
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
            if (col[p] < 0 || col[p] > r || col[p] <= prev)
                throw std::invalid_argument(
                    "SparseSym: columns must be strictly increasing and <= row");
            prev = col[p];
        }
    }
}

// matio.cpp:37-43: scan the row backwards for the diagonal entry
template <class T>
T Sparse<T>::diagonal(int i) const {
    for (int64_t p = rp[i + 1] - 1; p >= rp[i]; --p) {
        if (col[p] == i) return val[p];
        if (col[p] < i) break;
    }
    return T(0);
}

// ---------------------------------------------------------------- SpMV

// kernel.cpp:8-26 — lower CSR with the mirrored scatter.  Summation order is
// the reference's exactly: y[r] = acc_r (columns ascending) then mirrored
// contributions from later rows in ascending row order.
template <class T>
std::vector<T> spmv(const Sparse<T>& a, const T* x) {
    std::vector<T> y(static_cast<size_t>(a.n), T(0));
    for (int r = 0; r < a.n; ++r) {
        T acc = T(0);
        const T xr = x[r];
        for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) {
            const int c = a.col[p];
            const T v = a.val[p];
            acc += v * x[c];
            if (c != r) y[c] += conj_(v) * xr;  // Hermitian mirror (conj is identity for real)
        }
        y[r] += acc;
    }
    return y;
}

// kernel.cpp:28-33 — one column at a time.  Columns are independent, so the
// loop over columns is split into groups of up to 8 that share one sweep over
// the matrix; within a column every operation happens in the serial SpMV's
// order (spmv above), so the result is bit-identical to column-by-column and
// independent of the thread count.
template <class T, int G>
static void spmv_group(const Sparse<T>& a, const Mat<T>& x, Mat<T>& y, int j0) {
    const T* xc[G];
    T* yc[G];
    for (int g = 0; g < G; ++g) {
        xc[g] = x.col(j0 + g);
        yc[g] = y.col(j0 + g);
    }
    for (int r = 0; r < a.n; ++r) {
        T acc[G], xr[G];
        for (int g = 0; g < G; ++g) {
            acc[g] = T(0);
            xr[g] = xc[g][r];
        }
        for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) {
            const int c = a.col[p];
            const T v = a.val[p];
            const T vc = conj_(v);
            for (int g = 0; g < G; ++g) acc[g] += v * xc[g][c];
            if (c != r)
                for (int g = 0; g < G; ++g) yc[g][c] += vc * xr[g];
        }
        for (int g = 0; g < G; ++g) yc[g][r] += acc[g];
    }
}

template <class T>
Mat<T> spmv_block(const Sparse<T>& a, const Mat<T>& x) {
    if (x.r != a.n) throw std::invalid_argument("spmv_block: dimension mismatch");
    Mat<T> y(x.r, x.c);
    constexpr int G = 8;
    const int groups = (x.c + G - 1) / G;
#pragma omp parallel for schedule(dynamic) if (par_ok(double(a.nnz_lower()) * x.c))
    for (int gi = 0; gi < groups; ++gi) {
        const int j0 = gi * G;
        if (j0 + G <= x.c) {
            spmv_group<T, G>(a, x, y, j0);
        } else {
            for (int j = j0; j < x.c; ++j) spmv_group<T, 1>(a, x, y, j);
        }
    }
    return y;
}

// ---------------------------------------------------------------- dense helpers

template <class T>
double nrm2(int n, const T* x) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += abs2_(x[i]);
    return std::sqrt(s);
}

template <class T>
static inline T dotc(int n, const T* a, const T* b) {
    T s = T(0);
    for (int i = 0; i < n; ++i) s += conj_(a[i]) * b[i];
    return s;
}

// s[ii][jj] += conj(a_ii[k]) b_jj[k] for k in [k0, k1), ascending: BI x BJ
// independent dot products carried in registers through one sweep
template <class T, int BI, int BJ>
static inline void dot_tile(int k0, int k1, const T* const* a, const T* const* b, T (&s)[BI][BJ]) {
    for (int k = k0; k < k1; ++k) {
        T av[BI], bv[BJ];
        for (int i = 0; i < BI; ++i) av[i] = conj_(a[i][k]);
        for (int j = 0; j < BJ; ++j) bv[j] = b[j][k];
        for (int i = 0; i < BI; ++i)
            for (int j = 0; j < BJ; ++j) s[i][j] += av[i] * bv[j];
    }
}

// C = A^H B; each entry is one ascending-k dot product.  Blocked for the cache
// (row chunks of kKc: partial sums are stored in C between chunks, an exact
// round trip) and for registers (4 x 2 entries per sweep): every entry still
// accumulates its terms one at a time in ascending k — bit-identical to dotc.
template <class T>
Mat<T> gemm_hn(const Mat<T>& a, const Mat<T>& b) {
    if (a.r != b.r) throw std::invalid_argument("gemm_hn: dimension mismatch");
    Mat<T> c(a.c, b.c);
    const int n = a.r;
    constexpr int BI = 4, BJ = (sizeof(T) == 8 ? 4 : 2), kKc = 256;
    const int ni = (a.c + BI - 1) / BI, nj = (b.c + BJ - 1) / BJ;
    const bool par = par_ok(double(n) * a.c * b.c);
#pragma omp parallel if (par)
    for (int k0 = 0; k0 < n; k0 += kKc) {
        const int k1 = std::min(n, k0 + kKc);
#pragma omp for schedule(static) collapse(2)
        for (int jb = 0; jb < nj; ++jb)
            for (int ib = 0; ib < ni; ++ib) {
                const int i0 = ib * BI, j0 = jb * BJ;
                if (i0 + BI <= a.c && j0 + BJ <= b.c) {
                    const T* ap[BI];
                    const T* bp[BJ];
                    T s[BI][BJ];
                    for (int i = 0; i < BI; ++i) ap[i] = a.col(i0 + i);
                    for (int j = 0; j < BJ; ++j) bp[j] = b.col(j0 + j);
                    for (int i = 0; i < BI; ++i)
                        for (int j = 0; j < BJ; ++j) s[i][j] = c(i0 + i, j0 + j);
                    dot_tile<T, BI, BJ>(k0, k1, ap, bp, s);
                    for (int i = 0; i < BI; ++i)
                        for (int j = 0; j < BJ; ++j) c(i0 + i, j0 + j) = s[i][j];
                } else {
                    for (int j = j0; j < std::min(b.c, j0 + BJ); ++j)
                        for (int i = i0; i < std::min(a.c, i0 + BI); ++i) {
                            const T* ap[1] = {a.col(i)};
                            const T* bp[1] = {b.col(j)};
                            T s[1][1] = {{c(i, j)}};
                            dot_tile<T, 1, 1>(k0, k1, ap, bp, s);
                            c(i, j) = s[0][0];
                        }
                }
            }
    }
    return c;
}

// C = A B; each entry sums over l ascending
template <class T>
Mat<T> gemm_nn(const Mat<T>& a, const Mat<T>& b) {
    if (a.c != b.r) throw std::invalid_argument("gemm_nn: dimension mismatch");
    Mat<T> c(a.r, b.c);
    const int n = a.r;
    constexpr int kChunk = 256;
    const int nchunks = (n + kChunk - 1) / kChunk;
#pragma omp parallel for schedule(static) if (par_ok(double(n) * a.c * b.c))
    for (int ch = 0; ch < nchunks; ++ch) {
        const int i0 = ch * kChunk, i1 = std::min(n, i0 + kChunk);
        for (int j = 0; j < b.c; ++j) {
            T* cj = c.col(j);
            for (int l = 0; l < a.c; ++l) {
                const T blj = b(l, j);
                const T* al = a.col(l);
                for (int i = i0; i < i1; ++i) cj[i] += al[i] * blj;
            }
        }
    }
    return c;
}

// v -= Q (Q^H v) over the first m columns of q (Eigen: temp = Q*(Q^T v); v -= temp)
// coef[l] is one ascending-i dot product (8 of them per sweep); temp[i] sums
// over l ascending, formed for a chunk of rows at a time with l outermost
// (each temp[i] still adds its terms in ascending l) — bit-identical to the
// row-at-a-time form, with unit-stride streams through Q.
template <class T>
static void project_out(int n, const T* q, int m, T* v) {
    if (m == 0) return;
    std::vector<T> coef(static_cast<size_t>(m));
    constexpr int BL = 8;
    const int nb = (m + BL - 1) / BL;
    const T* vp[1] = {v};
#pragma omp parallel for schedule(dynamic) if (par_ok(double(n) * m))
    for (int lb = 0; lb < nb; ++lb) {
        const int l0 = lb * BL;
        if (l0 + BL <= m) {
            const T* qp[BL];
            T s[BL][1];
            for (int i = 0; i < BL; ++i) {
                qp[i] = q + static_cast<size_t>(l0 + i) * n;
                s[i][0] = T(0);
            }
            dot_tile<T, BL, 1>(0, n, qp, vp, s);
            for (int i = 0; i < BL; ++i) coef[l0 + i] = s[i][0];
        } else {
            for (int l = l0; l < m; ++l) coef[l] = dotc(n, q + static_cast<size_t>(l) * n, v);
        }
    }
    constexpr int kChunk = 512;
    const int nchunks = (n + kChunk - 1) / kChunk;
#pragma omp parallel for schedule(static) if (par_ok(double(n) * m))
    for (int ch = 0; ch < nchunks; ++ch) {
        const int i0 = ch * kChunk, i1 = std::min(n, i0 + kChunk);
        T t[kChunk];
        for (int i = 0; i < i1 - i0; ++i) t[i] = T(0);
        for (int l = 0; l < m; ++l) {
            const T* ql = q + static_cast<size_t>(l) * n + i0;
            const T cl = coef[l];
            for (int i = 0; i < i1 - i0; ++i) t[i] += ql[i] * cl;
        }
        for (int i = i0; i < i1; ++i) v[i] -= t[i - i0];
    }
}

// ---------------------------------------------------------------- CGS2

// kernel.cpp:65-89 — column-by-column classical Gram-Schmidt, two passes, with
// the drop test ||v|| < drop * ||w_j|| against the pre-projection norm.
template <class T>
Ortho<T> project_orthonormalize(const Mat<T>& w, const Mat<T>& q, double drop) {
    const int n = w.r;
    if (q.c > 0 && q.r != n)
        throw std::invalid_argument("project_orthonormalize: dimension mismatch");
    Ortho<T> o;
    o.q = Mat<T>(n, w.c);
    std::vector<T> v(static_cast<size_t>(n));
    for (int j = 0; j < w.c; ++j) {
        std::copy(w.col(j), w.col(j) + n, v.begin());
        const double ref = nrm2(n, v.data());
        if (ref == 0.0) continue;
        for (int pass = 0; pass < 2; ++pass) {
            if (q.c > 0) project_out(n, q.a.data(), q.c, v.data());
            if (o.kept > 0) project_out(n, o.q.a.data(), o.kept, v.data());
        }
        const double nrm = nrm2(n, v.data());
        if (nrm < drop * ref) continue;
        T* dst = o.q.col(o.kept);
        for (int i = 0; i < n; ++i) dst[i] = v[i] / nrm;
        ++o.kept;
    }
    o.q.resize_cols(o.kept);
    return o;
}

template <class T>
Ortho<T> orthonormalize(const Mat<T>& x, double drop) {
    return project_orthonormalize(x, Mat<T>(x.r, 0), drop);
}

// ---------------------------------------------------------------- eigensolver

// Householder reduction of a Hermitian matrix (lower triangle used) to a real
// symmetric tridiagonal T = Q^H A Q (the unblocked LAPACK ?hetd2 scheme).
// On return d/e hold the tridiagonal and the reflectors (v_k, tau_k) are kept
// for the back-transformation.
template <class T>
static void tridiagonalize(Mat<T>& a, std::vector<double>& d, std::vector<double>& e,
                           std::vector<T>& tau) {
    const int n = a.r;
    d.assign(n, 0.0);
    e.assign(n, 0.0);
    tau.assign(n, T(0));
    std::vector<T> w(static_cast<size_t>(n));
    for (int k = 0; k + 1 < n; ++k) {
        const int m = n - k - 1;  // length of x = a(k+1:n, k)
        T* x = &a(k + 1, k);
        const T alpha = x[0];
        double xnorm2 = 0.0;
        for (int i = 1; i < m; ++i) xnorm2 += abs2_(x[i]);
        const double ar = re_(alpha);
        const double ai = std::imag(std::complex<double>(alpha));
        T t(0);
        double beta;
        if (xnorm2 == 0.0 && ai == 0.0) {
            beta = ar;  // H = I
        } else {
            beta = -std::copysign(std::sqrt(ar * ar + ai * ai + xnorm2), ar);
            if constexpr (std::is_same_v<T, double>) {
                t = (beta - ar) / beta;
            } else {
                t = T((beta - ar) / beta, -ai / beta);
            }
            const T scal = T(1) / (alpha - T(beta));
            for (int i = 1; i < m; ++i) x[i] *= scal;
        }
        e[k] = beta;
        tau[k] = t;
        x[0] = T(1);
        if (t != T(0)) {
            // w = t * A22 v (A22 Hermitian, full storage kept current)
            for (int i = 0; i < m; ++i) {
                T s = T(0);
                for (int j = 0; j < m; ++j) s += a(k + 1 + i, k + 1 + j) * x[j];
                w[i] = t * s;
            }
            // w -= 1/2 t (w^H v) v
            T wv = T(0);
            for (int i = 0; i < m; ++i) wv += conj_(w[i]) * x[i];
            const T alpha2 = -0.5 * t * wv;
            for (int i = 0; i < m; ++i) w[i] += alpha2 * x[i];
            // A22 -= v w^H + w v^H
            for (int j = 0; j < m; ++j)
                for (int i = 0; i < m; ++i)
                    a(k + 1 + i, k + 1 + j) -= x[i] * conj_(w[j]) + w[i] * conj_(x[j]);
        }
    }
    for (int k = 0; k < n; ++k) d[k] = re_(a(k, k));
    e[n - 1] = 0.0;
}

// Implicit QL with shifts on the symmetric tridiagonal (d, e), accumulating the
// rotations into u (n x n, real).  e[i] couples i and i+1.
static void tridiag_ql(std::vector<double>& d, std::vector<double>& e, Mat<double>& u) {
    const int n = static_cast<int>(d.size());
    const double eps = std::numeric_limits<double>::epsilon();
    for (int l = 0; l < n; ++l) {
        int iter = 0;
        for (;;) {
            int m = l;
            for (; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= eps * dd) break;
            }
            if (m == l) break;
            if (++iter > 100) throw std::runtime_error("sym_eig_small: eigensolver failed");
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
            double s = 1.0, c = 1.0, p = 0.0;
            int i = m - 1;
            bool underflow = false;
            for (; i >= l; --i) {
                double f = s * e[i];
                const double b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    underflow = true;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * b;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - b;
                for (int k = 0; k < n; ++k) {
                    f = u(k, i + 1);
                    u(k, i + 1) = s * u(k, i) + c * f;
                    u(k, i) = c * u(k, i) - s * f;
                }
            }
            if (underflow) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        }
    }
}

// kernel.cpp:95-100 — eigendecomposition of 0.5 (H + H^H), ascending values,
// orthonormal vectors (stable order among ties).
template <class T>
Eig<T> sym_eig_small(const Mat<T>& h) {
    if (h.r != h.c) throw std::invalid_argument("sym_eig_small: matrix must be square");
    const int n = h.r;
    Mat<T> a(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) a(i, j) = 0.5 * (h(i, j) + conj_(h(j, i)));
    Eig<T> out;
    if (n == 0) return out;
    std::vector<double> d, e;
    std::vector<T> tau;
    tridiagonalize(a, d, e, tau);
    Mat<double> u(n, n);
    for (int i = 0; i < n; ++i) u(i, i) = 1.0;
    tridiag_ql(d, e, u);
    // Z = Q U with Q = H_0 H_1 ... H_{n-2}; apply reflectors right to left
    Mat<T> z(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) z(i, j) = T(u(i, j));
    for (int k = n - 2; k >= 0; --k) {
        const T t = tau[k];
        if (t == T(0)) continue;
        const int m = n - k - 1;
        const T* v = &a(k + 1, k);  // v[0] == 1
        for (int j = 0; j < n; ++j) {
            T s = T(0);
            for (int i = 0; i < m; ++i) s += conj_(v[i]) * z(k + 1 + i, j);
            s *= t;
            for (int i = 0; i < m; ++i) z(k + 1 + i, j) -= v[i] * s;
        }
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
    out.values.resize(n);
    out.vectors = Mat<T>(n, n);
    for (int k = 0; k < n; ++k) {
        out.values[k] = d[order[k]];
        std::copy(z.col(order[k]), z.col(order[k]) + n, out.vectors.col(k));
    }
    return out;
}

// ---------------------------------------------------------------- RNG / norm

// kernel.cpp:166-172 — fresh normal_distribution per call, filled column-major.
// Complex blocks draw the real part then the imaginary part of each entry.
template <class T>
Mat<T> random_block(int rows, int cols, std::mt19937_64& rng) {
    std::normal_distribution<double> dist(0.0, 1.0);
    Mat<T> x(rows, cols);
    for (int j = 0; j < cols; ++j)
        for (int i = 0; i < rows; ++i) {
            if constexpr (std::is_same_v<T, double>) {
                x(i, j) = dist(rng);
            } else {
                const double re = dist(rng);
                const double im = dist(rng);
                x(i, j) = T(re, im);
            }
        }
    return x;
}

// kernel.cpp:174-196 — 30 power steps on A^2 from a fixed seeded start, cached.
template <class T>
double estimate_norm2(const Sparse<T>& a) {
    const double cached = a.norm_cache->load(std::memory_order_relaxed);
    if (cached >= 0.0) return cached;
    const int n = a.n;
    if (n == 0) return 0.0;
    std::mt19937_64 rng(0x9e3779b97f4a7c15ULL);
    Mat<T> v0 = random_block<T>(n, 1, rng);
    std::vector<T> v(v0.a.begin(), v0.a.end());
    double nrm = nrm2(n, v.data());
    if (nrm == 0.0) return 0.0;
    for (auto& x : v) x /= nrm;
    for (int it = 0; it < 30; ++it) {
        std::vector<T> av = spmv(a, v.data());
        std::vector<T> w = spmv(a, av.data());
        nrm = nrm2(n, w.data());
        if (nrm == 0.0) {
            a.norm_cache->store(0.0, std::memory_order_relaxed);
            return 0.0;
        }
        for (int i = 0; i < n; ++i) v[i] = w[i] / nrm;
    }
    std::vector<T> av = spmv(a, v.data());
    const double est = nrm2(n, av.data());
    a.norm_cache->store(est, std::memory_order_relaxed);
    return est;
}

// ---------------------------------------------------------------- dense LLT

// kernel.cpp:102-137, dense path only (n <= 2000); the sparse AMD path is
// outside the oracle (SI on large n runs in operator mode).
template <class T>
DenseLLT<T>::DenseLLT(const Sparse<T>& a, double zeta) : n(a.n), l(a.n <= 2000 ? a.n : 0, a.n <= 2000 ? a.n : 0) {
    if (n > 2000) {
        // band Cholesky (kernel.cpp:109-134 restated; see orc.hpp)
        bw = 0;
        for (int r = 0; r < n; ++r)
            for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) bw = std::max(bw, r - a.col[p]);
        const int w = bw + 1;
        if (static_cast<double>(n) * w > 4e8) throw std::invalid_argument("oracle band Cholesky: bandwidth too large");
        band.assign(static_cast<size_t>(n) * w, T(0));
        auto L = [&](int i, int j) -> T& { return band[static_cast<size_t>(i) * w + j - i + bw]; };
        for (int r = 0; r < n; ++r)
            for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) L(r, a.col[p]) = a.val[p];
        for (int i = 0; i < n; ++i) L(i, i) -= zeta;
        for (int j = 0; j < n; ++j) {
            double djj = re_(L(j, j));
            for (int k = std::max(0, j - bw); k < j; ++k) djj -= abs2_(L(j, k));
            if (!(djj > 0.0)) throw std::runtime_error("SpdFactor: matrix is not positive definite");
            const double ljj = std::sqrt(djj);
            L(j, j) = ljj;
            for (int i = j + 1; i <= std::min(n - 1, j + bw); ++i) {
                T s = L(i, j);
                for (int k = std::max(0, i - bw); k < j; ++k) s -= L(i, k) * conj_(L(j, k));
                L(i, j) = s / ljj;
            }
        }
        return;
    }
    Mat<T> m(n, n);
    for (int r = 0; r < n; ++r)
        for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) {
            m(r, a.col[p]) = a.val[p];
            m(a.col[p], r) = conj_(a.val[p]);
        }
    for (int i = 0; i < n; ++i) m(i, i) -= zeta;
    for (int j = 0; j < n; ++j) {
        double djj = re_(m(j, j));
        for (int k = 0; k < j; ++k) djj -= abs2_(l(j, k));
        if (!(djj > 0.0)) throw std::runtime_error("SpdFactor: matrix is not positive definite");
        const double ljj = std::sqrt(djj);
        l(j, j) = ljj;
        for (int i = j + 1; i < n; ++i) {
            T s = m(i, j);
            for (int k = 0; k < j; ++k) s -= l(i, k) * conj_(l(j, k));
            l(i, j) = s / ljj;
        }
    }
}

template <class T>
Mat<T> DenseLLT<T>::solve(const Mat<T>& b) const {
    if (b.r != n) throw std::invalid_argument("SpdFactor::solve: dimension mismatch");
    Mat<T> x = b;
    if (bw >= 0) {
        const int w = bw + 1;
        auto L = [&](int i, int j) { return band[static_cast<size_t>(i) * w + j - i + bw]; };
        for (int c = 0; c < b.c; ++c) {
            T* y = x.col(c);
            for (int i = 0; i < n; ++i) {
                T s = y[i];
                for (int k = std::max(0, i - bw); k < i; ++k) s -= L(i, k) * y[k];
                y[i] = s / L(i, i);
            }
            for (int i = n - 1; i >= 0; --i) {
                T s = y[i];
                for (int k = i + 1; k <= std::min(n - 1, i + bw); ++k) s -= conj_(L(k, i)) * y[k];
                y[i] = s / L(i, i);
            }
        }
        return x;
    }
    for (int c = 0; c < b.c; ++c) {
        T* y = x.col(c);
        for (int i = 0; i < n; ++i) {  // L y = b
            T s = y[i];
            for (int k = 0; k < i; ++k) s -= l(i, k) * y[k];
            y[i] = s / l(i, i);
        }
        for (int i = n - 1; i >= 0; --i) {  // L^H x = y
            T s = y[i];
            for (int k = i + 1; k < n; ++k) s -= conj_(l(k, i)) * y[k];
            y[i] = s / l(i, i);
        }
    }
    return x;
}

// ---------------------------------------------------------------- generators

namespace {
struct Trip {
    int r, c;
    double v;
};
Sparse<double> from_trips(int n, std::vector<Trip>& ts) {
    std::sort(ts.begin(), ts.end(),
              [](const Trip& a, const Trip& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
    std::vector<int> col(ts.size());
    std::vector<double> val(ts.size());
    for (size_t i = 0; i < ts.size(); ++i) {
        rp[ts[i].r + 1]++;
        col[i] = ts[i].c;
        val[i] = ts[i].v;
    }
    for (int r = 0; r < n; ++r) rp[r + 1] += rp[r];
    return Sparse<double>(n, std::move(rp), std::move(col), std::move(val));
}
}  // namespace

Sparse<double> gen_diag(const std::vector<double>& v) {
    const int n = static_cast<int>(v.size());
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1);
    std::vector<int> col(static_cast<size_t>(n));
    for (int i = 0; i <= n; ++i) rp[i] = i;
    for (int i = 0; i < n; ++i) col[i] = i;
    return Sparse<double>(n, std::move(rp), std::move(col), v);
}

Sparse<double> gen_diag_geometric(int n, double ratio) {
    if (n < 1) throw std::invalid_argument("gen_diag_geometric: n must be positive");
    if (!(ratio > 0)) throw std::invalid_argument("gen_diag_geometric: ratio must be positive");
    std::vector<double> v(static_cast<size_t>(n));
    double x = 1.0;
    for (int i = 0; i < n; ++i, x *= ratio) v[i] = x;
    return gen_diag(v);
}

Sparse<double> gen_laplacian_1d(int n) {
    if (n < 1) throw std::invalid_argument("gen_laplacian_1d: n must be positive");
    std::vector<Trip> ts;
    for (int i = 0; i < n; ++i) {
        if (i > 0) ts.push_back({i, i - 1, -1.0});
        ts.push_back({i, i, 2.0});
    }
    return from_trips(n, ts);
}

Sparse<double> gen_from_spec(const std::string& spec) {
    const size_t colon = spec.find(':');
    if (colon == std::string::npos)
        throw std::invalid_argument("generator spec needs 'name:args', got '" + spec + "'");
    const std::string name = spec.substr(0, colon), args = spec.substr(colon + 1);
    auto parse_int = [](const std::string& s) {
        size_t pos = 0;
        const int v = std::stoi(s, &pos);
        if (pos != s.size()) throw std::invalid_argument("bad integer '" + s + "' in spec");
        return v;
    };
    auto parse_double = [](const std::string& s) {
        size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument("bad number '" + s + "' in spec");
        return v;
    };
    std::vector<std::string> parts;
    {
        std::string cur;
        for (char ch : args) {
            if (ch == ',') {
                parts.push_back(cur);
                cur.clear();
            } else {
                cur += ch;
            }
        }
        parts.push_back(cur);
    }
    if (name == "laplacian1d") return gen_laplacian_1d(parse_int(args));
    if (name == "diag") {
        std::vector<double> v;
        for (const auto& t : parts) v.push_back(parse_double(t));
        return gen_diag(v);
    }
    if (name == "diag-geom") {
        if (parts.size() != 2) throw std::invalid_argument("diag-geom needs 'diag-geom:n,ratio'");
        return gen_diag_geometric(parse_int(parts[0]), parse_double(parts[1]));
    }
    throw std::invalid_argument("unknown generator '" + name + "'");
}

double spd_shift_value(double lambda1) { return lambda1 <= 0.0 ? 1.05 * lambda1 : 0.0; }

Sparse<double> apply_spd_shift(const Sparse<double>& a, double lambda1) {
    const double shift = spd_shift_value(lambda1);
    if (shift == 0.0) return a;
    std::vector<Trip> ts;
    for (int r = 0; r < a.n; ++r) {
        bool has_diag = false;
        for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) {
            double v = a.val[p];
            if (a.col[p] == r) {
                v -= shift;
                has_diag = true;
            }
            ts.push_back({r, a.col[p], v});
        }
        if (!has_diag) ts.push_back({r, r, -shift});
    }
    return from_trips(a.n, ts);
}

// ---------------------------------------------------------------- instantiations
#define ORC_INST(T)                                                                      \
    template struct Sparse<T>;                                                           \
    template std::vector<T> spmv(const Sparse<T>&, const T*);                            \
    template Mat<T> spmv_block(const Sparse<T>&, const Mat<T>&);                         \
    template Ortho<T> project_orthonormalize(const Mat<T>&, const Mat<T>&, double);      \
    template Ortho<T> orthonormalize(const Mat<T>&, double);                             \
    template Eig<T> sym_eig_small(const Mat<T>&);                                        \
    template Mat<T> random_block<T>(int, int, std::mt19937_64&);                         \
    template double estimate_norm2(const Sparse<T>&);                                    \
    template Mat<T> gemm_hn(const Mat<T>&, const Mat<T>&);                               \
    template Mat<T> gemm_nn(const Mat<T>&, const Mat<T>&);                               \
    template double nrm2(int, const T*);                                                 \
    template struct DenseLLT<T>;
ORC_INST(double)
ORC_INST(cd)

}  // namespace orc
