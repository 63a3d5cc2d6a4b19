// K6 / K7 / K8 — residual + column norms, convergence finish, column movement.
//
// Replaces: residual_block (proj/src/rr.cpp:16-20), the norms of
// assess_convergence (rr.cpp:22-38), apply_precond (solvers.cpp:105-107) and the
// Eigen column selection / hcat copies of the solver loops (solvers.cpp:12-23).
// All reductions are two-level with a fixed order, so results are bit-stable
// run to run (the reference's determinism contract, kernel.hpp:21-23).
#include <cfloat>

#include <algorithm>

#include "bk_common.cuh"

namespace bk {
namespace {

constexpr int kRowsPerBlock = 256;
constexpr int kMaxRowBlocks = 512;

int row_blocks(int n) { return max(1, min(ceil_div(n, kRowsPerBlock), kMaxRowBlocks)); }

// column sums of squares over a row range; partial[rb][c]
__global__ void __launch_bounds__(256) colnorm2_partial(int n, const double* __restrict__ x, int ldx,
                                                         int k, double* __restrict__ partial) {
    __shared__ double red[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * 32 + tx;
    const int nb = gridDim.x;
    const int r0 = static_cast<int>((static_cast<int64_t>(n) * blockIdx.x) / nb);
    const int r1 = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.x + 1)) / nb);
    double acc = 0.0;
    if (c < k)
        for (int r = r0 + ty; r < r1; r += 8) {
            const double v = x[static_cast<size_t>(r) * ldx + c];
            acc = fma(v, v, acc);
        }
    red[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && c < k) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += red[i][tx];
        partial[static_cast<size_t>(blockIdx.x) * k + c] = s;
    }
}

// out[c] = sum_b partial[b][c]: one warp per column, lanes stride the row
// blocks, fixed butterfly — deterministic (a serial loop over 512 partials per
// thread cost ~100 us per call)
__device__ __forceinline__ double warp_colsum(int nb, int k, const double* __restrict__ partial, int c) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += partial[static_cast<size_t>(b) * k + c];
    return warp_sum(s);
}

__global__ void sum_partials(int nb, int k, const double* __restrict__ partial, double* __restrict__ out) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= k) return;
    const double s = warp_colsum(nb, k, partial, c);
    if ((threadIdx.x & 31) == 0) out[c] = s;
}

// R = AV - V diag(lambda); W = t .* R (columns >= w_from); norms of R and V
// (and, with pw, of W: the reference norms of K4's drop rule, fused here so
// the preconditioned block is not read again)
__global__ void __launch_bounds__(256) residual_partial(int n, const double* __restrict__ v, int ldv,
                                                         const double* __restrict__ av, int ldav,
                                                         const double* __restrict__ lambda, int k,
                                                         double* __restrict__ r, int ldr,
                                                         const double* __restrict__ t,
                                                         double* __restrict__ w, int ldw, int w_from,
                                                         double* __restrict__ pr, double* __restrict__ pv,
                                                         double* __restrict__ pw) {
    __shared__ double red_r[8][33];
    __shared__ double red_v[8][33];
    __shared__ double red_w[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * 32 + tx;
    const int nb = gridDim.x;
    const int r0 = static_cast<int>((static_cast<int64_t>(n) * blockIdx.x) / nb);
    const int r1 = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.x + 1)) / nb);
    double ar = 0.0, avv = 0.0, aw = 0.0;
    if (c < k) {
        const double lam = lambda[c];
        for (int i = r0 + ty; i < r1; i += 8) {
            const double vv = v[static_cast<size_t>(i) * ldv + c];
            const double rr = av[static_cast<size_t>(i) * ldav + c] - lam * vv;
            if (r) r[static_cast<size_t>(i) * ldr + c] = rr;
            if (w && c >= w_from) {
                const double ww = t ? t[i] * rr : rr;
                w[static_cast<size_t>(i) * ldw + (c - w_from)] = ww;
                aw = fma(ww, ww, aw);
            }
            ar = fma(rr, rr, ar);
            avv = fma(vv, vv, avv);
        }
    }
    red_r[ty][tx] = ar;
    red_v[ty][tx] = avv;
    red_w[ty][tx] = aw;
    __syncthreads();
    if (ty == 0 && c < k) {
        double s = 0.0, sv = 0.0, sw = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s += red_r[i][tx];
            sv += red_v[i][tx];
            sw += red_w[i][tx];
        }
        pr[static_cast<size_t>(blockIdx.x) * k + c] = s;
        pv[static_cast<size_t>(blockIdx.x) * k + c] = sv;
        if (pw) pw[static_cast<size_t>(blockIdx.x) * k + c] = sw;
    }
}

__global__ void residual_finish(int nb, int k, const double* __restrict__ pr, const double* __restrict__ pv,
                                const double* __restrict__ pw, int w_from, double* __restrict__ rn2,
                                double* __restrict__ vn2, double* __restrict__ wn2) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= k) return;
    const double s = warp_colsum(nb, k, pr, c), sv = warp_colsum(nb, k, pv, c);
    const double sw = pw && c >= w_from ? warp_colsum(nb, k, pw, c) : 0.0;
    if ((threadIdx.x & 31) == 0) {
        rn2[c] = s;
        vn2[c] = sv;
        if (pw && c >= w_from) wn2[c - w_from] = sw;
    }
}

// rr.cpp:22-38 on device; one CTA
__global__ void __launch_bounds__(1024) convergence_kernel(int k, const double* __restrict__ rn2,
                                                            const double* __restrict__ vn2,
                                                            const double* __restrict__ lambda,
                                                            double norm_a, int n_ev, double tol,
                                                            double* __restrict__ per_pair,
                                                            double* __restrict__ rec) {
    __shared__ double s_max[1024];
    __shared__ int s_first[1024];
    __shared__ int s_bad[1024];
    double mx = 0.0;
    int first = k;
    int bad = 0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const double vn = sqrt(vn2[i]);
        const double rn = sqrt(rn2[i]);
        const double denom = norm_a * vn + vn * fabs(lambda[i]);
        const double pp = denom > 0.0 ? rn / denom : rn;
        if (per_pair) per_pair[i] = pp;
        if (i < n_ev) mx = fmax(mx, pp);
        if (!(pp <= tol)) first = min(first, i);  // NaN counts as unconverged
        if (!isfinite(pp) || !isfinite(lambda[i])) bad = 1;
    }
    s_max[threadIdx.x] = mx;
    s_first[threadIdx.x] = first;
    s_bad[threadIdx.x] = bad;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + off]);
            s_first[threadIdx.x] = min(s_first[threadIdx.x], s_first[threadIdx.x + off]);
            s_bad[threadIdx.x] |= s_bad[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        rec[0] = s_max[0];
        rec[1] = static_cast<double>(s_first[0]);
        rec[2] = static_cast<double>(s_bad[0]);
        // decision margins: per_pair of the last pair inside the converged
        // prefix and of the first pair outside it (-1: none), same formula
        const int f = s_first[0];
        auto pp_at = [&](int i) {
            const double vn = sqrt(vn2[i]);
            const double denom = norm_a * vn + vn * fabs(lambda[i]);
            return denom > 0.0 ? sqrt(rn2[i]) / denom : sqrt(rn2[i]);
        };
        rec[3] = f > 0 ? pp_at(f - 1) : -1.0;
        rec[4] = f < k ? pp_at(f) : -1.0;
    }
}

// one warp per row; chunks of 32 columns moved through registers in the
// direction that makes overlapping (same-row) moves safe
__global__ void __launch_bounds__(256) copy_cols_kernel(int n, const double* src, int lds, int k,
                                                        double* dst, int ldd) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const double* s = src + static_cast<size_t>(row) * lds;
        double* d = dst + static_cast<size_t>(row) * ldd;
        const bool forward = d <= s;
        const int chunks = ceil_div(k, 32);
        for (int q = 0; q < chunks; ++q) {
            const int ch = forward ? q : chunks - 1 - q;
            const int c = ch * 32 + lane;
            double v = 0.0;
            if (c < k) v = s[c];
            __syncwarp();
            if (c < k) d[c] = v;
            __syncwarp();
        }
    }
}

__global__ void cm_to_rm_kernel(int n, int k, const double* __restrict__ cm, int ldcm,
                                double* __restrict__ rm, int ldrm) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        const int i = i0 + threadIdx.x, j = j0 + jj;
        if (i < n && j < k) tile[jj][threadIdx.x] = cm[static_cast<size_t>(j) * ldcm + i];
    }
    __syncthreads();
    for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
        const int i = i0 + ii, j = j0 + threadIdx.x;
        if (i < n && j < k) rm[static_cast<size_t>(i) * ldrm + j] = tile[threadIdx.x][ii];
    }
}

__global__ void rm_to_cm_kernel(int n, int k, const double* __restrict__ rm, int ldrm,
                                double* __restrict__ cm, int ldcm) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
        const int i = i0 + ii, j = j0 + threadIdx.x;
        if (i < n && j < k) tile[ii][threadIdx.x] = rm[static_cast<size_t>(i) * ldrm + j];
    }
    __syncthreads();
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        const int i = i0 + threadIdx.x, j = j0 + jj;
        if (i < n && j < k) cm[static_cast<size_t>(j) * ldcm + i] = tile[threadIdx.x][jj];
    }
}

__global__ void axpby_kernel(int n, int k, double a, const double* __restrict__ x, int ldx, double b,
                             double* __restrict__ y, int ldy) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), j = static_cast<int>(e % k);
        double* yp = y + static_cast<size_t>(i) * ldy + j;
        const double xv = x[static_cast<size_t>(i) * ldx + j];
        *yp = b == 0.0 ? a * xv : a * xv + b * *yp;
    }
}

__global__ void zero_rows_kernel(double* x, int ldx, int k, int r0, int r1) {
    const int64_t total = static_cast<int64_t>(r1 - r0) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = r0 + static_cast<int>(e / k), j = static_cast<int>(e % k);
        x[static_cast<size_t>(i) * ldx + j] = 0.0;
    }
}

__global__ void lincomb_kernel(int n, int k, double a, const double* x, int ldx, double b,
                               const double* y, int ldy, double* out, int ldo) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), j = static_cast<int>(e % k);
        const double xv = x[static_cast<size_t>(i) * ldx + j];
        const double yv = y[static_cast<size_t>(i) * ldy + j];
        out[static_cast<size_t>(i) * ldo + j] = a * xv + b * yv;
    }
}

__global__ void scale_rows_kernel(int n, int k, const double* __restrict__ t, const double* __restrict__ x,
                                  int ldx, double* __restrict__ y, int ldy) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), j = static_cast<int>(e % k);
        const double xv = x[static_cast<size_t>(i) * ldx + j];
        y[static_cast<size_t>(i) * ldy + j] = t ? t[i] * xv : xv;
    }
}

__global__ void __launch_bounds__(256) coldot_partial(int n, const double* __restrict__ x, int ldx,
                                                       const double* __restrict__ y, int ldy, int k,
                                                       double* __restrict__ partial) {
    __shared__ double red[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * 32 + tx;
    const int nb = gridDim.x;
    const int r0 = static_cast<int>((static_cast<int64_t>(n) * blockIdx.x) / nb);
    const int r1 = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.x + 1)) / nb);
    double acc = 0.0;
    if (c < k)
        for (int r = r0 + ty; r < r1; r += 8)
            acc = fma(x[static_cast<size_t>(r) * ldx + c], y[static_cast<size_t>(r) * ldy + c], acc);
    red[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && c < k) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += red[i][tx];
        partial[static_cast<size_t>(blockIdx.x) * k + c] = s;
    }
}

// bnorm = ||b|| per column, active = (bnorm != 0) (kernel.cpp:143-145)
__global__ void cg_init_kernel(int k, const double* rs, double* bnorm, int* active) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
        bnorm[c] = sqrt(rs[c]);
        active[c] = bnorm[c] != 0.0;
    }
}

__global__ void cg_check_kernel(int k, const double* rs, const double* bnorm, int* active, int* count) {
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        if (active[c] && sqrt(rs[c]) < 1e-14 * bnorm[c]) active[c] = 0;
        if (active[c]) atomicAdd(&cnt, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) count[0] = cnt;
}

// sh = 1: complex columns as (re, im) pairs of the real view; the CG scalars
// are per complex column (real for a Hermitian operator)
__global__ void cg_step1_kernel(int n, int k, const double* rs, const double* pap, int* active, double* x,
                                int ldx, double* r, int ldr, const double* p, int ldp, const double* ap,
                                int ldap, int sh) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), c = static_cast<int>(e % k), cs = c >> sh;
        if (!active[cs]) continue;
        if (!(pap[cs] > 0.0)) {  // kernel.cpp:153: this column's CG stops here
            active[cs] = 0;
            continue;
        }
        const double alpha = rs[cs] / pap[cs];
        x[static_cast<size_t>(i) * ldx + c] += alpha * p[static_cast<size_t>(i) * ldp + c];
        r[static_cast<size_t>(i) * ldr + c] -= alpha * ap[static_cast<size_t>(i) * ldap + c];
    }
}

__global__ void cg_deactivate_kernel(int k, const double* pap, int* active) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x)
        if (active[c] && !(pap[c] > 0.0)) active[c] = 0;
}

__global__ void cg_step2_kernel(int n, int k, const double* rs, const double* rs_new, const int* active,
                                const double* r, int ldr, double* p, int ldp, int sh) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), c = static_cast<int>(e % k), cs = c >> sh;
        if (!active[cs]) continue;
        const double beta = rs_new[cs] / rs[cs];
        double* pp = p + static_cast<size_t>(i) * ldp + c;
        *pp = r[static_cast<size_t>(i) * ldr + c] + beta * *pp;
    }
}

__global__ void cg_commit_rs(int k, double* rs, const double* rs_new, const int* active) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x)
        if (active[c]) rs[c] = rs_new[c];
}

int elem_grid(int64_t total) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div64(total, 256), kSMs * 8)));
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" size_t bk_colnorm2_work_bytes(int n, int k) {
    return static_cast<size_t>(row_blocks(n)) * static_cast<size_t>(k > 0 ? k : 1) * sizeof(double);
}

extern "C" int bk_colnorm2_d(int n, const double* x, int ldx, int k, double* out, void* work,
                             void* stream) {
    if (k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (n <= 0) {
        BK_RET(cudaMemsetAsync(out, 0, sizeof(double) * k, s));
        return 0;
    }
    const int nb = row_blocks(n);
    auto partial = static_cast<double*>(work);
    colnorm2_partial<<<dim3(nb, ceil_div(k, 32)), dim3(32, 8), 0, s>>>(n, x, ldx, k, partial);
    sum_partials<<<ceil_div(k, 8), 256, 0, s>>>(nb, k, partial, out);
    BK_LAUNCHED();
}

extern "C" size_t bk_residual_work_bytes(int n, int k) { return 3 * bk_colnorm2_work_bytes(n, k); }

extern "C" int bk_residual_w_d(int n, const double* v, int ldv, const double* av, int ldav,
                               const double* lambda, int k, double* r, int ldr, const double* t,
                               double* w, int ldw, int w_from, double* rn2, double* vn2, double* wn2,
                               void* work, void* stream) {
    if (k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const int nb = row_blocks(n);
    auto pr = static_cast<double*>(work);
    auto pv = pr + static_cast<size_t>(nb) * k;
    double* pw = w && wn2 ? pv + static_cast<size_t>(nb) * k : nullptr;
    residual_partial<<<dim3(nb, ceil_div(k, 32)), dim3(32, 8), 0, s>>>(
        n, v, ldv, av, ldav, lambda, k, r, ldr, t, w, ldw, w_from, pr, pv, pw);
    residual_finish<<<ceil_div(k, 8), 256, 0, s>>>(nb, k, pr, pv, pw, w_from, rn2, vn2, wn2);
    BK_LAUNCHED();
}

extern "C" int bk_residual_d(int n, const double* v, int ldv, const double* av, int ldav,
                             const double* lambda, int k, double* r, int ldr, const double* t,
                             double* w, int ldw, int w_from, double* rn2, double* vn2, void* work,
                             void* stream) {
    return bk_residual_w_d(n, v, ldv, av, ldav, lambda, k, r, ldr, t, w, ldw, w_from, rn2, vn2, nullptr, work,
                           stream);
}

extern "C" int bk_convergence_d(int k, const double* rn2, const double* vn2, const double* lambda,
                                double norm_a, int n_ev, double tol, double* per_pair, double* rec,
                                void* stream) {
    convergence_kernel<<<1, 1024, 0, as_stream(stream)>>>(k, rn2, vn2, lambda, norm_a, n_ev, tol,
                                                          per_pair, rec);
    BK_LAUNCHED();
}

extern "C" int bk_copy_cols_d(int n, const double* src, int lds, int k, double* dst, int ldd,
                              void* stream) {
    if (n <= 0 || k <= 0 || src == dst) return 0;
    const int grid = max(1, min(ceil_div(n, 8), kSMs * 16));
    copy_cols_kernel<<<grid, 256, 0, as_stream(stream)>>>(n, src, lds, k, dst, ldd);
    BK_LAUNCHED();
}

extern "C" int bk_cm_to_rm_d(int n, int k, const double* cm, int ldcm, double* rm, int ldrm,
                             void* stream) {
    if (n <= 0 || k <= 0) return 0;
    cm_to_rm_kernel<<<dim3(ceil_div(n, 32), ceil_div(k, 32)), dim3(32, 8), 0, as_stream(stream)>>>(
        n, k, cm, ldcm, rm, ldrm);
    BK_LAUNCHED();
}

extern "C" int bk_rm_to_cm_d(int n, int k, const double* rm, int ldrm, double* cm, int ldcm,
                             void* stream) {
    if (n <= 0 || k <= 0) return 0;
    rm_to_cm_kernel<<<dim3(ceil_div(n, 32), ceil_div(k, 32)), dim3(32, 8), 0, as_stream(stream)>>>(
        n, k, rm, ldrm, cm, ldcm);
    BK_LAUNCHED();
}

extern "C" int bk_axpby_d(int n, int k, double a, const double* x, int ldx, double b, double* y,
                          int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    axpby_kernel<<<elem_grid(static_cast<int64_t>(n) * k), 256, 0, as_stream(stream)>>>(n, k, a, x, ldx,
                                                                                       b, y, ldy);
    BK_LAUNCHED();
}

extern "C" int bk_zero_rows_d(double* x, int ldx, int k, int r0, int r1, void* stream) {
    if (r1 <= r0 || k <= 0) return 0;
    zero_rows_kernel<<<elem_grid(static_cast<int64_t>(r1 - r0) * k), 256, 0, as_stream(stream)>>>(
        x, ldx, k, r0, r1);
    BK_LAUNCHED();
}

extern "C" int bk_lincomb_d(int n, int k, double a, const double* x, int ldx, double b, const double* y,
                            int ldy, double* out, int ldo, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    lincomb_kernel<<<elem_grid(static_cast<int64_t>(n) * k), 256, 0, as_stream(stream)>>>(n, k, a, x, ldx, b,
                                                                                          y, ldy, out, ldo);
    BK_LAUNCHED();
}

extern "C" int bk_scale_rows_d(int n, int k, const double* t, const double* x, int ldx, double* y, int ldy,
                               void* stream) {
    if (n <= 0 || k <= 0) return 0;
    scale_rows_kernel<<<elem_grid(static_cast<int64_t>(n) * k), 256, 0, as_stream(stream)>>>(n, k, t, x, ldx,
                                                                                             y, ldy);
    BK_LAUNCHED();
}

extern "C" int bk_coldot_d(int n, const double* x, int ldx, const double* y, int ldy, int k, double* out,
                           void* work, void* stream) {
    if (k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (n <= 0) {
        BK_RET(cudaMemsetAsync(out, 0, sizeof(double) * k, s));
        return 0;
    }
    const int nb = row_blocks(n);
    auto partial = static_cast<double*>(work);
    coldot_partial<<<dim3(nb, ceil_div(k, 32)), dim3(32, 8), 0, s>>>(n, x, ldx, y, ldy, k, partial);
    sum_partials<<<ceil_div(k, 8), 256, 0, s>>>(nb, k, partial, out);
    BK_LAUNCHED();
}

extern "C" int bk_cg_init_d(int k, const double* rs, double* bnorm, int* active, void* stream) {
    if (k <= 0) return 0;
    cg_init_kernel<<<ceil_div(k, 256), 256, 0, as_stream(stream)>>>(k, rs, bnorm, active);
    BK_LAUNCHED();
}

extern "C" int bk_cg_check_d(int k, const double* rs, const double* bnorm, int* active, int* count,
                             void* stream) {
    cg_check_kernel<<<1, 1024, 0, as_stream(stream)>>>(k, rs, bnorm, active, count);
    BK_LAUNCHED();
}

static int cg_step1(int n, int k, const double* rs, const double* pap, int* active, double* x, int ldx, double* r,
                    int ldr, const double* p, int ldp, const double* ap, int ldap, void* stream, int sh) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const int kr = k << sh;
    cg_step1_kernel<<<elem_grid(static_cast<int64_t>(n) * kr), 256, 0, s>>>(
        n, kr, rs, pap, active, x, ldx << sh, r, ldr << sh, p, ldp << sh, ap, ldap << sh, sh);
    cg_deactivate_kernel<<<ceil_div(k, 256), 256, 0, s>>>(k, pap, active);
    BK_LAUNCHED();
}
static int cg_step2(int n, int k, double* rs, const double* rs_new, const int* active, const double* r, int ldr,
                    double* p, int ldp, void* stream, int sh) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const int kr = k << sh;
    cg_step2_kernel<<<elem_grid(static_cast<int64_t>(n) * kr), 256, 0, s>>>(n, kr, rs, rs_new, active, r,
                                                                            ldr << sh, p, ldp << sh, sh);
    cg_commit_rs<<<ceil_div(k, 256), 256, 0, s>>>(k, rs, rs_new, active);
    BK_LAUNCHED();
}

extern "C" int bk_cg_step1_d(int n, int k, const double* rs, const double* pap, int* active, double* x,
                             int ldx, double* r, int ldr, const double* p, int ldp, const double* ap, int ldap,
                             void* stream) {
    return cg_step1(n, k, rs, pap, active, x, ldx, r, ldr, p, ldp, ap, ldap, stream, 0);
}
extern "C" int bk_cg_step1_z(int n, int k, const double* rs, const double* pap, int* active, double* x,
                             int ldx, double* r, int ldr, const double* p, int ldp, const double* ap, int ldap,
                             void* stream) {
    return cg_step1(n, k, rs, pap, active, x, ldx, r, ldr, p, ldp, ap, ldap, stream, 1);
}
extern "C" int bk_cg_step2_d(int n, int k, double* rs, const double* rs_new, const int* active,
                             const double* r, int ldr, double* p, int ldp, void* stream) {
    return cg_step2(n, k, rs, rs_new, active, r, ldr, p, ldp, stream, 0);
}
extern "C" int bk_cg_step2_z(int n, int k, double* rs, const double* rs_new, const int* active,
                             const double* r, int ldr, double* p, int ldp, void* stream) {
    return cg_step2(n, k, rs, rs_new, active, r, ldr, p, ldp, stream, 1);
}

namespace bk {
namespace {
__global__ void cgs2_commit_kernel(int n, const double* __restrict__ v, const double* __restrict__ nrm2,
                                   const double* __restrict__ ref2, double drop, double* __restrict__ out, int ldo,
                                   int* __restrict__ counter, int cw) {
    // every block evaluates the (identical) decision; block 0 bumps the counter.
    // v: n x cw real view (cw = 2: one complex column), out: real view, ldo doubles
    const double r2 = *ref2, v2 = *nrm2;
    const bool keep = r2 > 0.0 && isfinite(v2) && sqrt(v2) >= drop * sqrt(r2);
    if (!keep) return;
    const int col = *counter;
    const double inv = 1.0 / sqrt(v2);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * cw; e += gridDim.x * blockDim.x)
        out[static_cast<size_t>(e / cw) * ldo + col * cw + e % cw] = v[e] * inv;
}
__global__ void counter_bump(const double* __restrict__ nrm2, const double* __restrict__ ref2, double drop,
                             int* __restrict__ counter) {
    const double r2 = *ref2, v2 = *nrm2;
    if (r2 > 0.0 && isfinite(v2) && sqrt(v2) >= drop * sqrt(r2)) *counter += 1;
}
}  // namespace
}  // namespace bk

extern "C" int bk_cgs2_commit_d(int n, const double* v, const double* nrm2, const double* ref2, double drop,
                                double* out, int ldo, int* counter, void* stream) {
    const cudaStream_t s = as_stream(stream);
    cgs2_commit_kernel<<<elem_grid(n), 256, 0, s>>>(n, v, nrm2, ref2, drop, out, ldo, counter, 1);
    counter_bump<<<1, 1, 0, s>>>(nrm2, ref2, drop, counter);
    BK_LAUNCHED();
}
extern "C" int bk_cgs2_commit_z(int n, const double* v, const double* nrm2, const double* ref2, double drop,
                                double* out, int ldo, int* counter, void* stream) {
    const cudaStream_t s = as_stream(stream);
    cgs2_commit_kernel<<<elem_grid(2 * static_cast<int64_t>(n)), 256, 0, s>>>(n, v, nrm2, ref2, drop, out, 2 * ldo,
                                                                             counter, 2);
    counter_bump<<<1, 1, 0, s>>>(nrm2, ref2, drop, counter);
    BK_LAUNCHED();
}

// "Twice is enough" test (Daniel-Gragg-Kaufman-Stewart, eta = 1/sqrt(2)) for the
// block Gram-Schmidt of K4: after pass 1, ||w_j - Q c_j||^2 = ||w_j||^2 - ||c_j||^2
// (Q orthonormal), and pass 2 is only needed when some column lost more than
// half its squared norm (eta2 = 1/2).  flag[0] = 1 requests pass 2; the pass-2
// kernels are launched unconditionally and predicated on it (bk_*_if_d), so no
// host round trip.  c: m x a coefficient block (ldc elements, cw = 2 complex).
namespace bk {
namespace {
__global__ void __launch_bounds__(1024) dgks_flag_kernel(int m, int a, const double* __restrict__ c, int ldc,
                                                          int cw, const double* __restrict__ ref2, double eta2,
                                                          int* __restrict__ flag) {
    // one warp per column, lanes over the m coefficient rows
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int need = 0;
    for (int j = wid; j < a; j += nw) {
        double s = 0.0;
        for (int l = lane; l < m; l += 32)
            for (int q = 0; q < cw; ++q) {
                const double v = c[(static_cast<size_t>(l) * ldc + j) * cw + q];
                s = fma(v, v, s);
            }
        s = warp_sum(s);
        const double r2 = ref2[j];
        if (r2 > 0.0 && !(s <= (1.0 - eta2) * r2)) need = 1;  // NaN -> pass 2
    }
    need = __syncthreads_or(need);
    if (threadIdx.x == 0) flag[0] = need;
}
}  // namespace
}  // namespace bk

extern "C" int bk_dgks_flag_d(int m, int a, const double* c, int ldc, int cw, const double* ref2, double eta2,
                              int* flag, void* stream) {
    const cudaStream_t s = as_stream(stream);
    if (a <= 0) return static_cast<int>(cudaMemsetAsync(flag, 0, sizeof(int), s));
    dgks_flag_kernel<<<1, 1024, 0, s>>>(m, a, c, ldc, cw, ref2, eta2, flag);
    BK_LAUNCHED();
}
