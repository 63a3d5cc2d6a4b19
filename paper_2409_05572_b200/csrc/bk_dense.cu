// K2 / K3 — tall-skinny dense contractions on the FP64 tensor cores (sm_100a).
//
// sm_100a has no tcgen05 f64 kind; the FP64 tensor path is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured on this pool's B200:
// 37 TFLOP/s raw DMMA, cuBLAS DGEMM 35.5 TFLOP/s (profiles/r01_fp64_peaks.json).
//
//   K2 Gram    C = X^T Y   (X n x a, Y n x b, reduce over the long n axis)
//      replaces s.transpose()*as (proj/src/rr.cpp:11) and q.transpose()*v
//      inside CGS2 (proj/src/kernel.cpp:76,79).  Split-K over n so ~2 CTAs per
//      SM are busy even when a x b is only a few 64x64 tiles; partial tiles go
//      to a workspace and are summed in a fixed split order (deterministic).
//   K3 update  Y = alpha X C + beta Y   (X n x d, C d x k)
//      replaces s*e.vectors (rr.cpp:13), s*z1 / s*o.q (solvers.cpp:195) and
//      q*(q^T v) (kernel.cpp:76,79).
//
// Both: 64x64 output tile per CTA, 8 warps each owning a 32x16 sub-tile
// (4 x 2 DMMA fragments), 16-deep K stages streamed global->shared with
// cp.async in a 3-stage ring.  Shared-memory pitches are 4 (mod 16) doubles so
// the fragment loads (lanes g=0..3, t=0..3 of a half-warp) hit 16 distinct
// 8-byte banks.
#include <algorithm>

#include "bk_common.cuh"

namespace bk {
namespace {

constexpr int TM = 64, TN = 64, TK = 16, STAGES = 3;
constexpr int PITCH_T = TM + 4;  // [TK][PITCH_T] tiles (row = k)
constexpr int PITCH_X = TK + 4;  // [TM][PITCH_X] tile of X rows in the update

// ------------------------------------------------------------------ Gram
// smem per stage: Xs[TK][PITCH_T], Ys[TK][PITCH_T]
__global__ void __launch_bounds__(256) gram_kernel(int n, const double* __restrict__ x, int ldx, int a,
                                                    const double* __restrict__ y, int ldy, int b,
                                                    double* __restrict__ out, int ldo, int rows_per_split) {
    extern __shared__ double smem[];
    double* xs = smem;                         // STAGES * TK * PITCH_T
    double* ys = smem + STAGES * TK * PITCH_T;  // STAGES * TK * PITCH_T
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int i0 = blockIdx.x * TM, j0 = blockIdx.y * TN;
    const int split = blockIdx.z;
    const int r_begin = split * rows_per_split;
    const int r_end = min(n, r_begin + rows_per_split);
    const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;

    double acc[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    const int nk = ceil_div(max(r_end - r_begin, 0), TK);
    auto load_stage = [&](int kt, int st) {
        const int r0 = r_begin + kt * TK;
        double* xd = xs + st * TK * PITCH_T;
        double* yd = ys + st * TK * PITCH_T;
#pragma unroll
        for (int e = 0; e < (TK * TM) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int rr = idx / TM, cc = idx % TM;
            const int row = r0 + rr;
            const bool okx = row < r_end && i0 + cc < a;
            const bool oky = row < r_end && j0 + cc < b;
            cp_async8(xd + rr * PITCH_T + cc, okx ? x + static_cast<size_t>(row) * ldx + i0 + cc : x, okx);
            cp_async8(yd + rr * PITCH_T + cc, oky ? y + static_cast<size_t>(row) * ldy + j0 + cc : y, oky);
        }
    };

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, st);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load_stage(nxt, nxt % STAGES);
        cp_async_commit();
        const double* xd = xs + (kt % STAGES) * TK * PITCH_T;
        const double* yd = ys + (kt % STAGES) * TK * PITCH_T;
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = xd[(k4 + t) * PITCH_T + wm + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bf[ni] = yd[(k4 + t) * PITCH_T + wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

    double* o = out + static_cast<size_t>(split) * a * ldo;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
            const int i = i0 + wm + mi * 8 + g;
            const int j = j0 + wn + ni * 8 + 2 * t;
            if (i < a) {
                if (j < b) o[static_cast<size_t>(i) * ldo + j] = acc[mi][ni][0];
                if (j + 1 < b) o[static_cast<size_t>(i) * ldo + j + 1] = acc[mi][ni][1];
            }
        }
}

// C[i][j] = sum_s work[s][i][j] in split order
__global__ void gram_reduce(int splits, int a, int b, const double* __restrict__ work,
                            double* __restrict__ c, int ldc) {
    const int64_t total = static_cast<int64_t>(a) * b;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / b), j = static_cast<int>(e % b);
        double s = 0.0;
        for (int p = 0; p < splits; ++p) s += work[static_cast<size_t>(p) * total + e];
        c[static_cast<size_t>(i) * ldc + j] = s;
    }
}

struct GramPlan {
    int splits, rows_per_split;
};

GramPlan gram_plan(int n, int a, int b) {
    const int tiles = ceil_div(a, TM) * ceil_div(b, TN);
    int splits = ceil_div(2 * kSMs, tiles);
    splits = max(1, min(splits, ceil_div(n, 4 * TK * 8)));  // >= 512 rows per split
    splits = min(splits, 64);
    int rps = ceil_div(n, splits);
    rps = ceil_div(rps, TK) * TK;
    splits = max(1, ceil_div(n, rps));
    return {splits, rps};
}

// ------------------------------------------------------------------ update
// smem per stage: Xs[TM][PITCH_X], Cs[TK][PITCH_T]
__global__ void __launch_bounds__(256) gemm_kernel(int n, const double* __restrict__ x, int ldx, int d,
                                                    const double* __restrict__ cm, int ldc, int k,
                                                    double alpha, double beta, double* __restrict__ y,
                                                    int ldy) {
    extern __shared__ double smem[];
    double* xs = smem;                            // STAGES * TM * PITCH_X
    double* cs = smem + STAGES * TM * PITCH_X;    // STAGES * TK * PITCH_T
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int r0 = blockIdx.x * TM, c0 = blockIdx.y * TN;
    const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;

    double acc[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    const int nk = ceil_div(d, TK);
    auto load_stage = [&](int kt, int st) {
        const int k0 = kt * TK;
        double* xd = xs + st * TM * PITCH_X;
        double* cd = cs + st * TK * PITCH_T;
#pragma unroll
        for (int e = 0; e < (TM * TK) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int rr = idx / TK, kk = idx % TK;
            const bool ok = r0 + rr < n && k0 + kk < d;
            cp_async8(xd + rr * PITCH_X + kk, ok ? x + static_cast<size_t>(r0 + rr) * ldx + k0 + kk : x, ok);
        }
#pragma unroll
        for (int e = 0; e < (TK * TN) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int kk = idx / TN, cc = idx % TN;
            const bool ok = k0 + kk < d && c0 + cc < k;
            cp_async8(cd + kk * PITCH_T + cc, ok ? cm + static_cast<size_t>(k0 + kk) * ldc + c0 + cc : cm, ok);
        }
    };

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, st);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load_stage(nxt, nxt % STAGES);
        cp_async_commit();
        const double* xd = xs + (kt % STAGES) * TM * PITCH_X;
        const double* cd = cs + (kt % STAGES) * TK * PITCH_T;
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = xd[(wm + mi * 8 + g) * PITCH_X + k4 + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bf[ni] = cd[(k4 + t) * PITCH_T + wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
            const int i = r0 + wm + mi * 8 + g;
            const int j = c0 + wn + ni * 8 + 2 * t;
            if (i < n) {
                double* yr = y + static_cast<size_t>(i) * ldy;
                if (j < k) yr[j] = beta == 0.0 ? alpha * acc[mi][ni][0] : fma(alpha, acc[mi][ni][0], beta * yr[j]);
                if (j + 1 < k)
                    yr[j + 1] = beta == 0.0 ? alpha * acc[mi][ni][1] : fma(alpha, acc[mi][ni][1], beta * yr[j + 1]);
            }
        }
}

constexpr size_t kGramSmem = sizeof(double) * 2 * STAGES * TK * PITCH_T;
constexpr size_t kGemmSmem = sizeof(double) * (STAGES * TM * PITCH_X + STAGES * TK * PITCH_T);

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" size_t bk_gram_work_bytes(int n, int a, int b) {
    const GramPlan p = gram_plan(max(n, 1), max(a, 1), max(b, 1));
    return static_cast<size_t>(p.splits) * max(a, 1) * max(b, 1) * sizeof(double);
}

extern "C" int bk_gram_d(int n, const double* x, int ldx, int a, const double* y, int ldy, int b,
                         double* c, int ldc, void* work, void* stream) {
    if (a <= 0 || b <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (n <= 0) {
        for (int i = 0; i < a; ++i) BK_RET(cudaMemsetAsync(c + static_cast<size_t>(i) * ldc, 0, sizeof(double) * b, s));
        return 0;
    }
    static const cudaError_t attr = cudaFuncSetAttribute(
        gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGramSmem));
    BK_RET(attr);
    const GramPlan p = gram_plan(n, a, b);
    const dim3 grid(ceil_div(a, TM), ceil_div(b, TN), p.splits);
    auto w = static_cast<double*>(work);
    gram_kernel<<<grid, 256, kGramSmem, s>>>(n, x, ldx, a, y, ldy, b, w, b, p.rows_per_split);
    const int64_t total = static_cast<int64_t>(a) * b;
    gram_reduce<<<static_cast<int>(std::min<int64_t>(ceil_div64(total, 256), 4 * kSMs)), 256, 0, s>>>(
        p.splits, a, b, w, c, ldc);
    BK_LAUNCHED();
}

extern "C" int bk_gemm_d(int n, const double* x, int ldx, int d, const double* c, int ldc, int k,
                         double alpha, double beta, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (d <= 0) {
        if (beta == 1.0) return 0;
        return bk_axpby_d(n, k, 0.0, y, ldy, beta, y, ldy, stream);
    }
    static const cudaError_t attr = cudaFuncSetAttribute(
        gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGemmSmem));
    BK_RET(attr);
    const dim3 grid(ceil_div(n, TM), ceil_div(k, TN));
    gemm_kernel<<<grid, 256, kGemmSmem, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy);
    BK_LAUNCHED();
}
