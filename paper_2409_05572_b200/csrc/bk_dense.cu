// K2 / K3 — tall-skinny dense contractions on the FP64 tensor cores (sm_100a).
//
// sm_100a has no tcgen05 f64 kind; the FP64 tensor path is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured on this pool's B200:
// 37 TFLOP/s raw DMMA, cuBLAS DGEMM 35.5 TFLOP/s (profiles/r01_fp64_peaks.json).
//
//   K2 Gram    C = X^T Y   (X n x a, Y n x b, reduce over the long n axis)
//      replaces s.transpose()*as (proj/src/rr.cpp:11) and q.transpose()*v
//      inside CGS2 (proj/src/kernel.cpp:76,79).  Split-K over n so ~2 CTAs per
//      SM are busy even when a x b is a handful of tiles; partial tiles go to a
//      workspace and are summed in a fixed split order (deterministic).
//   K3 update  Y = alpha X C + beta Y   (X n x d, C d x k)
//      replaces s*e.vectors (rr.cpp:13), s*z1 / s*o.q (solvers.cpp:195) and
//      q*(q^T v) (kernel.cpp:76,79).
//
// Tiles are sized to the block widths of the solver (multiples of 96 at the
// reference defaults n_ex = 1.5 n_ev): Gram 96 x 96 per CTA with 4 warps of
// 48 x 48 (36 DMMA per 4-deep k step against 12 fragment loads); update 128 rows
// x 96 columns with 4 warps of 64 x 48 (48 DMMA per k step).  Operands stream
// global -> shared with cp.async (16-byte when the view is 16-byte aligned,
// tails zero-filled) through a multi-stage ring; shared pitches are 4 (mod 16)
// doubles so fragment loads of a half-warp hit 16 distinct 8-byte banks.
#include <algorithm>
#include <cstdlib>

#include "bk_dense.cuh"

namespace bk {
namespace {

// ------------------------------------------------------------------ Gram
// Diagonal tiles of the symmetric Gram with 72 x 72 tiles of 3 warps: only the
// 45 upper 8 x 8 fragments of the 81 are computed, dealt 15 per warp by row
// fragments {0,5,7} {1,3,8} {2,4,6} (9+4+2, 8+6+1, 7+5+3); the warp role is a
// template parameter so every skip is decided at compile time.
template <int W>
struct TriRows {
    static constexpr int r0 = W == 0 ? 0 : (W == 1 ? 1 : 2);
    static constexpr int r1 = W == 0 ? 5 : (W == 1 ? 3 : 4);
    static constexpr int r2 = W == 0 ? 7 : (W == 1 ? 8 : 6);
    static constexpr int lo = r0;  // smallest row fragment: no column below it is needed
    __host__ __device__ static constexpr int row(int mi) { return mi == 0 ? r0 : (mi == 1 ? r1 : r2); }
};

template <int W, int PX, int PY, int FN>
__device__ __forceinline__ void tri_k4(double (&acc)[3][FN][2], const double* xd, const double* yd, int k4, int t,
                                       int g) {
    double af[3], bf[FN];
#pragma unroll
    for (int mi = 0; mi < 3; ++mi) af[mi] = xd[(k4 + t) * PX + TriRows<W>::row(mi) * 8 + g];
#pragma unroll
    for (int ni = TriRows<W>::lo; ni < FN; ++ni) bf[ni] = yd[(k4 + t) * PY + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 3; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni)
            if (ni >= TriRows<W>::row(mi)) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
}

template <int TM, int TN, int TK, int WM, int WN, int STAGES, bool V16, bool SYM = false>
__global__ void __launch_bounds__(WM * WN * 32) gram_kernel(int n, const double* __restrict__ x, int ldx, int a,
                                                             const double* __restrict__ y, int ldy, int b,
                                                             double* __restrict__ out, int ldo, int rows_per_split,
                                                             const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;  // device-side predication (bk_*_if_d)
    constexpr int NT = WM * WN * 32;
    constexpr int PX = TM + 4, PY = TN + 4;
    constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
    extern __shared__ __align__(16) double smem[];
    double* xs = smem;                      // STAGES x TK x PX
    double* ys = smem + STAGES * TK * PX;   // STAGES x TK x PY
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    int ti = blockIdx.x, tj = blockIdx.y;
    if constexpr (SYM) {  // blockIdx.x enumerates the upper-triangular tile pairs ti <= tj
        const int nt = ceil_div(a, TM);
        int rem = blockIdx.x;
        ti = 0;
        while (rem >= nt - ti) {
            rem -= nt - ti;
            ++ti;
        }
        tj = ti + rem;
    }
    const int i0 = ti * TM, j0 = tj * TN;
    const int split = blockIdx.z;
    const int r_begin = split * rows_per_split;
    const int r_end = min(n, r_begin + rows_per_split);
    const int wm = (warp / WN) * (TM / WM), wn = (warp % WN) * (TN / WN);
    // X^T X on a diagonal tile of the symmetric Gram (CholQR's W^T W): the Y
    // tile is the X tile — staged once, read through both fragment paths
    const bool same = SYM && ti == tj && x == y && ldx == ldy;
    constexpr bool TRI = SYM && TM == 72 && TN == 72 && WM == 3 && WN == 1;
    const bool diag = SYM && ti == tj;

    double acc[FM][FN][2];
#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    const int nk = ceil_div(max(r_end - r_begin, 0), TK);
    auto load_stage = [&](int kt, int st) {
        const int r0 = r_begin + kt * TK;
        load_tile<V16, TK, TM, NT>(xs + st * TK * PX, PX, x, ldx, r0, r_end, i0, a, tid);
        if (!same) load_tile<V16, TK, TN, NT>(ys + st * TK * PY, PY, y, ldy, r0, r_end, j0, b, tid);
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, st);
        cp_async_commit();
    }
    // the k loop, with the per-stage compute as a parameter: the diagonal tiles'
    // warp roles select their loop once, outside it (a role branch inside every
    // k-step was 15 % of the stall samples, ncu source page)
    auto k_loop = [&](auto&& compute) {
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) load_stage(nxt, nxt % STAGES);
            cp_async_commit();
            const double* xd = xs + (kt % STAGES) * TK * PX;
            const double* yd = same ? xd : ys + (kt % STAGES) * TK * PY;
            compute(xd, yd);
        }
    };
    auto generic = [&](const double* xd, const double* yd) {
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double af[FM], bf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) af[mi] = xd[(k4 + t) * PX + wm + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) bf[ni] = yd[(k4 + t) * PY + wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    };
    if constexpr (TRI) {
        if (diag) {
            if (warp == 0)
                k_loop([&](const double* xd, const double* yd) {
#pragma unroll
                    for (int k4 = 0; k4 < TK; k4 += 4) tri_k4<0, PX, PY, FN>(acc, xd, yd, k4, t, g);
                });
            else if (warp == 1)
                k_loop([&](const double* xd, const double* yd) {
#pragma unroll
                    for (int k4 = 0; k4 < TK; k4 += 4) tri_k4<1, PX, PY, FN>(acc, xd, yd, k4, t, g);
                });
            else
                k_loop([&](const double* xd, const double* yd) {
#pragma unroll
                    for (int k4 = 0; k4 < TK; k4 += 4) tri_k4<2, PX, PY, FN>(acc, xd, yd, k4, t, g);
                });
        } else {
            k_loop(generic);
        }
    } else {
        k_loop(generic);
    }
    cp_async_wait<0>();

    double* o = out + static_cast<size_t>(split) * a * ldo;
    if constexpr (TRI) {
        if (diag) {  // computed upper fragments, each also written at its mirror position
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) {
                const int rf = warp == 0 ? TriRows<0>::row(mi) : (warp == 1 ? TriRows<1>::row(mi) : TriRows<2>::row(mi));
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) {
                    if (ni < rf) continue;
                    const int i = i0 + rf * 8 + g;
                    const int j = j0 + ni * 8 + 2 * t;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int jj = j + h;
                        if (i < a && jj < b) {
                            o[static_cast<size_t>(i) * ldo + jj] = acc[mi][ni][h];
                            if (ni > rf) o[static_cast<size_t>(jj) * ldo + i] = acc[mi][ni][h];
                        }
                    }
                }
            }
            return;
        }
    }
#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const int i = i0 + wm + mi * 8 + g;
            const int j = j0 + wn + ni * 8 + 2 * t;
            if (i < a) {
                if (j < b) o[static_cast<size_t>(i) * ldo + j] = acc[mi][ni][0];
                if (j + 1 < b) o[static_cast<size_t>(i) * ldo + j + 1] = acc[mi][ni][1];
            }
        }
}

// C[i][j] = sum_s work[s][i][j] in a fixed order; with `sym`, entries of the
// strictly-lower tiles (never computed) are mirrored from the upper ones
// (tile-level: an element-wise mirror reads the partials with stride b — one
// 69 x 69 Gram over 293 splits 137 -> 230 us)
__global__ void __launch_bounds__(256) gram_reduce(int splits, int a, int b, const double* __restrict__ work,
                                                    double* __restrict__ c, int ldc, int sym, int tile,
                                                    const int* __restrict__ run_if) {
    // 32 outputs per CTA (coalesced along the partial tiles), the splits dealt
    // to 8 fixed contiguous groups summed in split order, the group sums added
    // in group order: deterministic, and 8 loads in flight per output instead
    // of one serial chain over all splits
    if (run_if && *run_if == 0) return;
    __shared__ double red[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t total = static_cast<int64_t>(a) * b;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * 32 + tx;
    int i = 0, j = 0;
    int64_t src = 0;
    if (e < total) {
        i = static_cast<int>(e / b);
        j = static_cast<int>(e % b);
        src = sym && i / tile > j / tile ? static_cast<int64_t>(j) * b + i : e;
    }
    const int p0 = static_cast<int>(static_cast<int64_t>(splits) * ty / 8);
    const int p1 = static_cast<int>(static_cast<int64_t>(splits) * (ty + 1) / 8);
    double sacc = 0.0;
    if (e < total)
        for (int p = p0; p < p1; ++p) sacc += work[static_cast<size_t>(p) * total + src];
    red[ty][tx] = sacc;
    __syncthreads();
    if (ty == 0 && e < total) {
        double t = red[0][tx];
#pragma unroll
        for (int g = 1; g < 8; ++g) t += red[g][tx];
        c[static_cast<size_t>(i) * ldc + j] = t;
    }
}

constexpr int GTM = 96, GTN = 96, GTK = 16, GWM = 2, GWN = 2, GST = 4;

// ------------------------------------------------------------------ update
template <int TM, int TN, int TK, int WM, int WN, int STAGES, bool V16, bool V16C>
__global__ void __launch_bounds__(WM * WN * 32) gemm_kernel(int n, const double* __restrict__ x, int ldx, int d,
                                                             const double* __restrict__ cm, int ldc, int k,
                                                             double alpha, double beta, double* __restrict__ y,
                                                             int ldy, const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    constexpr int NT = WM * WN * 32;
    constexpr int PX = TK + 4, PC = TN + 4;
    constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
    extern __shared__ __align__(16) double smem[];
    double* xs = smem;                     // STAGES x TM x PX
    double* cs = smem + STAGES * TM * PX;  // STAGES x TK x PC
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    // 1-D grid, the column tiles of a row panel adjacent: the CTAs that share X rows
    // run together, so X is read from DRAM once (a 2-D grid read it once per column
    // tile: 1.26x the algorithmic bytes on config 2's two-tile lifts)
    const int nct = ceil_div(k, TN);
    const int r0 = (blockIdx.x / nct) * TM, c0 = (blockIdx.x % nct) * TN;
    const int wm = (warp / WN) * (TM / WM), wn = (warp % WN) * (TN / WN);

    double acc[FM][FN][2];
#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    const int nk = ceil_div(d, TK);
    auto load_stage = [&](int kt, int st) {
        const int k0 = kt * TK;
        load_rows<V16>(xs + st * TM * PX, PX, x, ldx, r0, n, k0, d, TM, TK, tid, NT);
        load_rows<V16C>(cs + st * TK * PC, PC, cm, ldc, k0, d, c0, k, TK, TN, tid, NT);
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
        const double* xd = xs + (kt % STAGES) * TM * PX;
        const double* cd = cs + (kt % STAGES) * TK * PC;
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double af[FM], bf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) af[mi] = xd[(wm + mi * 8 + g) * PX + k4 + t];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) bf[ni] = cd[(k4 + t) * PC + wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
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

constexpr int UTM = 128, UTN = 96, UTK = 16, UWM = 2, UWN = 2, UST = 3;

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" size_t bk_gram_work_bytes(int n, int a, int b) {
    // partials = splits x a' x b' for any call with a' <= a, b' <= b: at most the
    // budget of gram_plan (monotone in a, b), and splits <= n / 256 + 1
    const size_t small = (static_cast<size_t>(ceil_div(max(n, 1), 256)) + 1) * max(a, 1) * max(b, 1);
    return std::min(gram_budget(n, a, b), small) * sizeof(double);
}

namespace bk {
namespace {
template <int TK, int WM, int WN, int ST, int CPS, bool SYM, int TM = GTM, int TN = GTN>
int gram_launch_v(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                  void* work, cudaStream_t s, const int* run_if) {
    static_assert(!SYM || TM == TN, "symmetric tiles are square");
    constexpr size_t smem = sizeof(double) * ST * TK * ((TM + 4) + (TN + 4));
    auto k16 = gram_kernel<TM, TN, TK, WM, WN, ST, true, SYM>;
    auto k8 = gram_kernel<TM, TN, TK, WM, WN, ST, false, SYM>;
    const cudaError_t a1 = BK_ONCE_PER_DEVICE(prep(k16, smem));
    const cudaError_t a2 = BK_ONCE_PER_DEVICE(prep(k8, smem));
    BK_RET(a1);
    BK_RET(a2);
    const int nt = ceil_div(a, TM);
    const int tiles = SYM ? nt * (nt + 1) / 2 : nt * ceil_div(b, TN);
    // plan with the number of tiles actually launched
    const GramPlan p = gram_plan(n, tiles, a, b, CPS, TK);
    const dim3 grid(SYM ? tiles : nt, SYM ? 1 : ceil_div(b, TN), p.splits);
    auto w = static_cast<double*>(work);
    const bool direct = p.splits == 1 && !SYM;  // a single split writes C directly
    double* dst = direct ? c : w;
    const int ldo = direct ? ldc : b;
    if (aligned16(x, ldx) && aligned16(y, ldy))
        k16<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, a, y, ldy, b, dst, ldo, p.rows_per_split, run_if);
    else
        k8<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, a, y, ldy, b, dst, ldo, p.rows_per_split, run_if);
    if (!direct) {
        const int64_t total = static_cast<int64_t>(a) * b;
        gram_reduce<<<static_cast<int>(ceil_div64(total, 32)), 256, 0, s>>>(
            p.splits, a, b, w, c, ldc, SYM ? 1 : 0, TM, run_if);
    }
    BK_LAUNCHED();
}

// tile width (72 or 96) that wastes the least of a block width x: the solver's
// widths are multiples of n_ex and n_es (96 and 69 at config 2), and a 69-wide
// block in a 96-wide tile leaves 28 % of the DMMA work idle
inline bool narrow_tile(int x) {
    // the 72-wide tiles run ~25 % below the 96-wide ones per tile, so they only
    // pay when they cut the padding by more than a quarter of the width
    const int w96 = ceil_div(x, 96) * 96 - x, w72 = ceil_div(x, 72) * 72 - x;
    return 4 * (w96 - w72) > x;
}

// BK_GRAM_VARIANT selects a tile shape for tuning runs (default 0)
int gram_variant() {
    static const int v = [] {
        const char* e = getenv("BK_GRAM_VARIANT");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <bool SYM>
int gram_launch(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                void* work, cudaStream_t s, const int* run_if = nullptr) {
    switch (gram_variant()) {
        // measured at n = 262144 (tools/tune_dense.sh): 288^2 / 288x96 / 192x96 / 96^2 TF/s
        case 1:  // 8 warps of 48 x 24, 32-deep k steps, 3 stages, 1 CTA / SM: 23.8 / 23.8 / 23.6 / 21.7
            return gram_launch_v<32, 2, 4, 3, 1, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        case 2:  // 8 warps of 48 x 24, 4 stages: 28.3 / 27.7 / 26.9 / 22.5
            return gram_launch_v<16, 2, 4, 4, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        case 3:  // 8 warps of 48 x 24, 3 stages: 28.2 / 27.5 / 26.8 / 22.4
            return gram_launch_v<16, 2, 4, 3, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        case 4:  // 4 warps of 48 x 48, 32-deep, 3 stages, 1 CTA / SM: 24.6 / 24.5 / 24.3 / 22.2
            return gram_launch_v<32, 2, 2, 3, 1, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        default: {  // 4 warps of 48 x 48 (36 DMMA per 12 fragment loads), 4 stages, 2 CTAs / SM:
                    // 30.3 / 29.6 / 28.8 / 24.4; 72-wide tiles (24-wide warp tiles) for widths
                    // that fit them better
            const bool na = narrow_tile(a), nb = narrow_tile(b);
            // BK_NARROW: warp layout of the 72-wide tiles (tuning runs).  Default 2:
            // 72 x 72 tiles at 4 CTAs per SM, n = 262144 (tools/dense_probe.py):
            // 138 x 69 18.8 -> 21.1 TF/s, symmetric 207 14.8 -> 17.9 TF/s
            static const int nv = [] {
                const char* e = getenv("BK_NARROW");
                return e ? atoi(e) : 2;
            }();
            if (nv == 0) {
                if (SYM) {
                    if (na) return gram_launch_v<GTK, 3, 3, GST, 2, SYM, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work,
                                                                                s, run_if);
                } else if (na && nb) {
                    return gram_launch_v<GTK, 3, 3, GST, 2, false, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                } else if (nb) {
                    return gram_launch_v<GTK, 2, 3, GST, 2, false, 96, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                } else if (na) {
                    return gram_launch_v<GTK, 3, 2, GST, 2, false, 72, 96>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                }
            } else if (nv == 2 || nv == 3) {
                // 72 x 72 tiles of 3 warps at 4 (nv 2: 8-deep k steps) or 3 (nv 3) CTAs
                // per SM, so the 4 SM sub-partitions carry equal warp counts
                if (na && (SYM || nb)) {
                    if (nv == 2)
                        return gram_launch_v<8, 3, 1, 4, 4, SYM, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                        run_if);
                    return gram_launch_v<16, 3, 1, 3, 3, SYM, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                     run_if);
                }
                if (!SYM && nb)
                    return gram_launch_v<GTK, 4, 1, GST, 2, false, 96, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                if (!SYM && na)
                    return gram_launch_v<GTK, 1, 4, GST, 2, false, 72, 96>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
            } else {  // full-width warp tiles along the 72 side: 27 DMMA per 12 fragment loads
                if (SYM) {
                    if (na) return gram_launch_v<GTK, 3, 1, GST, 2, SYM, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work,
                                                                                s, run_if);
                } else if (na && nb) {
                    return gram_launch_v<GTK, 3, 1, GST, 2, false, 72, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                } else if (nb) {
                    return gram_launch_v<GTK, 4, 1, GST, 2, false, 96, 72>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                } else if (na) {
                    return gram_launch_v<GTK, 1, 4, GST, 2, false, 72, 96>(n, x, ldx, a, y, ldy, b, c, ldc, work, s,
                                                                          run_if);
                }
            }
            return gram_launch_v<GTK, GWM, GWN, GST, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        }
    }
}
}  // namespace
}  // namespace bk

// ------------------------------------------------------------------ single-column forms
// X^T v and X c for one vector (the exact column CGS2 of K4's fallback): HBM-bound
// GEMV shapes, where a 96 x 96 DMMA tile would waste 95 % of its work.
namespace bk {
namespace {
constexpr int kGvRows = 256, kGvMaxBlocks = 512;

__global__ void __launch_bounds__(256) xtv_partial(int n, const double* __restrict__ x, int ldx, int a,
                                                   const double* __restrict__ v, int ldv,
                                                   double* __restrict__ partial) {
    __shared__ double red[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * 32 + tx;
    const int nb = gridDim.x;
    const int r0 = static_cast<int>((static_cast<int64_t>(n) * blockIdx.x) / nb);
    const int r1 = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.x + 1)) / nb);
    double acc = 0.0;
    if (c < a)
        for (int r = r0 + ty; r < r1; r += 8) acc = fma(x[static_cast<size_t>(r) * ldx + c], v[static_cast<size_t>(r) * ldv], acc);
    red[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && c < a) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += red[i][tx];
        partial[static_cast<size_t>(blockIdx.x) * a + c] = s;
    }
}

__global__ void xtv_finish(int nb, int a, const double* __restrict__ partial, double* __restrict__ out, int ldo) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (c >= a) return;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += partial[static_cast<size_t>(b) * a + c];
    s = warp_sum(s);
    if (lane == 0) out[static_cast<size_t>(c) * ldo] = s;
}

// y[i] = alpha (x[i, 0:d] . c) + beta y[i], warp per row
__global__ void __launch_bounds__(256) xc_kernel(int n, const double* __restrict__ x, int ldx, int d,
                                                 const double* __restrict__ cv, int ldc, double alpha, double beta,
                                                 double* __restrict__ y, int ldy) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const double* xr = x + static_cast<size_t>(i) * ldx;
        double s = 0.0;
        for (int q = lane; q < d; q += 32) s = fma(xr[q], cv[static_cast<size_t>(q) * ldc], s);
        s = warp_sum(s);
        if (lane == 0) {
            double* yi = y + static_cast<size_t>(i) * ldy;
            *yi = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *yi);
        }
    }
}
// ------------------------------------------------------------------ short-axis forms
// Contractions over a short axis (n <= kSmallN: the coefficient-space Grams and
// lifts of the HL trick and of K5's cluster orthonormalisation, n = d <= 3k) are a
// few MFLOP: a DMMA tile walks the rows serially on one or two SMs (~27 us for
// 207 x 69 x 69).  Here 32 x 32 output tiles per CTA, the contraction axis in
// 32-deep chunks staged through shared memory (the next chunk prefetched into
// registers while the current one is consumed), each thread 4 outputs summed
// in a fixed order (deterministic).

// C[i][j] = sum_r X[r][i] Y[r][j]; sym: tiles below the diagonal skipped, the
// upper triangle mirrored (exactly symmetric)
__global__ void __launch_bounds__(256) gram_small_kernel(int n, const double* __restrict__ x, int ldx, int a,
                                                          const double* __restrict__ y, int ldy, int b,
                                                          double* __restrict__ c, int ldc, int sym,
                                                          const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    if (sym && i0 > j0) return;
    __shared__ double xs[32][33], ys[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const bool xi = i0 + tx < a, yj = j0 + tx < b;
    double px[4], py[4], acc[4] = {0.0, 0.0, 0.0, 0.0};
    auto fetch = [&](int r0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = r0 + ty + 8 * q;
            px[q] = r < n && xi ? x[static_cast<size_t>(r) * ldx + i0 + tx] : 0.0;
            py[q] = r < n && yj ? y[static_cast<size_t>(r) * ldy + j0 + tx] : 0.0;
        }
    };
    fetch(0);
    for (int r0 = 0; r0 < n; r0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            xs[ty + 8 * q][tx] = px[q];
            ys[ty + 8 * q][tx] = py[q];
        }
        __syncthreads();
        if (r0 + 32 < n) fetch(r0 + 32);
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const double yv = ys[rr][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(xs[rr][ty + 8 * q], yv, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < a && j < b && (!sym || i <= j)) {
            c[static_cast<size_t>(i) * ldc + j] = acc[q];
            if (sym && i != j) c[static_cast<size_t>(j) * ldc + i] = acc[q];
        }
    }
}

// Y[r][j] = alpha sum_q X[r][q] C[q][j] + beta Y[r][j]
__global__ void __launch_bounds__(256) gemm_small_kernel(int n, const double* __restrict__ x, int ldx, int d,
                                                          const double* __restrict__ cm, int ldc, int k,
                                                          double alpha, double beta, double* __restrict__ y,
                                                          int ldy, const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    const int r0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    __shared__ double xs[32][33], cs[32][33];  // xs[q][row], cs[q][col]
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double px[4], pc[4], acc[4] = {0.0, 0.0, 0.0, 0.0};
    auto fetch = [&](int q0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int rr = ty + 8 * u;  // X: row r0 + rr, column q0 + tx (coalesced along q)
            px[u] = r0 + rr < n && q0 + tx < d ? x[static_cast<size_t>(r0 + rr) * ldx + q0 + tx] : 0.0;
            // C: row q0 + rr, column j0 + tx
            pc[u] = q0 + rr < d && j0 + tx < k ? cm[static_cast<size_t>(q0 + rr) * ldc + j0 + tx] : 0.0;
        }
    };
    fetch(0);
    for (int q0 = 0; q0 < d; q0 += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xs[tx][ty + 8 * u] = px[u];
            cs[ty + 8 * u][tx] = pc[u];
        }
        __syncthreads();
        if (q0 + 32 < d) fetch(q0 + 32);
#pragma unroll 8
        for (int qq = 0; qq < 32; ++qq) {
            const double cv = cs[qq][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(xs[qq][ty + 8 * u], cv, acc[u]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int r = r0 + ty + 8 * u, j = j0 + tx;
        if (r < n && j < k) {
            double* yr = y + static_cast<size_t>(r) * ldy + j;
            *yr = beta == 0.0 ? alpha * acc[u] : fma(alpha, acc[u], beta * *yr);
        }
    }
}

int gram_small(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc, bool sym,
               cudaStream_t s, const int* run_if) {
    gram_small_kernel<<<dim3(ceil_div(b, 32), ceil_div(a, 32)), 256, 0, s>>>(n, x, ldx, a, y, ldy, b, c, ldc,
                                                                             sym ? 1 : 0, run_if);
    BK_LAUNCHED();
}

int gemm_small(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
               double* y, int ldy, cudaStream_t s, const int* run_if) {
    gemm_small_kernel<<<dim3(ceil_div(k, 32), ceil_div(n, 32)), 256, 0, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta,
                                                                             y, ldy, run_if);
    BK_LAUNCHED();
}
}  // namespace
}  // namespace bk

extern "C" int bk_gram_d(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                         int ldc, void* work, void* stream) {
    if (a <= 0 || b <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (n <= 0) {
        for (int i = 0; i < a; ++i) BK_RET(cudaMemsetAsync(c + static_cast<size_t>(i) * ldc, 0, sizeof(double) * b, s));
        return 0;
    }
    if (n <= kSmallN) return gram_small(n, x, ldx, a, y, ldy, b, c, ldc, false, s, nullptr);
    if (b == 1 && n >= 4096) {  // X^T v (work: row blocks x a <= bk_gram_work_bytes(n, a, 1))
        const int nb = max(1, min(ceil_div(n, kGvRows), kGvMaxBlocks));
        auto partial = static_cast<double*>(work);
        xtv_partial<<<dim3(nb, ceil_div(a, 32)), dim3(32, 8), 0, s>>>(n, x, ldx, a, y, ldy, partial);
        xtv_finish<<<ceil_div(a, 8), 256, 0, s>>>(nb, a, partial, c, ldc);
        BK_LAUNCHED();
    }
    return gram_launch<false>(n, x, ldx, a, y, ldy, b, c, ldc, work, s);
}

extern "C" int bk_gram_sym_d(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c, int ldc,
                             void* work, void* stream) {
    if (d <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    if (n <= 0) return bk_gram_d(n, x, ldx, d, y, ldy, d, c, ldc, work, stream);
    if (n <= kSmallN) return gram_small(n, x, ldx, d, y, ldy, d, c, ldc, true, s, nullptr);
    return gram_launch<true>(n, x, ldx, d, y, ldy, d, c, ldc, work, s);
}

namespace bk {
namespace {
template <int TM, int TN, int TK, int WM, int WN, int ST>
int gemm_launch_v(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
                  double* y, int ldy, cudaStream_t s, const int* run_if) {
    constexpr size_t smem = sizeof(double) * ST * (TM * (TK + 4) + TK * (TN + 4));
    auto k16 = gemm_kernel<TM, TN, TK, WM, WN, ST, true, false>;
    auto k16c = gemm_kernel<TM, TN, TK, WM, WN, ST, true, true>;
    auto k8 = gemm_kernel<TM, TN, TK, WM, WN, ST, false, false>;
    const cudaError_t a1 = BK_ONCE_PER_DEVICE(prep(k16, smem));
    const cudaError_t a2 = BK_ONCE_PER_DEVICE(prep(k8, smem));
    const cudaError_t a3 = BK_ONCE_PER_DEVICE(prep(k16c, smem));
    BK_RET(a1);
    BK_RET(a2);
    BK_RET(a3);
    const dim3 grid(ceil_div(n, TM) * ceil_div(k, TN));
    // 16-byte copies of C too when its view allows them (fewer copy instructions)
    if (aligned16(x, ldx) && aligned16(c, ldc))
        k16c<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, run_if);
    else if (aligned16(x, ldx))
        k16<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, run_if);
    else
        k8<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, run_if);
    BK_LAUNCHED();
}

// BK_GEMM_VARIANT selects a tile shape for tuning runs (default 0)
int gemm_launch(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
                double* y, int ldy, cudaStream_t s, const int* run_if) {
    static const int v = [] {
        const char* e = getenv("BK_GEMM_VARIANT");
        return e ? atoi(e) : 0;
    }();
    switch (v) {
        // n = 262144 (tools/tune_dense.sh), 288x192 / 288x96 / 192x96 / 96x96 TF/s
        case 1:  // 32-deep, 1 CTA / SM: 23.7 / 23.5 / 22.6 / 20.0
            return gemm_launch_v<128, 96, 32, 4, 2, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 2:  // 4 stages: 21.3 / 21.1 / 20.3 / 18.2
            return gemm_launch_v<128, 96, 16, 4, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 3:  // 64-row tiles: 24.1 / 23.9 / 22.7 / 19.5
            return gemm_launch_v<64, 96, 16, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 4:  // 8 warps of 32 x 48 (the round-1 first shape): 27.8 / 27.4 / 26.0 / 22.5
            return gemm_launch_v<128, 96, 16, 4, 2, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        default:  // 4 warps of 64 x 48: 28.3 / 28.1 / 26.3 / 22.2; 72-wide output tiles when they fit k better
            if (narrow_tile(k)) {
                // BK_GEMM_NARROW: 72-wide tile shape (tuning runs).  Default: 64-row
                // tiles at 4 CTAs per SM for short contractions (d <= 144: 138 -> 69
                // with beta = 1 373 -> 338 us, 69 -> 69 144 -> 130 us), 128-row tiles
                // otherwise (207 -> 138: 613 vs 618 us)
                static const int nv_env = [] {
                    const char* e = getenv("BK_GEMM_NARROW");
                    return e ? atoi(e) : 0;
                }();
                // default: 64-row tiles of 6 warps of 32 x 24 (24 accumulators per
                // thread, ~70 registers: 4 CTAs = 24 warps per SM); 138 -> 69 with
                // beta = 1 313 -> 238 us, 207 -> 138 572 -> 556 us (dense_probe)
                const int nv = nv_env ? nv_env : 5;
                if (nv == 2)  // 8-deep k steps, 4 stages: 3 CTAs per SM
                    return gemm_launch_v<128, 72, 8, 2, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
                if (nv == 3)  // 256-row tiles of 12 warps
                    return gemm_launch_v<256, 72, 16, 4, 3, 2>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                               run_if);
                if (nv == 4)  // 64-row tiles of 3 warps, 8-deep, 4 stages: 4 CTAs per SM
                    return gemm_launch_v<64, 72, 8, 1, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
                if (nv == 5)  // 64-row tiles of 6 warps of 32 x 24 (half the accumulators per thread)
                    return gemm_launch_v<64, 72, 8, 2, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
                if (nv == 6)  // 128-row tiles of 12 warps of 32 x 24
                    return gemm_launch_v<128, 72, 8, 4, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                              run_if);
                if (nv == 7)  // 64-row tiles of 6 warps, 16-deep, 3 stages
                    return gemm_launch_v<64, 72, 16, 2, 3, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                              run_if);
                return gemm_launch_v<128, 72, 16, 2, 3, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
            }
            {
                // BK_GEMM_WIDE: 96-wide tile shape (tuning runs).  Default: 64-row tiles
                // of 6 warps of 32 x 32 for short contractions (192 -> 96 with beta = 1
                // 555 -> 419 us, 96 -> 96 214 -> 192 us), 128-row tiles of 4 warps of
                // 64 x 48 for long ones (288 -> 192: 996 vs 1023 us)
                static const int wv_env = [] {
                    const char* e = getenv("BK_GEMM_WIDE");
                    return e ? atoi(e) : 0;
                }();
                const int wv = wv_env ? wv_env : (d <= 200 ? 2 : 1);
                if (wv == 2)  // 64-row tiles of 6 warps of 32 x 32
                    return gemm_launch_v<64, 96, 8, 2, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
                if (wv == 3)  // 128-row tiles of 12 warps of 32 x 32
                    return gemm_launch_v<128, 96, 8, 4, 3, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                              run_if);
                if (wv == 4)  // 64-row tiles of 6 warps, 16-deep, 3 stages
                    return gemm_launch_v<64, 96, 16, 2, 3, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                              run_if);
            }
            return gemm_launch_v<UTM, UTN, UTK, UWM, UWN, UST>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s,
                                                               run_if);
    }
}
}  // namespace
}  // namespace bk

extern "C" int bk_gemm_d(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                         double beta, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    if (d <= 0) {
        if (beta == 1.0) return 0;
        return bk_axpby_d(n, k, 0.0, y, ldy, beta, y, ldy, stream);
    }
    if (n <= kSmallN) return gemm_small(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, as_stream(stream), nullptr);
    if (k == 1 && n >= 4096) {  // X c for one column: a GEMV
        xc_kernel<<<max(1, min(ceil_div(n, 8), kSMs * 16)), 256, 0, as_stream(stream)>>>(n, x, ldx, d, c, ldc, alpha,
                                                                                         beta, y, ldy);
        BK_LAUNCHED();
    }
    return gemm_launch(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, as_stream(stream), nullptr);
}

// predicated variants: the launch is unconditional (no host round trip), the
// kernels return at once unless *run_if != 0 (device flag, e.g. bk_dgks_flag_d)
extern "C" int bk_gram_if_d(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                            int ldc, void* work, const int* run_if, void* stream) {
    if (a <= 0 || b <= 0 || n <= 0) return 0;
    if (n <= kSmallN) return gram_small(n, x, ldx, a, y, ldy, b, c, ldc, false, as_stream(stream), run_if);
    return gram_launch<false>(n, x, ldx, a, y, ldy, b, c, ldc, work, as_stream(stream), run_if);
}

extern "C" int bk_gemm_if_d(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                            double beta, double* y, int ldy, const int* run_if, void* stream) {
    if (n <= 0 || k <= 0 || d <= 0) return 0;
    if (n <= kSmallN) return gemm_small(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, as_stream(stream), run_if);
    return gemm_launch(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, as_stream(stream), run_if);
}
