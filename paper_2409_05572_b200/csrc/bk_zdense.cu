// K2 / K3 for complex128 blocks with the 3M (Gauss) product on the FP64 tensor
// cores — config 5's Gram and update are >90 % of its solve.
//
// The real-view form (bk_complex.cu: a complex n x k block is a real n x 2k
// block, every contraction a real DMMA GEMM of twice the width in both
// dimensions) spends 4 real products per complex product.  Here the operands
// are staged as interleaved (re, im) tiles exactly as before, but each lane
// splits its fragment into re / im in registers and the warp runs THREE real
// DMMA products per complex fragment pair:
//
//   Gram   C = X^H Y :  T1 = Xr^T Yr,  T2 = Xi^T Yi,  T3 = (Xr - Xi)^T (Yr + Yi)
//                       Re C = T1 + T2,   Im C = T3 - T1 + T2
//   update Y = a X C + b Y :  T1 = Xr Cr,  T2 = Xi Ci,  T3 = (Xr + Xi)(Cr + Ci)
//                       Re = T1 - T2,     Im = T3 - T1 - T2
//
// 25 % fewer DMMA instructions for the same complex flop count (the roofline
// numerator stays the complex count, 8 n a b).  The rounding differs from the
// 4-product form only in the imaginary parts, whose error bound becomes
// eps (|Xr| + |Xi|)^T (|Yr| + |Yi|) instead of eps (|Xr|^T |Yi| + |Xi|^T |Yr|)
// — the same norm-wise fp64 bound (tests/test_gpu_complex.py checks against
// numpy at 1e-12 relative to |X|^T |Y|).
//
// Fragment loads are 16-byte (one lane reads one complex element); shared
// pitches are chosen so the quarter-warp phases of those loads hit distinct
// banks (Gram / C tiles: pitch = 4 mod 16 doubles; update X tiles: 8 mod 16).
// Split-K partial tiles of the Grams are reduced in a fixed order as in
// bk_dense.cu (deterministic).  References: rr.cpp:11,13 (S^T AS, S Z),
// kernel.cpp:76,79 (q^T v, q c), solvers.cpp:195 (hl_trick lifts).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "bk_dense.cuh"

namespace bk {
namespace {

// ------------------------------------------------------------------ Gram
// TM x TN complex output tile per CTA, WM x WN warps, TK rows of the
// contraction per stage
template <int TM, int TN, int TK, int WM, int WN, int STAGES, bool SYM>
__global__ void __launch_bounds__(WM * WN * 32) zgram3m_kernel(int n, const double* __restrict__ x, int ldx, int a,
                                                               const double* __restrict__ y, int ldy, int b,
                                                               double* __restrict__ out, int ldo, int rows_per_split,
                                                               const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    constexpr int NT = WM * WN * 32;
    constexpr int PX = 2 * TM + 4, PY = 2 * TN + 4;  // doubles
    constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
    static_assert(FM * WM * 8 == TM && FN * WN * 8 == TN, "warp tiling");
    extern __shared__ __align__(16) double smem[];
    double* xs = smem;
    double* ys = smem + STAGES * TK * PX;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    int ti = blockIdx.x, tj = blockIdx.y;
    if constexpr (SYM) {
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
    const bool same = SYM && ti == tj && x == y && ldx == ldy;

    double acc[3][FM][FN][2];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) acc[p][mi][ni][0] = acc[p][mi][ni][1] = 0.0;

    const int nk = ceil_div(max(r_end - r_begin, 0), TK);
    auto load_stage = [&](int kt, int st) {
        const int r0 = r_begin + kt * TK;
        load_tile16<TK, TM, NT>(xs + st * TK * PX, PX, x, 2 * ldx, r0, r_end, 2 * i0, 2 * a, tid);
        if (!same) load_tile16<TK, TN, NT>(ys + st * TK * PY, PY, y, 2 * ldy, r0, r_end, 2 * j0, 2 * b, tid);
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
        const double* xd = xs + (kt % STAGES) * TK * PX;
        const double* yd = same ? xd : ys + (kt % STAGES) * TK * PY;
        const int py = same ? PX : PY;
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double2 xf[FM], yf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
                xf[mi] = *reinterpret_cast<const double2*>(xd + (k4 + t) * PX + 2 * (wm + mi * 8 + g));
#pragma unroll
            for (int ni = 0; ni < FN; ++ni)
                yf[ni] = *reinterpret_cast<const double2*>(yd + (k4 + t) * py + 2 * (wn + ni * 8 + g));
            // T1 and T2 products first, the operand sums of T3 meanwhile: the
            // DADDs' latency is off the DMMA issue path
            double ysum[FN], xdiff[FM];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) ysum[ni] = yf[ni].x + yf[ni].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) xdiff[mi] = xf[mi].x - xf[mi].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) {
                    dmma_8x8x4(acc[0][mi][ni][0], acc[0][mi][ni][1], xf[mi].x, yf[ni].x);
                    dmma_8x8x4(acc[1][mi][ni][0], acc[1][mi][ni][1], xf[mi].y, yf[ni].y);
                }
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni)
                    dmma_8x8x4(acc[2][mi][ni][0], acc[2][mi][ni][1], xdiff[mi], ysum[ni]);
        }
    }
    cp_async_wait<0>();

    double* o = out + static_cast<size_t>(split) * a * ldo * 2;
#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const int i = i0 + wm + mi * 8 + g;
            const int j = j0 + wn + ni * 8 + 2 * t;
            if (i >= a) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (j + h >= b) continue;
                const double t1 = acc[0][mi][ni][h], t2 = acc[1][mi][ni][h], t3 = acc[2][mi][ni][h];
                *reinterpret_cast<double2*>(o + 2 * (static_cast<size_t>(i) * ldo + j + h)) =
                    make_double2(t1 + t2, (t3 - t1) + t2);
            }
        }
}

// C[i][j] = sum_s work[s][i][j] (complex) in a fixed order; with `sym`, entries
// of the strictly-lower tiles (never computed) are the conjugates of the upper
__global__ void __launch_bounds__(256) zgram_reduce(int splits, int a, int b, const double2* __restrict__ work,
                                                     double2* __restrict__ c, int ldc, int sym, int tile,
                                                     const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    __shared__ double2 red[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t total = static_cast<int64_t>(a) * b;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * 32 + tx;
    int i = 0, j = 0;
    int64_t src = 0;
    bool mirror = false;
    if (e < total) {
        i = static_cast<int>(e / b);
        j = static_cast<int>(e % b);
        mirror = sym && i / tile > j / tile;
        src = mirror ? static_cast<int64_t>(j) * b + i : e;
    }
    const int p0 = static_cast<int>(static_cast<int64_t>(splits) * ty / 8);
    const int p1 = static_cast<int>(static_cast<int64_t>(splits) * (ty + 1) / 8);
    double sr = 0.0, si = 0.0;
    if (e < total)
        for (int p = p0; p < p1; ++p) {
            const double2 v = work[static_cast<size_t>(p) * total + src];
            sr += v.x;
            si += v.y;
        }
    red[ty][tx] = make_double2(sr, si);
    __syncthreads();
    if (ty == 0 && e < total) {
        double2 s = red[0][tx];
#pragma unroll
        for (int q = 1; q < 8; ++q) {
            s.x += red[q][tx].x;
            s.y += red[q][tx].y;
        }
        if (mirror) s.y = -s.y;
        c[static_cast<size_t>(i) * ldc + j] = s;
    }
}

template <int TM, int TN, int TK, int WM, int WN, int ST, int CPS, bool SYM>
int zgram_launch_v(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                   void* work, cudaStream_t s, const int* run_if) {
    static_assert(!SYM || TM == TN, "symmetric tiles are square");
    constexpr size_t smem = sizeof(double) * ST * TK * ((2 * TM + 4) + (2 * TN + 4));
    auto kern = zgram3m_kernel<TM, TN, TK, WM, WN, ST, SYM>;
    BK_RET(BK_ONCE_PER_DEVICE(prep(kern, smem)));
    const int nt = ceil_div(a, TM);
    const int tiles = SYM ? nt * (nt + 1) / 2 : nt * ceil_div(b, TN);
    // partials are 2ab doubles per split; plan as for the 2a x 2b real view so
    // the workspace sized by bk_gram_z_work_bytes always suffices
    const GramPlan p = gram_plan(n, tiles, 2 * a, 2 * b, CPS, TK);
    const dim3 grid(SYM ? tiles : nt, SYM ? 1 : ceil_div(b, TN), p.splits);
    auto w = static_cast<double*>(work);
    const bool direct = p.splits == 1 && !SYM;
    kern<<<grid, WM * WN * 32, smem, s>>>(n, x, ldx, a, y, ldy, b, direct ? c : w, direct ? ldc : b,
                                          p.rows_per_split, run_if);
    if (!direct) {
        const int64_t total = static_cast<int64_t>(a) * b;
        zgram_reduce<<<static_cast<int>(ceil_div64(total, 32)), 256, 0, s>>>(
            p.splits, a, b, reinterpret_cast<const double2*>(w), reinterpret_cast<double2*>(c), ldc, SYM ? 1 : 0, TM,
            run_if);
    }
    BK_LAUNCHED();
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <bool SYM>
int zgram_launch(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                 void* work, cudaStream_t s, const int* run_if) {
    // BK_ZGRAM: tile shape (tuning runs, tools/zdense_probe.py)
    static const int v = env_int("BK_ZGRAM", 0);
    switch (v) {
        case 1:  // 64 x 64 complex, 8 warps of 32 x 16, 8-deep, 4 stages
            return zgram_launch_v<64, 64, 8, 2, 4, 4, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        case 2:  // 64 x 64 complex, 8 warps of 16 x 32
            return zgram_launch_v<64, 64, 8, 4, 2, 4, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        case 3:  // 48 x 48, 16-deep, 4 stages, 2 CTAs / SM
            return zgram_launch_v<48, 48, 16, 2, 2, 4, 2, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
        default:  // 48 x 48 complex (the 96 x 96 real-view footprint), 4 warps of 24 x 24 (156 registers),
                  // 8-deep, 4 stages, 3 CTAs / SM; config 5 shapes (tools/zdense_probe.py): symmetric
                  // d = 1152 36.7 -> 37.1, 768 x 384 38.2 -> 39.0, 384^2 37.2 -> 38.4 complex TF/s
                  // against 16-deep at 2 CTAs / SM
            return zgram_launch_v<48, 48, 8, 2, 2, 4, 3, SYM>(n, x, ldx, a, y, ldy, b, c, ldc, work, s, run_if);
    }
}

// ------------------------------------------------------------------ update
// TM rows x TN complex columns per CTA, TK complex contraction columns per stage;
// 1-D grid with the column tiles of one row panel adjacent, so the CTAs that
// read the same X rows run together and share them through L2
template <int TM, int TN, int TK, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB) zgemm3m_kernel(int n, const double* __restrict__ x, int ldx, int d,
                                                               const double* __restrict__ cm, int ldc, int k,
                                                               double alpha, double beta, double* __restrict__ y,
                                                               int ldy, int nct, const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    constexpr int NT = WM * WN * 32;
    constexpr int PX = 2 * TK + 8, PC = 2 * TN + 4;  // doubles
    constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
    static_assert(FM * WM * 8 == TM && FN * WN * 8 == TN, "warp tiling");
    extern __shared__ __align__(16) double smem[];
    double* xs = smem;                     // STAGES x TM x PX
    double* cs = smem + STAGES * TM * PX;  // STAGES x TK x PC
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int ct = blockIdx.x % nct, rt = blockIdx.x / nct;
    const int r0 = rt * TM, c0 = ct * TN;
    const int wm = (warp / WN) * (TM / WM), wn = (warp % WN) * (TN / WN);

    double acc[3][FM][FN][2];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) acc[p][mi][ni][0] = acc[p][mi][ni][1] = 0.0;

    const int nk = ceil_div(d, TK);
    auto load_stage = [&](int kt, int st) {
        const int k0 = kt * TK;
        load_tile16<TM, TK, NT>(xs + st * TM * PX, PX, x, 2 * ldx, r0, n, 2 * k0, 2 * d, tid);
        load_tile16<TK, TN, NT>(cs + st * TK * PC, PC, cm, 2 * ldc, k0, d, 2 * c0, 2 * k, tid);
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
            double2 xf[FM], cf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
                xf[mi] = *reinterpret_cast<const double2*>(xd + (wm + mi * 8 + g) * PX + 2 * (k4 + t));
#pragma unroll
            for (int ni = 0; ni < FN; ++ni)
                cf[ni] = *reinterpret_cast<const double2*>(cd + (k4 + t) * PC + 2 * (wn + ni * 8 + g));
            double csum[FN], xsum[FM];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) csum[ni] = cf[ni].x + cf[ni].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) xsum[mi] = xf[mi].x + xf[mi].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) {
                    dmma_8x8x4(acc[0][mi][ni][0], acc[0][mi][ni][1], xf[mi].x, cf[ni].x);
                    dmma_8x8x4(acc[1][mi][ni][0], acc[1][mi][ni][1], xf[mi].y, cf[ni].y);
                }
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni)
                    dmma_8x8x4(acc[2][mi][ni][0], acc[2][mi][ni][1], xsum[mi], csum[ni]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const int i = r0 + wm + mi * 8 + g;
            const int j = c0 + wn + ni * 8 + 2 * t;
            if (i >= n) continue;
            double2* yr = reinterpret_cast<double2*>(y + 2 * static_cast<size_t>(i) * ldy);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (j + h >= k) continue;
                const double t1 = acc[0][mi][ni][h], t2 = acc[1][mi][ni][h], t3 = acc[2][mi][ni][h];
                const double re = t1 - t2, im = (t3 - t1) - t2;
                double2 v;
                if (beta == 0.0) {
                    v = make_double2(alpha * re, alpha * im);
                } else {
                    const double2 old = yr[j + h];
                    v = make_double2(fma(alpha, re, beta * old.x), fma(alpha, im, beta * old.y));
                }
                yr[j + h] = v;
            }
        }
}

template <int TM, int TN, int TK, int WM, int WN, int ST, int MINB = 1>
int zgemm_launch_v(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
                   double* y, int ldy, cudaStream_t s, const int* run_if) {
    constexpr size_t smem = sizeof(double) * ST * (TM * (2 * TK + 8) + TK * (2 * TN + 4));
    auto kern = zgemm3m_kernel<TM, TN, TK, WM, WN, ST, MINB>;
    BK_RET(BK_ONCE_PER_DEVICE(prep(kern, smem)));
    const int nct = ceil_div(k, TN);
    const int64_t blocks = static_cast<int64_t>(ceil_div(n, TM)) * nct;
    kern<<<static_cast<unsigned>(blocks), WM * WN * 32, smem, s>>>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, nct,
                                                                  run_if);
    BK_LAUNCHED();
}


// ------------------------------------------------------------------ update, TMA-fed
// The same 3M update with the X operand (TM rows x 8 complex = 128-byte rows per
// stage) moved by the Tensor Memory Accelerator: one cp.async.bulk.tensor box per
// stage issued by one thread, completion on an mbarrier, 128-byte swizzle (16-byte
// chunk c of row r lands at chunk c ^ (r & 7)).  The swizzle alone would leave the
// fragment loads 2-way bank-conflicted (the two rows of a quarter-warp phase XOR
// their chunks with 0 and 1), so fragment row g of the DMMA reads tile row
// sigma(g) = 4 (g & 1) + g / 2: the rows of a phase then differ in bit 2 and their
// chunks cover all 8 of a 128-byte line.  The output rows follow the same map.
// C (8 k-rows x TN complex) stays on cp.async with its padded pitch.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <int TM, int TN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(WM * WN * 32) zgemm3m_tma_kernel(const __grid_constant__ CUtensorMap tmx, int n,
                                                                   int d, const double* __restrict__ cm, int ldc,
                                                                   int k, double alpha, double beta,
                                                                   double* __restrict__ y, int ldy, int nct,
                                                                   const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    constexpr int TK = 8;                 // complex columns per stage: one 128-byte row
    constexpr int NT = WM * WN * 32;
    constexpr int PC = 2 * TN + 4;        // doubles
    constexpr int XB = TM * 128;          // bytes of one X stage
    constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
    static_assert(FM * WM * 8 == TM && FN * WN * 8 == TN, "warp tiling");
    extern __shared__ __align__(1024) unsigned char zsm[];
    unsigned char* xs = zsm;                                          // STAGES x XB (1024-aligned)
    double* cs = reinterpret_cast<double*>(zsm + STAGES * XB);        // STAGES x TK x PC
    uint64_t* bar = reinterpret_cast<uint64_t*>(cs + STAGES * TK * PC);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int sg = ((g & 1) << 2) | (g >> 1);  // fragment row g -> tile row
    const int ct = blockIdx.x % nct, rt = blockIdx.x / nct;
    const int r0 = rt * TM, c0 = ct * TN;
    const int wm = (warp / WN) * (TM / WM), wn = (warp % WN) * (TN / WN);
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) mbar_init(bar + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    double acc[3][FM][FN][2];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) acc[p][mi][ni][0] = acc[p][mi][ni][1] = 0.0;

    const int nk = ceil_div(d, TK);
    auto load_stage = [&](int kt, int st) {
        if (tid == 0) {
            mbar_expect_tx(bar + st, XB);
            tma_load_2d(xs + st * XB, &tmx, 2 * kt * TK, r0, bar + st);
        }
        load_tile16<TK, TN, NT>(cs + st * TK * PC, PC, cm, 2 * ldc, kt * TK, d, 2 * c0, 2 * k, tid);
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, st);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();  // C stage kt visible; every warp is past stage kt - 1
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load_stage(nxt, nxt % STAGES);
        cp_async_commit();
        const int st = kt % STAGES;
        mbar_wait(bar + st, (kt / STAGES) & 1);
        const unsigned char* xd = xs + st * XB;
        const double* cd = cs + st * TK * PC;
#pragma unroll
        for (int k4 = 0; k4 < TK; k4 += 4) {
            double2 xf[FM], cf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) {
                const int r = wm + mi * 8 + sg;
                xf[mi] = *reinterpret_cast<const double2*>(xd + r * 128 + (((k4 + t) ^ (r & 7)) << 4));
            }
#pragma unroll
            for (int ni = 0; ni < FN; ++ni)
                cf[ni] = *reinterpret_cast<const double2*>(cd + (k4 + t) * PC + 2 * (wn + ni * 8 + g));
            double csum[FN], xsum[FM];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) csum[ni] = cf[ni].x + cf[ni].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) xsum[mi] = xf[mi].x + xf[mi].y;
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) {
                    dmma_8x8x4(acc[0][mi][ni][0], acc[0][mi][ni][1], xf[mi].x, cf[ni].x);
                    dmma_8x8x4(acc[1][mi][ni][0], acc[1][mi][ni][1], xf[mi].y, cf[ni].y);
                }
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni)
                    dmma_8x8x4(acc[2][mi][ni][0], acc[2][mi][ni][1], xsum[mi], csum[ni]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const int i = r0 + wm + mi * 8 + sg;
            const int j = c0 + wn + ni * 8 + 2 * t;
            if (i >= n) continue;
            double2* yr = reinterpret_cast<double2*>(y + 2 * static_cast<size_t>(i) * ldy);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (j + h >= k) continue;
                const double t1 = acc[0][mi][ni][h], t2 = acc[1][mi][ni][h], t3 = acc[2][mi][ni][h];
                const double re = t1 - t2, im = (t3 - t1) - t2;
                double2 v;
                if (beta == 0.0) {
                    v = make_double2(alpha * re, alpha * im);
                } else {
                    const double2 old = yr[j + h];
                    v = make_double2(fma(alpha, re, beta * old.x), fma(alpha, im, beta * old.y));
                }
                yr[j + h] = v;
            }
        }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <int TM, int TN, int WM, int WN, int ST>
int zgemm_tma_launch_v(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                       double beta, double* y, int ldy, cudaStream_t s, const int* run_if) {
    auto enc = encode_fn();
    if (!enc) return static_cast<int>(cudaErrorNotSupported);
    // X as a 2-D tensor of doubles: 2d columns in use, n rows, row pitch 16 ldx bytes
    CUtensorMap map;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2) * d, static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 16};
    const cuuint32_t box[2] = {16, TM};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return static_cast<int>(cudaErrorInvalidValue);
    constexpr size_t smem = ST * TM * 128 + sizeof(double) * ST * 8 * (2 * TN + 4) + ST * 8 + 1024;
    auto kern = zgemm3m_tma_kernel<TM, TN, WM, WN, ST>;
    BK_RET(BK_ONCE_PER_DEVICE(prep(kern, smem)));
    const int nct = ceil_div(k, TN);
    const int64_t blocks = static_cast<int64_t>(ceil_div(n, TM)) * nct;
    kern<<<static_cast<unsigned>(blocks), WM * WN * 32, smem, s>>>(map, n, d, c, ldc, k, alpha, beta, y, ldy, nct,
                                                                  run_if);
    BK_LAUNCHED();
}

int zgemm_launch(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
                 double* y, int ldy, cudaStream_t s, const int* run_if) {
    static const int v = env_int("BK_ZGEMM", 0);
    switch (v) {
        case 1:  // 128 rows x 48, 8 warps of 32 x 24, 8-deep, 4 stages
            return zgemm_launch_v<128, 48, 8, 4, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 2:  // 64 x 48, 4 warps of 32 x 24, 16-deep, 3 stages
            return zgemm_launch_v<64, 48, 16, 2, 2, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 3:  // 64 x 32, 4 warps of 32 x 16, 8-deep, 4 stages
            return zgemm_launch_v<64, 32, 8, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 4:  // 64 x 48 at 3 CTAs / SM (register-capped)
            return zgemm_launch_v<64, 48, 8, 2, 2, 4, 3>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 5:  // 32 x 48, 2 warps of 16 x 24... as 2 x 1 warps of 16 x 48
            return zgemm_launch_v<32, 48, 8, 2, 1, 4, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 6:  // TMA-fed X (64 x 48, 4 warps of 32 x 24, 4 stages)
            return zgemm_tma_launch_v<64, 48, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 7:  // TMA-fed X, 6 stages
            return zgemm_tma_launch_v<64, 48, 2, 2, 6>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        case 8:  // cp.async only
            return zgemm_launch_v<64, 48, 8, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
        default:  // 64 x 48, 4 warps of 32 x 24, 8-deep, 4 stages; X by TMA when beta = 0 (the lifts and
                  // the CholQR update: 1152 -> 768 42.5 -> 42.6 TF/s), cp.async when the update also
                  // reads Y (768 -> 384, beta = 1: 41.4 with cp.async against 40.6 with TMA)
            if (beta == 0.0)
                return zgemm_tma_launch_v<64, 48, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
            return zgemm_launch_v<64, 48, 8, 2, 2, 4>(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, s, run_if);
    }
}

}  // namespace
}  // namespace bk

using namespace bk;

// 3M forms behind the bk_*_z entry points (bk_complex.cu) for long contractions;
// BK_Z3M=0 selects the 4-product real-view form (A/B runs)
extern "C" int bk_z3m_enabled() {
    static const int on = env_int("BK_Z3M", 1);
    return on;
}

extern "C" int bk_gram_z3m(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                           void* work, const int* run_if, void* stream) {
    if (a <= 0 || b <= 0 || n <= 0) return 0;
    return zgram_launch<false>(n, x, ldx, a, y, ldy, b, c, ldc, work, as_stream(stream), run_if);
}

extern "C" int bk_gram_sym_z3m(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c, int ldc,
                               void* work, void* stream) {
    if (d <= 0 || n <= 0) return 0;
    return zgram_launch<true>(n, x, ldx, d, y, ldy, d, c, ldc, work, as_stream(stream), nullptr);
}

extern "C" int bk_gemm_z3m(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                           double beta, double* y, int ldy, const int* run_if, void* stream) {
    if (n <= 0 || k <= 0 || d <= 0) return 0;
    return zgemm_launch(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, as_stream(stream), run_if);
}
