// K1 — CSR sparse matrix x tall-skinny block, Y = A X (sm_100a).
//
// Replaces the reference's symmetric lower-CSR SpMV applied one column at a
// time (proj/src/kernel.cpp:8-33), which re-reads the matrix once per column
// and scatters into y[c].  Here the matrix is expanded once to full CSR and
// X / Y are row-major, so each nonzero gathers a contiguous k-vector of X and
// every row of Y is written exactly once: no atomics, deterministic (fixed
// column-ascending order per row), one pass over the matrix per call.
//
// Mapping: one warp per matrix row (half a warp with 16-byte loads for k <= 32);
// rows are dealt in tiles of 64 to the resident CTAs so all SMs sweep the
// matrix together and the live band of X stays in L2.  The warp loads up to 32
// of the row's (col, val) pairs with one coalesced load each and broadcasts them
// by shuffle; lane l accumulates columns l, l+32, ..., so every X-row gather
// is a coalesced 256-byte transaction per 32 columns, four nonzeros' gathers in
// flight per step.  Accumulators stay in registers (VPL per lane); widths
// beyond 32*VPL loop over column chunks.  Complex: double2 per lane, the same
// sweep.  HBM-bound: algorithmic bytes = nnz*12 + (n+1)*4 + 2*n*k*8 (real;
// complex nnz*20 + (n+1)*4 + 2*n*k*16); for wide k and many nonzeros per row
// the X-row gathers (nnz*k*8) through L1/L2 are the practical bound.
#include <cstdlib>

#include "bk_common.cuh"

namespace bk {
namespace {

template <int VPL>
__global__ void __launch_bounds__(256) spmm_d_kernel(int n, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x, int ldx, int k,
                                                      double* __restrict__ y, int ldy, int tile) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // Rows are dealt out in tiles of `tile` consecutive rows, tile t to CTA
    // t mod grid (grid = resident CTAs), so all SMs sweep the matrix together:
    // the X rows live at any moment are a narrow band around the sweep front
    // (plus the stencil's far offsets) that stays in L2, and neighbouring rows
    // inside a tile re-hit L1.  (Contiguous per-CTA chunks spread the band over
    // the whole matrix and re-read X from HBM ~6x at k = 160.)
    for (int t0 = blockIdx.x * tile; t0 < n; t0 += gridDim.x * tile)
    for (int row = t0 + warp; row < min(n, t0 + tile); row += nw) {
        const int s = __ldg(rp + row), e = __ldg(rp + row + 1);
        for (int c0 = 0; c0 < k; c0 += 32 * VPL) {
            double acc[VPL];
#pragma unroll
            for (int u = 0; u < VPL; ++u) acc[u] = 0.0;
            for (int pb = s; pb < e; pb += 32) {
                const int p = pb + lane;
                int my_c = 0;
                double my_v = 0.0;
                if (p < e) {
                    my_c = __ldg(ci + p);
                    my_v = __ldg(val + p);
                }
                const int cnt = min(32, e - pb);
                // 4 nonzeros per step: all their X-row gathers are issued before
                // any is consumed (memory-level parallelism; the kernel is
                // latency-bound otherwise).  Accumulation order is unchanged.
                constexpr int G = 4;
                int t = 0;
                for (; t + G <= cnt; t += G) {
                    double xv[G][VPL], vv[G];
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const int c = __shfl_sync(0xffffffffu, my_c, t + q);
                        vv[q] = __shfl_sync(0xffffffffu, my_v, t + q);
                        const double* xr = x + static_cast<size_t>(c) * ldx + c0 + lane;
#pragma unroll
                        for (int u = 0; u < VPL; ++u) xv[q][u] = c0 + lane + 32 * u < k ? __ldg(xr + 32 * u) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q)
#pragma unroll
                        for (int u = 0; u < VPL; ++u) acc[u] = fma(vv[q], xv[q][u], acc[u]);
                }
                // tail (< G nonzeros): for narrow blocks all its gathers issued
                // together too (wide ones: one at a time, registers)
                if (VPL > 3) {
                    for (; t < cnt; ++t) {
                        const int c = __shfl_sync(0xffffffffu, my_c, t);
                        const double v = __shfl_sync(0xffffffffu, my_v, t);
                        const double* xr = x + static_cast<size_t>(c) * ldx + c0 + lane;
#pragma unroll
                        for (int u = 0; u < VPL; ++u)
                            if (c0 + lane + 32 * u < k) acc[u] = fma(v, __ldg(xr + 32 * u), acc[u]);
                    }
                } else if (t < cnt) {
                    double xv[G][VPL], vv[G];
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const bool live = t + q < cnt;
                        const int c = __shfl_sync(0xffffffffu, my_c, live ? t + q : t);
                        vv[q] = __shfl_sync(0xffffffffu, my_v, live ? t + q : t);
                        const double* xr = x + static_cast<size_t>(c) * ldx + c0 + lane;
#pragma unroll
                        for (int u = 0; u < VPL; ++u)
                            xv[q][u] = live && c0 + lane + 32 * u < k ? __ldg(xr + 32 * u) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q)
                        if (t + q < cnt)
#pragma unroll
                            for (int u = 0; u < VPL; ++u) acc[u] = fma(vv[q], xv[q][u], acc[u]);
                }
            }
            double* yr = y + static_cast<size_t>(row) * ldy + c0 + lane;
#pragma unroll
            for (int u = 0; u < VPL; ++u)
                if (c0 + lane + 32 * u < k) yr[32 * u] = acc[u];
        }
    }
}

// complex Hermitian: full CSR already holds conj() of the mirrored entries
template <int VPL>
__global__ void __launch_bounds__(256) spmm_z_kernel(int n, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci,
                                                      const double2* __restrict__ val,
                                                      const double2* __restrict__ x, int ldx, int k,
                                                      double2* __restrict__ y, int ldy, int tile) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // the real kernel's tiled sweep (tile rows per CTA step, resident CTAs)
    for (int t0 = blockIdx.x * tile; t0 < n; t0 += gridDim.x * tile)
    for (int row = t0 + warp; row < min(n, t0 + tile); row += nw) {
        const int s = __ldg(rp + row), e = __ldg(rp + row + 1);
        for (int c0 = 0; c0 < k; c0 += 32 * VPL) {
            double2 acc[VPL];
#pragma unroll
            for (int u = 0; u < VPL; ++u) acc[u] = make_double2(0.0, 0.0);
            for (int pb = s; pb < e; pb += 32) {
                const int p = pb + lane;
                int my_c = 0;
                double2 my_v = make_double2(0.0, 0.0);
                if (p < e) {
                    my_c = __ldg(ci + p);
                    my_v = __ldg(val + p);
                }
                const int cnt = min(32, e - pb);
                for (int t = 0; t < cnt; ++t) {
                    const int c = __shfl_sync(0xffffffffu, my_c, t);
                    const double vr = __shfl_sync(0xffffffffu, my_v.x, t);
                    const double vi = __shfl_sync(0xffffffffu, my_v.y, t);
                    const double2* xr = x + static_cast<size_t>(c) * ldx + c0 + lane;
#pragma unroll
                    for (int u = 0; u < VPL; ++u)
                        if (c0 + lane + 32 * u < k) {
                            const double2 xv = __ldg(xr + 32 * u);
                            acc[u].x = fma(vr, xv.x, fma(-vi, xv.y, acc[u].x));
                            acc[u].y = fma(vr, xv.y, fma(vi, xv.x, acc[u].y));
                        }
                }
            }
            double2* yr = y + static_cast<size_t>(row) * ldy + c0 + lane;
#pragma unroll
            for (int u = 0; u < VPL; ++u)
                if (c0 + lane + 32 * u < k) yr[32 * u] = acc[u];
        }
    }
}

// Half-warp per row, 16-byte X loads (k even, 16-byte aligned rows): two rows
// per warp in flight, so each lane keeps twice the bytes in flight at the same
// instruction count (the real kernel is gather-latency bound at k <= 96).
template <int V2>
__global__ void __launch_bounds__(256) spmm_d_half_kernel(int n, const int32_t* __restrict__ rp,
                                                           const int32_t* __restrict__ ci,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ x, int ldx, int k,
                                                           double* __restrict__ y, int ldy, int tile) {
    const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
    const int k2 = k >> 1;
    const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x);
    const int ldx2 = ldx >> 1, ldy2 = ldy >> 1;
    double2* __restrict__ y2 = reinterpret_cast<double2*>(y);
    for (int t0 = blockIdx.x * tile; t0 < n; t0 += gridDim.x * tile)
        for (int rb = t0 + 2 * warp; rb < min(n, t0 + tile); rb += 2 * nw) {
            const int row = rb + half;
            const bool live = row < min(n, t0 + tile);
            const int s = live ? __ldg(rp + row) : 0, e = live ? __ldg(rp + row + 1) : 0;
            double2 acc[V2];
#pragma unroll
            for (int u = 0; u < V2; ++u) acc[u] = make_double2(0.0, 0.0);
            for (int pb = s; pb < e; pb += 16) {
                const int p = pb + hl;
                int my_c = 0;
                double my_v = 0.0;
                if (p < e) {
                    my_c = __ldg(ci + p);
                    my_v = __ldg(val + p);
                }
                const int cnt = min(16, e - pb);
                int t = 0;
                for (; t + 4 <= cnt; t += 4) {
                    double2 xv[4][V2];
                    double vv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = __shfl_sync(hmask, my_c, t + q, 16);
                        vv[q] = __shfl_sync(hmask, my_v, t + q, 16);
                        const double2* xr = x2 + static_cast<size_t>(c) * ldx2 + hl;
#pragma unroll
                        for (int u = 0; u < V2; ++u)
                            xv[q][u] = hl + 16 * u < k2 ? __ldg(xr + 16 * u) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int u = 0; u < V2; ++u) {
                            acc[u].x = fma(vv[q], xv[q][u].x, acc[u].x);
                            acc[u].y = fma(vv[q], xv[q][u].y, acc[u].y);
                        }
                }
                if (t < cnt) {  // tail: its gathers issued together
                    double2 xv[4][V2];
                    double vv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool lv = t + q < cnt;
                        const int c = __shfl_sync(hmask, my_c, lv ? t + q : t, 16);
                        vv[q] = __shfl_sync(hmask, my_v, lv ? t + q : t, 16);
                        const double2* xr = x2 + static_cast<size_t>(c) * ldx2 + hl;
#pragma unroll
                        for (int u = 0; u < V2; ++u)
                            xv[q][u] = lv && hl + 16 * u < k2 ? __ldg(xr + 16 * u) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (t + q < cnt)
#pragma unroll
                            for (int u = 0; u < V2; ++u) {
                                acc[u].x = fma(vv[q], xv[q][u].x, acc[u].x);
                                acc[u].y = fma(vv[q], xv[q][u].y, acc[u].y);
                            }
                }
            }
            if (live) {
                double2* yr = y2 + static_cast<size_t>(row) * ldy2 + hl;
#pragma unroll
                for (int u = 0; u < V2; ++u)
                    if (hl + 16 * u < k2) yr[16 * u] = acc[u];
            }
        }
}

// tile rows per CTA step and resident CTAs per SM for spmm_d_kernel
// (BK_SPMM_TILE / BK_SPMM_CPS override, for tuning runs only)
struct SpmmShape {
    int tile, cps;
};
SpmmShape spmm_shape() {
    static const SpmmShape sh = [] {
        SpmmShape r{64, 4};
        if (const char* e = getenv("BK_SPMM_TILE")) r.tile = max(8, atoi(e));
        if (const char* e = getenv("BK_SPMM_CPS")) r.cps = max(1, atoi(e));
        return r;
    }();
    return sh;
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" int bk_spmm_d(int n, const int32_t* rp, const int32_t* ci, const double* val,
                         const double* x, int ldx, int k, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const SpmmShape sh = spmm_shape();
    // wide blocks (k > 96: 4-6 accumulators per lane, fewer resident warps) run
    // with twice the CTAs per SM in the sweep: config 4's k = 160 2.39 -> 1.90 ms
    // (BK_SPMM_CPS overrides; 8 nonzeros in flight per step measured slower at
    // k = 96 and no better at k = 160)
    const int cps = getenv("BK_SPMM_CPS") ? sh.cps : (k > 96 ? 8 : 4);
    const int tg = max(1, min(ceil_div(n, sh.tile), kSMs * cps));
    // narrow blocks (k <= 32): half a warp per row with 16-byte loads, two rows per
    // warp in flight (config 2, k = 26: 0.127 -> 0.082 ms); wider blocks measured
    // slower that way (BK_SPMM_HALF=1 forces it up to k = 96, tuning runs only)
    static const bool half_all = getenv("BK_SPMM_HALF") != nullptr;
    const bool vec16 = (k % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                       (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(y) % 16 == 0);
    if (vec16 && (k <= 32 || (half_all && k <= 96))) {
        if (k <= 32)
            spmm_d_half_kernel<1><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
        else if (k <= 64)
            spmm_d_half_kernel<2><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
        else
            spmm_d_half_kernel<3><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
        BK_LAUNCHED();
    }
    if (k <= 32)
        spmm_d_kernel<1><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    else if (k <= 64)
        spmm_d_kernel<2><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    else if (k <= 96)
        spmm_d_kernel<3><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    else if (k <= 128)
        spmm_d_kernel<4><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    else if (k <= 160)
        spmm_d_kernel<5><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    else
        spmm_d_kernel<6><<<tg, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy, sh.tile);
    BK_LAUNCHED();
}

extern "C" int bk_spmm_z(int n, const int32_t* rp, const int32_t* ci, const double* val,
                         const double* x, int ldx, int k, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const SpmmShape sh = spmm_shape();
    // wide complex blocks: 128 columns per lane chunk (4 x 16 B), 8 CTAs per SM in
    // the sweep — config 5's k = 384 SpMM 3.38 -> 2.96 ms (68 % of HBM)
    const int cps = getenv("BK_SPMM_CPS") ? sh.cps : (k > 96 ? 8 : 4);
    const int grid = max(1, min(ceil_div(n, sh.tile), kSMs * cps));
    auto v = reinterpret_cast<const double2*>(val);
    auto xx = reinterpret_cast<const double2*>(x);
    auto yy = reinterpret_cast<double2*>(y);
    static const int vz = [] {  // BK_SPMM_ZV: complex columns per lane for wide k (tuning runs)
        const char* e = getenv("BK_SPMM_ZV");
        return e ? atoi(e) : 4;
    }();
    if (k <= 32)
        spmm_z_kernel<1><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy, sh.tile);
    else if (k <= 64)
        spmm_z_kernel<2><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy, sh.tile);
    else if (k <= 96 || vz == 3)
        spmm_z_kernel<3><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy, sh.tile);
    else if (vz == 4)
        spmm_z_kernel<4><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy, sh.tile);
    else
        spmm_z_kernel<6><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy, sh.tile);
    BK_LAUNCHED();
}
