// K1 — CSR sparse matrix x tall-skinny block, Y = A X (sm_100a).
//
// Replaces the reference's symmetric lower-CSR SpMV applied one column at a
// time (proj/src/kernel.cpp:8-33), which re-reads the matrix once per column
// and scatters into y[c].  Here the matrix is expanded once to full CSR and
// X / Y are row-major, so each nonzero gathers a contiguous k-vector of X and
// every row of Y is written exactly once: no atomics, deterministic (fixed
// column-ascending order per row), one pass over the matrix per call.
//
// Mapping: one warp per matrix row (grid-stride).  The warp loads up to 32 of
// the row's (col, val) pairs with one coalesced load each and broadcasts them
// by shuffle; lane l accumulates columns l, l+32, ..., so every X-row gather
// is a coalesced 256-byte transaction per 32 columns.  Accumulators stay in
// registers (VPL per lane); widths beyond 32*VPL loop over column chunks.
// HBM-bound: algorithmic bytes = nnz*12 + (n+1)*4 + 2*n*k*8 (real).
#include "bk_common.cuh"

namespace bk {
namespace {

template <int VPL>
__global__ void __launch_bounds__(256) spmm_d_kernel(int n, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x, int ldx, int k,
                                                      double* __restrict__ y, int ldy) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
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
                for (int t = 0; t < cnt; ++t) {
                    const int c = __shfl_sync(0xffffffffu, my_c, t);
                    const double v = __shfl_sync(0xffffffffu, my_v, t);
                    const double* xr = x + static_cast<size_t>(c) * ldx + c0 + lane;
#pragma unroll
                    for (int u = 0; u < VPL; ++u)
                        if (c0 + lane + 32 * u < k) acc[u] = fma(v, __ldg(xr + 32 * u), acc[u]);
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
                                                      double2* __restrict__ y, int ldy) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
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

int spmm_grid(int n) {
    // 8 warps per CTA, one row per warp per grid-stride step; enough CTAs to
    // fill every SM several times over (148 SMs x 8 resident CTAs)
    const int want = ceil_div(n, 8);
    return max(1, min(want, kSMs * 16));
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" int bk_spmm_d(int n, const int32_t* rp, const int32_t* ci, const double* val,
                         const double* x, int ldx, int k, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const int grid = spmm_grid(n);
    if (k <= 32)
        spmm_d_kernel<1><<<grid, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy);
    else if (k <= 64)
        spmm_d_kernel<2><<<grid, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy);
    else if (k <= 96)
        spmm_d_kernel<3><<<grid, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy);
    else
        spmm_d_kernel<4><<<grid, 256, 0, s>>>(n, rp, ci, val, x, ldx, k, y, ldy);
    BK_LAUNCHED();
}

extern "C" int bk_spmm_z(int n, const int32_t* rp, const int32_t* ci, const double* val,
                         const double* x, int ldx, int k, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    const int grid = spmm_grid(n);
    auto v = reinterpret_cast<const double2*>(val);
    auto xx = reinterpret_cast<const double2*>(x);
    auto yy = reinterpret_cast<double2*>(y);
    if (k <= 32)
        spmm_z_kernel<1><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy);
    else if (k <= 64)
        spmm_z_kernel<2><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy);
    else
        spmm_z_kernel<3><<<grid, 256, 0, s>>>(n, rp, ci, v, xx, ldx, k, yy, ldy);
    BK_LAUNCHED();
}
