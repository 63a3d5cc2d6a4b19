// Sparse Cholesky for shift-and-invert subspace iteration on n > 2000
// (reference SpdFactor sparse path: Eigen SimplicialLLT with AMD ordering,
// proj/src/kernel.cpp:110-134, used at solvers.cpp:207,234).
//
// The symbolic analysis (AMD ordering, elimination tree, the pattern of L and
// the etree level sets) runs once on the host (host/spchol.cpp); the numeric
// factorisation and every solve run here:
//
//  * factor: left-looking column Cholesky, one warp per column, the columns of
//    one etree level at a time (a column depends only on its etree
//    descendants, all on lower levels).  Column j receives, for each k in the
//    row pattern of L(j, :) in ascending order, the update -L(j,k) L(j:n, k):
//    the lanes walk column k's suffix below row j and find each row's slot in
//    column j by binary search (column j's pattern contains it, a property of
//    the Cholesky fill).  Fixed k order per column: deterministic.
//  * solve: Y = P^T L^-T L^-1 P X for a row-major block of m right-hand sides,
//    one persistent cooperative kernel — the forward substitution by ascending
//    levels (row j of L gathers the rows of its row pattern, one warp per row,
//    lanes across the m columns), the backward substitution by descending
//    levels (column j of L gathers its ancestors' rows), one grid barrier per
//    level.
#include <cooperative_groups.h>

#include <algorithm>

#include "bk_common.cuh"

namespace bk {
namespace {

__global__ void spchol_scatter_kernel(int64_t nnz_c, const int64_t* __restrict__ aidx, const double* __restrict__ aval,
                                      double* __restrict__ val) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz_c;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        val[aidx[e]] = aval[e];
}

__global__ void __launch_bounds__(256) spchol_level_kernel(int ncols, const int* __restrict__ cols,
                                                            const int64_t* __restrict__ colptr,
                                                            const int* __restrict__ rowind, double* __restrict__ val,
                                                            const int64_t* __restrict__ rptr,
                                                            const int* __restrict__ rk,
                                                            const int64_t* __restrict__ rpos, int* __restrict__ fail) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= ncols) return;
    const int j = cols[w];
    const int64_t c0 = colptr[j], c1 = colptr[j + 1];
    for (int64_t e = rptr[j]; e < rptr[j + 1]; ++e) {
        const int k = rk[e];
        const int64_t pos = rpos[e];  // L(j, k)
        const double f = val[pos];
        const int64_t kend = colptr[k + 1];
        for (int64_t idx = pos + lane; idx < kend; idx += 32) {
            const int i = rowind[idx];
            // slot of row i in column j (rows ascending, diagonal first)
            int64_t lo = c0, hi = c1 - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (rowind[mid] < i) lo = mid + 1;
                else hi = mid;
            }
            val[lo] -= f * val[idx];
        }
        __syncwarp();
    }
    const double d = val[c0];
    if (!(d > 0.0) || !isfinite(d)) {
        if (lane == 0) atomicExch(fail, 1);
        return;
    }
    const double s = sqrt(d);
    for (int64_t idx = c0 + 1 + lane; idx < c1; idx += 32) val[idx] /= s;
    if (lane == 0) val[c0] = s;
}

__global__ void __launch_bounds__(256) spchol_solve_kernel(int n, int m, const double* __restrict__ x, int ldx,
                                                            double* __restrict__ y, int ldy, double* __restrict__ t,
                                                            int ldt, const int* __restrict__ perm, int nlev,
                                                            const int* __restrict__ lvlptr,
                                                            const int* __restrict__ order,
                                                            const int64_t* __restrict__ colptr,
                                                            const int* __restrict__ rowind,
                                                            const double* __restrict__ val,
                                                            const int64_t* __restrict__ rptr,
                                                            const int* __restrict__ rk,
                                                            const int64_t* __restrict__ rpos) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    // T = P X
    for (int i = gw; i < n; i += nw) {
        const double* xr = x + static_cast<size_t>(perm[i]) * ldx;
        double* tr = t + static_cast<size_t>(i) * ldt;
        for (int c = lane; c < m; c += 32) tr[c] = xr[c];
    }
    grid.sync();
    // L z = T, ascending levels
    for (int l = 0; l < nlev; ++l) {
        for (int q = lvlptr[l] + gw; q < lvlptr[l + 1]; q += nw) {
            const int j = order[q];
            const double djj = val[colptr[j]];
            double* tj = t + static_cast<size_t>(j) * ldt;
            for (int c = lane; c < m; c += 32) {
                double s = tj[c];
                for (int64_t e = rptr[j]; e < rptr[j + 1]; ++e) s -= val[rpos[e]] * t[static_cast<size_t>(rk[e]) * ldt + c];
                tj[c] = s / djj;
            }
        }
        grid.sync();
    }
    // L^T w = z, descending levels
    for (int l = nlev - 1; l >= 0; --l) {
        for (int q = lvlptr[l] + gw; q < lvlptr[l + 1]; q += nw) {
            const int j = order[q];
            const int64_t c0 = colptr[j], c1 = colptr[j + 1];
            const double djj = val[c0];
            double* tj = t + static_cast<size_t>(j) * ldt;
            for (int c = lane; c < m; c += 32) {
                double s = tj[c];
                for (int64_t e = c0 + 1; e < c1; ++e) s -= val[e] * t[static_cast<size_t>(rowind[e]) * ldt + c];
                tj[c] = s / djj;
            }
        }
        grid.sync();
    }
    // Y = P^T W
    for (int i = gw; i < n; i += nw) {
        double* yr = y + static_cast<size_t>(perm[i]) * ldy;
        const double* tr = t + static_cast<size_t>(i) * ldt;
        for (int c = lane; c < m; c += 32) yr[c] = tr[c];
    }
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" int bk_spchol_factor_d(int n, int nlev, const int* lvlptr_host, const int* order, const int64_t* colptr,
                                  const int* rowind, double* val, int64_t nnz_l, const int64_t* rptr, const int* rk,
                                  const int64_t* rpos, int64_t nnz_c, const int64_t* aidx, const double* aval,
                                  int* fail, void* stream) {
    if (n <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    BK_RET(cudaMemsetAsync(val, 0, static_cast<size_t>(nnz_l) * sizeof(double), s));
    BK_RET(cudaMemsetAsync(fail, 0, sizeof(int), s));
    const int sg = static_cast<int>(std::min<int64_t>(ceil_div64(std::max<int64_t>(nnz_c, 1), 256), 8 * kSMs));
    spchol_scatter_kernel<<<sg, 256, 0, s>>>(nnz_c, aidx, aval, val);
    BK_RET(cudaGetLastError());
    for (int l = 0; l < nlev; ++l) {
        const int nc = lvlptr_host[l + 1] - lvlptr_host[l];
        spchol_level_kernel<<<ceil_div(nc * 32, 256), 256, 0, s>>>(nc, order + lvlptr_host[l], colptr, rowind, val,
                                                                    rptr, rk, rpos, fail);
        BK_RET(cudaGetLastError());
    }
    return 0;
}

extern "C" int bk_spchol_solve_d(int n, int m, const double* x, int ldx, double* y, int ldy, double* t, int ldt,
                                 const int* perm, int nlev, const int* lvlptr, const int* order,
                                 const int64_t* colptr, const int* rowind, const double* val, const int64_t* rptr,
                                 const int* rk, const int64_t* rpos, void* stream) {
    if (n <= 0 || m <= 0) return 0;
    int per_sm = 0;
    BK_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spchol_solve_kernel, 256, 0));
    const int grid = std::max(1, std::min(per_sm, 2)) * kSMs;
    void* args[] = {&n, &m, const_cast<double**>(&x), &ldx, &y, &ldy, &t, &ldt, const_cast<int**>(&perm), &nlev,
                    const_cast<int**>(&lvlptr), const_cast<int**>(&order), const_cast<int64_t**>(&colptr),
                    const_cast<int**>(&rowind), const_cast<double**>(&val), const_cast<int64_t**>(&rptr),
                    const_cast<int**>(&rk), const_cast<int64_t**>(&rpos)};
    BK_RET(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(spchol_solve_kernel), dim3(grid), dim3(256), args,
                                       0, as_stream(stream)));
    return 0;
}
