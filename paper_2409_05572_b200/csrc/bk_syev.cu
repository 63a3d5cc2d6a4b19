// K5 — symmetric eigensolver for the projected (Rayleigh-Ritz) problem, on device.
//
// Replaces sym_eig_small (proj/src/kernel.cpp:95-100: Eigen's
// SelfAdjointEigenSolver = Householder tridiagonalisation + implicit QR) with the
// same first stage and a parallel second stage:
//   1. tridiag_*        Householder reduction of 0.5(H + H^T) to tridiagonal
//                       T = Q^T H Q: a thread-block cluster holding H in
//                       distributed shared memory (d <= ~640), else a
//                       cooperative grid kernel over an L2-resident copy
//                       (also the complex Hermitian path, config 5).
//   2. bisect_kernel    the wanted eigenvalues of T by Sturm-count multisection,
//                       one warp per eigenvalue (32 probe points per round).
//   3. invit_kernel     eigenvectors of T by inverse iteration, one warp per
//                       wanted eigenvalue, distinct pseudo-random starts.
//   4. group_kernel +   clusters of (near-)degenerate eigenvalues (gap <
//      group_chol +     1e-7 ||T||) orthonormalised as blocks (K2 Gram, one-CTA
//      Newton-Schulz    Cholesky per cluster, K3 update), then two Newton-Schulz
//                       steps: vectors of distinct clusters are orthogonal to
//                       O(eps ||T|| / gap), so the polish moves residuals by
//                       only O(eps ||T||).
//   5. backtr_*         Z = Q U applying the stored reflectors.
// Why not Jacobi for d > 64: a cyclic Jacobi sweep is d-1 dependent rounds and
// ~10 sweeps are needed, so it is latency-bound (96 ms at d = 288 on one CTA,
// profiles/r01_bench_first.log); this path has O(d) dependent steps in total.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>
#include <utility>

#include "bk_chol.cuh"

namespace bk {
namespace {

constexpr int kTriThreads = 1024;
constexpr int kTriSmemMaxM = 150;  // trailing block m x m in shared memory when m <= 150
constexpr int kSyevMaxD = 1200;  // 4d + 151^2 doubles of shared memory <= 227 KB
// the one-CTA Jacobi path is kept for BK_SYEV_JACOBI_MAX=<d> tuning runs: the
// tridiagonal path measured faster at every d (tools/syev_probe.py, all pairs:
// d = 16 173 -> 115 us, 40 568 -> 208 us; config 1 end to end 2.90 -> 2.37 s)
constexpr int kSyevJacobiMaxD = 0;

// ------------------------------------------------------------------ 1. tridiagonalisation
// a: d x d working copy (row-major, lda = d), symmetric, both triangles kept.
// On exit: diag[k], off[k] (T(k+1,k)), reflector k stored in vref[k*d + i]
// for i < d-k-1 (v[0] = 1), tau[k].

// Fused variant (the one launched): the rank-2 update of step k-1 is applied
// lazily inside step k's single pass over the trailing block, which also
// accumulates p = A v for step k — one read + one write of the trailing block
// per step instead of two reads + one write.
__global__ void __launch_bounds__(kTriThreads) tridiag_fused_kernel(int d, const double* __restrict__ h, int ldh,
                                                                     double* __restrict__ a,
                                                                     double* __restrict__ vref,
                                                                     double* __restrict__ tau,
                                                                     double* __restrict__ diag,
                                                                     double* __restrict__ off) {
    extern __shared__ double sm[];
    __shared__ double red[kTriThreads / 32];
    __shared__ double s_scal[2];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    double* v = sm;           // current reflector (absolute row index)
    double* vp = sm + d;      // pending update: previous reflector
    double* wp = sm + 2 * d;  // pending update: previous w
    double* col = sm + 3 * d; // column k after the pending update; reused for p / w
    double* tri = sm + 4 * d; // trailing block once it fits
    for (int e = tid; e < d * d; e += nt) {
        const int i = e / d, j = e - i * d;
        a[e] = 0.5 * (h[static_cast<size_t>(i) * ldh + j] + h[static_cast<size_t>(j) * ldh + i]);
    }
    for (int i = tid; i < d; i += nt) {
        vp[i] = 0.0;
        wp[i] = 0.0;
    }
    __syncthreads();
    bool in_smem = false;
    int base = 0, ld = d;
    double* st = a;  // storage of rows/cols >= base
    auto block_sum = [&](double x) {
        x = warp_sum(x);
        if (lane == 0) red[wid] = x;
        __syncthreads();
        // second level by shuffles in every warp (one LDS per lane instead of a
        // serial walk over the warp partials): same butterfly everywhere, so every
        // thread — and every CTA of a cluster — gets bit-identical results
        const double s = warp_sum(lane < nw ? red[lane] : 0.0);
        __syncthreads();
        return s;
    };
    for (int k = 0; k + 2 < d; ++k) {
        const int m = d - k - 1;
        if (!in_smem && m + 1 <= kTriSmemMaxM + 1) {
            const int mm = d - k;
            for (int e = tid; e < mm * mm; e += nt) {
                const int i = e / mm, j = e - i * mm;
                tri[e] = a[static_cast<size_t>(k + i) * d + k + j];
            }
            __syncthreads();
            in_smem = true;
            base = k;
            ld = mm;
            st = tri;
        }
        // (1) column k with the pending update applied
        const double vpk = vp[k], wpk = wp[k];
        double xs = 0.0;
        for (int r = k + tid; r < d; r += nt) {
            const double x = st[static_cast<size_t>(r - base) * ld + (k - base)] - (vp[r] * wpk + wp[r] * vpk);
            col[r] = x;
            if (r >= k + 2) xs = fma(x, x, xs);
        }
        const double xnorm2 = block_sum(xs);  // includes a __syncthreads: col[] visible
        // (2) reflector
        if (tid == 0) {
            const double alpha = col[k + 1];
            diag[k] = col[k];
            double t = 0.0, beta = alpha, scal = 0.0;
            if (xnorm2 > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
                t = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            off[k] = beta;
            tau[k] = t;
            s_scal[0] = t;
            s_scal[1] = scal;
        }
        __syncthreads();
        const double t = s_scal[0], scal = s_scal[1];
        for (int r = k + 1 + tid; r < d; r += nt) {
            const double vr = r == k + 1 ? 1.0 : col[r] * scal;
            v[r] = vr;
            vref[static_cast<size_t>(k) * d + (r - k - 1)] = vr;
        }
        __syncthreads();
        // (3) fused pass: apply the pending update to the trailing block and
        //     accumulate p = t * A22 v (warp per row, lanes across the row)
        // 8 independent loads per lane in flight: one CTA must cover L2 latency
        constexpr int U = 8;
        for (int i = k + 1 + wid; i < d; i += nw) {
            double* row = st + static_cast<size_t>(i - base) * ld - base;
            const double vpi = vp[i], wpi = wp[i];
            double s = 0.0;
            for (int j0 = k + 1 + lane; j0 < d; j0 += 32 * U) {
                double x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + 32 * u;
                    x[u] = j < d ? row[j] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + 32 * u;
                    if (j < d) {
                        const double y = x[u] - (vpi * wp[j] + wpi * vp[j]);
                        row[j] = y;
                        s = fma(y, v[j], s);
                    }
                }
            }
            s = warp_sum(s);
            if (lane == 0) col[i] = t * s;  // p_i (column k no longer needed)
        }
        __syncthreads();
        // (4) w = p - (t/2)(p^T v) v becomes the pending update
        double pv = 0.0;
        for (int i = k + 1 + tid; i < d; i += nt) pv = fma(col[i], v[i], pv);
        const double kk = -0.5 * t * block_sum(pv);
        for (int i = k + 1 + tid; i < d; i += nt) {
            wp[i] = fma(kk, v[i], col[i]);
            vp[i] = v[i];
        }
        __syncthreads();
    }
    // last 2 x 2 block with the final pending update
    if (tid == 0) {
        const int k = d - 2;
        auto at = [&](int i, int j) { return st[static_cast<size_t>(i - base) * ld + (j - base)] - (vp[i] * wp[j] + wp[i] * vp[j]); };
        diag[k] = at(k, k);
        off[k] = at(k + 1, k);
        diag[k + 1] = at(k + 1, k + 1);
        off[k + 1] = 0.0;
        tau[k] = 0.0;
        tau[k + 1] = 0.0;
    }
}

// Cluster variant (used whenever the matrix fits in the cluster's shared
// memory): a thread-block cluster of C CTAs (C = 1..16) keeps the whole
// symmetric matrix resident in distributed shared memory, rows distributed
// cyclically (row i on rank i % C).  Per step: every rank updates its part of
// column k and scatters it to all ranks through DSMEM; after one cluster
// barrier each rank computes the (identical) reflector redundantly; the fused
// update + matvec runs on local rows; the p slices are all-gathered through
// DSMEM and, after a second barrier, every rank forms w redundantly.
// Reductions run in the same fixed order on every rank, so the replicated
// scalars are bit-identical.
constexpr int kClThreads = 512;

template <int NT = kClThreads>
__global__ void __launch_bounds__(NT) tridiag_cluster_kernel(int d, const double* __restrict__ h, int ldh,
                                                                      double* __restrict__ vref,
                                                                      double* __restrict__ tau,
                                                                      double* __restrict__ diag,
                                                                      double* __restrict__ off) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int C = static_cast<int>(cl.num_blocks());
    const int rank = static_cast<int>(cl.block_rank());
    extern __shared__ double sm[];
    __shared__ double red[NT / 32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int nloc = (d + C - 1) / C;
    double* A = sm;                       // local rows: A[t*d + j] is row rank + C*t
    double* v = A + static_cast<size_t>(nloc) * d;
    double* vp = v + d;
    double* wp = vp + d;
    double* col = wp + d;
    double* p = col + d;
    for (int e = tid; e < nloc * d; e += nt) {
        const int t = e / d, j = e - t * d;
        const int i = rank + C * t;
        if (i < d) A[e] = 0.5 * (h[static_cast<size_t>(i) * ldh + j] + h[static_cast<size_t>(j) * ldh + i]);
    }
    for (int i = tid; i < d; i += nt) {
        vp[i] = 0.0;
        wp[i] = 0.0;
    }
    auto block_sum = [&](double x) {
        x = warp_sum(x);
        if (lane == 0) red[wid] = x;
        __syncthreads();
        // second level by shuffles in every warp (one LDS per lane instead of a
        // serial walk over the warp partials): same butterfly everywhere, so every
        // thread — and every CTA of a cluster — gets bit-identical results
        const double s = warp_sum(lane < nw ? red[lane] : 0.0);
        __syncthreads();
        return s;
    };
    cl.sync();
    for (int k = 0; k + 2 < d; ++k) {
        // phase 1: own rows r >= k of column k (pending update applied), scattered to every rank
        const int t0 = k <= rank ? 0 : (k - rank + C - 1) / C;
        const double vpk = vp[k], wpk = wp[k];
        for (int t = t0 + tid; t < nloc; t += nt) {
            const int r = rank + C * t;
            if (r >= d) break;
            const double x = A[static_cast<size_t>(t) * d + k] - (vp[r] * wpk + wp[r] * vpk);
            for (int q = 0; q < C; ++q) cl.map_shared_rank(col, q)[r] = x;
        }
        cl.sync();
        // phase 1b (replicated): reflector from col[k+1:]
        double xs = 0.0;
        for (int r = k + 2 + tid; r < d; r += nt) xs = fma(col[r], col[r], xs);
        const double xnorm2 = block_sum(xs);
        const double alpha = col[k + 1];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (xnorm2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        for (int r = k + 1 + tid; r < d; r += nt) {
            const double vr = r == k + 1 ? 1.0 : col[r] * scal;
            v[r] = vr;
            if (rank == 0) vref[static_cast<size_t>(k) * d + (r - k - 1)] = vr;
        }
        if (rank == 0 && tid == 0) {
            diag[k] = col[k];
            off[k] = beta;
            tau[k] = t;
        }
        __syncthreads();
        // phase 2: fused pending update + p = t A22 v on local rows i >= k+1
        // four local rows per warp pass: v / vp / wp are loaded once for the four
        // rows and the four dot-product chains overlap (latency, not flops, bounds
        // this phase)
        const int t1 = k + 1 <= rank ? 0 : (k + 1 - rank + C - 1) / C;
        for (int tb = t1 + 4 * wid; tb < nloc; tb += 4 * nw) {
            int ii[4];
            double* rows[4];
            double vpi[4], wpi[4], s[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int tt = tb + q;
                ii[q] = rank + C * tt;
                const bool ok = tt < nloc && ii[q] < d;
                rows[q] = ok ? A + static_cast<size_t>(tt) * d : nullptr;
                vpi[q] = ok ? vp[ii[q]] : 0.0;
                wpi[q] = ok ? wp[ii[q]] : 0.0;
                s[q] = 0.0;
            }
            for (int j = k + 1 + lane; j < d; j += 32) {
                const double vj = v[j], vpj = vp[j], wpj = wp[j];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (rows[q]) {
                        const double x = rows[q][j] - (vpi[q] * wpj + wpi[q] * vpj);
                        rows[q][j] = x;
                        s[q] = fma(x, vj, s[q]);
                    }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) s[q] = warp_sum(s[q]) * t;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (rows[q] && lane < C) cl.map_shared_rank(p, lane)[ii[q]] = s[q];
        }
        cl.sync();
        // phase 3 (replicated): w = p - (t/2)(p^T v) v becomes the pending update
        double pv = 0.0;
        for (int i = k + 1 + tid; i < d; i += nt) pv = fma(p[i], v[i], pv);
        const double kk = -0.5 * t * block_sum(pv);
        for (int i = k + 1 + tid; i < d; i += nt) wp[i] = fma(kk, v[i], p[i]);
        {  // v becomes the pending vp (local buffers: a pointer swap, no copy)
            double* t2 = vp;
            vp = v;
            v = t2;
        }
        __syncthreads();
    }
    // last 2 x 2 block: owners of rows d-2, d-1 publish their entries to rank 0
    if (d >= 2) {
        const int k = d - 2;
        for (int r = k + tid; r < d; r += nt) {
            if (r % C != rank) continue;
            const int t = r / C;
            const double* row = A + static_cast<size_t>(t) * d;
            double* c0 = cl.map_shared_rank(col, 0);
            c0[r] = row[k] - (vp[r] * wp[k] + wp[r] * vp[k]);                               // A(r, d-2)
            if (r == d - 1) c0[d] = row[d - 1] - (vp[r] * wp[d - 1] + wp[r] * vp[d - 1]);  // A(d-1, d-1)
        }
    }
    cl.sync();
    if (rank == 0 && tid == 0) {
        const int k = d - 2;
        diag[k] = col[k];
        off[k] = col[k + 1];
        diag[k + 1] = col[d];
        off[k + 1] = 0.0;
        tau[k] = 0.0;
        tau[k + 1] = 0.0;
    }
}

// Packed single-CTA variant (d <= kPackedMaxD, config 2's shrunk d = 3 x 69 =
// 207): the lower triangle (d(d+1)/2 doubles, 171 KB at d = 207) stays in one
// SM's shared memory for the whole reduction, so a step costs CTA barriers
// (~100 cycles) instead of cluster barriers and DSMEM round trips.  The fused
// pass reads and writes each trailing lower element once: lane l owns columns
// j = k+1+l+32m (their v / vp / wp in registers for the step), warp w owns rows
// i = k+1+w+16r; an element x_ij (j <= i) adds x_ij v_j to row i's sum (lane
// partials in rowacc[r], reduced once per row at the end of the pass) and, off
// the diagonal, x_ij v_i to column j's sum (colacc[m], combined over warps in a
// fixed order) — the symmetric matvec without storing the upper triangle.
constexpr int kPkThreads = 512, kPkWarps = kPkThreads / 32;
constexpr int kPkM = 7, kPkR = 14;  // column chunks per lane, rows per warp (<= 16): d - 1 <= 224
constexpr int kPackedMaxD = 218;    // d(d+1)/2 + 22 d doubles <= 227 KB
// launched up to d = 160: one SM's issue rate bounds the fused pass, and above
// ~165 the 8-CTA cluster kernel is faster (tools/syev_probe.py, syev incl.
// bisection etc.: d = 100 480 vs 522 us, 160 815 vs 818, 207 1160 vs 1076)
constexpr int kPackedUseMaxD = 160;

inline size_t packed_smem_bytes(int d) {
    return sizeof(double) * (static_cast<size_t>(d) * (d + 1) / 2 + static_cast<size_t>(6 + kPkWarps) * d);
}

template <int NT_, int PM, int PR>
__global__ void __launch_bounds__(NT_, 1) tridiag_packed_kernel(int d, const double* __restrict__ h, int ldh,
                                                                        double* __restrict__ vref,
                                                                        double* __restrict__ tau,
                                                                        double* __restrict__ diag,
                                                                        double* __restrict__ off) {
    extern __shared__ double sm[];
    __shared__ double red[NT_ / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int nt = NT_, nw = NT_ / 32;
    static_assert(PR <= 16, "the row reduce-scatter serves 16 rows per warp");
    double* A = sm;  // row i of the lower triangle at A + i(i+1)/2
    double* v = A + static_cast<size_t>(d) * (d + 1) / 2;
    double* vp = v + d;
    double* wp = vp + d;
    double* col = wp + d;  // column k after the pending update
    double* rp = col + d;  // row parts of p
    double* p = rp + d;
    double* cp = p + d;  // [nw][d] column partials
    auto rowp = [&](int i) { return A + (static_cast<size_t>(i) * (i + 1) >> 1); };
    for (int i = wid; i < d; i += nw) {
        double* r = rowp(i);
        for (int j = lane; j <= i; j += 32)
            r[j] = 0.5 * (h[static_cast<size_t>(i) * ldh + j] + h[static_cast<size_t>(j) * ldh + i]);
    }
    for (int i = tid; i < d; i += nt) {
        vp[i] = 0.0;
        wp[i] = 0.0;
    }
    auto block_sum = [&](double x) {  // same butterfly in every thread: bit-identical results
        x = warp_sum(x);
        if (lane == 0) red[wid] = x;
        __syncthreads();
        const double s = warp_sum(lane < nw ? red[lane] : 0.0);
        __syncthreads();
        return s;
    };
    __syncthreads();
    for (int k = 0; k + 2 < d; ++k) {
        // (1) column k (rows r >= k) with the pending update applied; reflector norm
        const double vpk = vp[k], wpk = wp[k];
        double xs = 0.0;
        for (int r = k + tid; r < d; r += nt) {
            const double x = rowp(r)[k] - (vp[r] * wpk + wp[r] * vpk);
            col[r] = x;
            if (r >= k + 2) xs = fma(x, x, xs);
        }
        const double xnorm2 = block_sum(xs);  // barrier inside: col[] visible
        const double alpha = col[k + 1];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (xnorm2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
            t = (beta - alpha) * __drcp_rn(beta);  // reciprocals: no division routine on the step's chain
            scal = __drcp_rn(alpha - beta);
        }
        for (int r = k + 1 + tid; r < d; r += nt) {
            const double vr = r == k + 1 ? 1.0 : col[r] * scal;
            v[r] = vr;
            vref[static_cast<size_t>(k) * d + (r - k - 1)] = vr;
        }
        if (tid == 0) {
            diag[k] = col[k];
            off[k] = beta;
            tau[k] = t;
        }
        __syncthreads();
        // (2) fused pass over the trailing lower triangle (rows, cols >= j0)
        const int j0 = k + 1;
        double vj[PM], vpj[PM], wpj[PM], cacc[PM];
#pragma unroll
        for (int m = 0; m < PM; ++m) {
            const int j = j0 + lane + 32 * m;
            const bool ok = j < d;
            vj[m] = ok ? v[j] : 0.0;
            vpj[m] = ok ? vp[j] : 0.0;
            wpj[m] = ok ? wp[j] : 0.0;
            cacc[m] = 0.0;
        }
        // loops leave by warp-uniform breaks: the trailing triangle shrinks with k,
        // and guarded-but-unrolled bodies would be predicated, not skipped
        double racc[PR];
#pragma unroll
        for (int r = 0; r < PR; ++r) racc[r] = 0.0;
#pragma unroll
        for (int r = 0; r < PR; ++r) {
            const int i = j0 + wid + nw * r;
            if (i >= d) break;
            double* row = rowp(i);
            const double vi = v[i], vpi = vp[i], wpi = wp[i];
            const int mhi = (i - j0) >> 5;  // last chunk holding a j <= i
#pragma unroll
            for (int m = 0; m < PM; ++m) {
                if (m > mhi) break;
                const int j = j0 + lane + 32 * m;
                if (j <= i) {
                    const double x = row[j] - (vpi * wpj[m] + wpi * vpj[m]);
                    row[j] = x;
                    racc[r] = fma(x, vj[m], racc[r]);
                    if (j < i) cacc[m] = fma(x, vi, cacc[m]);
                }
            }
        }
        // the 16 row sums of the warp by one reduce-scatter across the lanes
        // (16 shuffles instead of 16 warp_sums' 80); lane pair (2q, 2q+1) ends
        // with row q's sum, the butterfly order fixed (deterministic)
        {
            double v8[8], v4[4], v2[2];
            const bool h1 = lane & 16, h2 = lane & 8, h3 = lane & 4, h4 = lane & 2;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double lo8 = q < PR ? racc[q] : 0.0, hi8 = q + 8 < PR ? racc[q + 8] : 0.0;
                v8[q] = (h1 ? hi8 : lo8) + __shfl_xor_sync(0xffffffffu, h1 ? lo8 : hi8, 16);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                v4[q] = (h2 ? v8[q + 4] : v8[q]) + __shfl_xor_sync(0xffffffffu, h2 ? v8[q] : v8[q + 4], 8);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                v2[q] = (h3 ? v4[q + 2] : v4[q]) + __shfl_xor_sync(0xffffffffu, h3 ? v4[q] : v4[q + 2], 4);
            double v1 = (h4 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? v2[0] : v2[1], 2);
            v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
            const int r = (h1 ? 8 : 0) + (h2 ? 4 : 0) + (h3 ? 2 : 0) + (h4 ? 1 : 0);
            const int i = j0 + wid + nw * r;
            if (!(lane & 1) && i < d) rp[i] = v1;
        }
#pragma unroll
        for (int m = 0; m < PM; ++m) {
            const int j = j0 + lane + 32 * m;
            if (j < d) cp[wid * d + j] = cacc[m];
        }
        __syncthreads();
        // (3) p = t (row part + column parts, fixed warp order); w = p - (t/2)(p^T v) v
        double pv = 0.0;
        for (int j = j0 + tid; j < d; j += nt) {
            double s = rp[j];
#pragma unroll
            for (int w = 0; w < nw; ++w) s += cp[w * d + j];
            const double pj = t * s;
            p[j] = pj;
            pv = fma(pj, v[j], pv);
        }
        const double kk = -0.5 * t * block_sum(pv);
        for (int j = j0 + tid; j < d; j += nt) wp[j] = fma(kk, v[j], p[j]);
        {  // v becomes the pending vp (pointer swap)
            double* t2 = vp;
            vp = v;
            v = t2;
        }
        __syncthreads();
    }
    if (tid == 0) {
        const int k = d - 2;
        auto at = [&](int i, int j) { return rowp(i)[j] - (vp[i] * wp[j] + wp[i] * vp[j]); };
        diag[k] = at(k, k);
        off[k] = at(k + 1, k);
        diag[k + 1] = at(k + 1, k + 1);
        off[k + 1] = 0.0;
        tau[k] = 0.0;
        tau[k + 1] = 0.0;
    }
}

// One-barrier cluster variant: the reflector of step k+1 needs column k+1,
// which by symmetry is row k+1 — owned by one rank, and final for step k+1 as
// soon as step k's fused pass has updated it.  So that pass also broadcasts the
// stored row k+1 (DSMEM, double-buffered by step parity) next to the p slices,
// and after the one cluster barrier every rank applies the pending rank-2 update
// to it locally and forms the reflector redundantly: one cluster barrier per
// step instead of two (the column scatter and its barrier are gone).  Column k
// is read from the stored row k instead of the stored column (equal up to the
// rounding of the contracted rank-2 update), otherwise the arithmetic is the
// two-barrier kernel's.
template <int NT>
__global__ void __launch_bounds__(NT) tridiag_cluster1_kernel(int d, const double* __restrict__ h, int ldh,
                                                              double* __restrict__ vref, double* __restrict__ tau,
                                                              double* __restrict__ diag, double* __restrict__ off) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int C = static_cast<int>(cl.num_blocks());
    const int rank = static_cast<int>(cl.block_rank());
    extern __shared__ double sm[];
    __shared__ double red[NT / 32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int nloc = (d + C - 1) / C;
    double* A = sm;  // local rows: A[t*d + j] is row rank + C*t
    double* v = A + static_cast<size_t>(nloc) * d;
    double* vp = v + d;
    double* wp = vp + d;
    double* col = wp + d;
    double* pb[2] = {col + d, col + 2 * d};     // p slices, by step parity
    double* rb[2] = {col + 3 * d, col + 4 * d};  // broadcast stored row k, by step parity
    for (int e = tid; e < nloc * d; e += nt) {
        const int t = e / d, j = e - t * d;
        const int i = rank + C * t;
        if (i < d) A[e] = 0.5 * (h[static_cast<size_t>(i) * ldh + j] + h[static_cast<size_t>(j) * ldh + i]);
    }
    for (int i = tid; i < d; i += nt) {
        vp[i] = 0.0;
        wp[i] = 0.0;
    }
    auto block_sum = [&](double x) {
        x = warp_sum(x);
        if (lane == 0) red[wid] = x;
        __syncthreads();
        const double s = warp_sum(lane < nw ? red[lane] : 0.0);
        __syncthreads();
        return s;
    };
    cl.sync();  // every rank's rows are loaded before row 0 is read remotely
    if (rank == 0)  // row 0 (rank 0's local row 0), symmetrised above, to every rank
        for (int j = tid; j < d; j += nt) {
            const double x = A[j];
            for (int q = 0; q < C; ++q) cl.map_shared_rank(rb[0], q)[j] = x;
        }
    cl.sync();
    for (int k = 0; k + 2 < d; ++k) {
        // (1) column k = stored row k with the pending update applied (replicated)
        const double* rk = rb[k & 1];
        const double vpk = vp[k], wpk = wp[k];
        double xs = 0.0;
        for (int r = k + tid; r < d; r += nt) {
            const double x = rk[r] - (vp[r] * wpk + wp[r] * vpk);
            col[r] = x;
            if (r >= k + 2) xs = fma(x, x, xs);
        }
        const double xnorm2 = block_sum(xs);
        const double alpha = col[k + 1];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (xnorm2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
            t = (beta - alpha) * __drcp_rn(beta);  // reciprocals: no division routine on the step's chain
            scal = __drcp_rn(alpha - beta);
        }
        for (int r = k + 1 + tid; r < d; r += nt) {
            const double vr = r == k + 1 ? 1.0 : col[r] * scal;
            v[r] = vr;
            if (rank == 0) vref[static_cast<size_t>(k) * d + (r - k - 1)] = vr;
        }
        if (rank == 0 && tid == 0) {
            diag[k] = col[k];
            off[k] = beta;
            tau[k] = t;
        }
        __syncthreads();
        // (2) fused pending update + p = t A22 v on local rows i >= k+1; the
        // owner of row k+1 also broadcasts it (its stored values for step k+1)
        double* p = pb[k & 1];
        double* rn = rb[(k + 1) & 1];
        const int t1 = k + 1 <= rank ? 0 : (k + 1 - rank + C - 1) / C;
        for (int tb = t1 + 4 * wid; tb < nloc; tb += 4 * nw) {
            int ii[4];
            double* rows[4];
            double vpi[4], wpi[4], sacc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int tt = tb + q;
                ii[q] = rank + C * tt;
                const bool ok = tt < nloc && ii[q] < d;
                rows[q] = ok ? A + static_cast<size_t>(tt) * d : nullptr;
                vpi[q] = ok ? vp[ii[q]] : 0.0;
                wpi[q] = ok ? wp[ii[q]] : 0.0;
                sacc[q] = 0.0;
            }
            const int bq = ii[0] == k + 1 ? 0 : -1;  // row k+1 is the first local row it can be
            for (int j = k + 1 + lane; j < d; j += 32) {
                const double vj = v[j], vpj = vp[j], wpj = wp[j];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (rows[q]) {
                        const double x = rows[q][j] - (vpi[q] * wpj + wpi[q] * vpj);
                        rows[q][j] = x;
                        sacc[q] = fma(x, vj, sacc[q]);
                        if (q == bq)
                            for (int r = 0; r < C; ++r) cl.map_shared_rank(rn, r)[j] = x;
                    }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) sacc[q] = warp_sum(sacc[q]) * t;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (rows[q] && lane < C) cl.map_shared_rank(p, lane)[ii[q]] = sacc[q];
        }
        cl.sync();
        // (3) w = p - (t/2)(p^T v) v becomes the pending update (replicated)
        double pv = 0.0;
        for (int i = k + 1 + tid; i < d; i += nt) pv = fma(p[i], v[i], pv);
        const double kk = -0.5 * t * block_sum(pv);
        for (int i = k + 1 + tid; i < d; i += nt) wp[i] = fma(kk, v[i], p[i]);
        {
            double* t2 = vp;
            vp = v;
            v = t2;
        }
        __syncthreads();
    }
    // last 2 x 2 block: owners of rows d-2, d-1 publish their entries to rank 0
    if (d >= 2) {
        const int k = d - 2;
        for (int r = k + tid; r < d; r += nt) {
            if (r % C != rank) continue;
            const int t = r / C;
            const double* row = A + static_cast<size_t>(t) * d;
            double* c0 = cl.map_shared_rank(col, 0);
            c0[r] = row[k] - (vp[r] * wp[k] + wp[r] * vp[k]);
            if (r == d - 1) c0[d] = row[d - 1] - (vp[r] * wp[d - 1] + wp[r] * vp[d - 1]);
        }
    }
    cl.sync();
    if (rank == 0 && tid == 0) {
        const int k = d - 2;
        diag[k] = col[k];
        off[k] = col[k + 1];
        diag[k + 1] = col[d];
        off[k + 1] = 0.0;
        tau[k] = 0.0;
        tau[k + 1] = 0.0;
    }
}

template <class K>
cudaError_t prep_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

// cluster size for the distributed tridiagonalisation, 0 when it does not fit
int tridiag_cluster_size(int d, size_t* smem) {
    // at least 8 CTAs: shorter per-rank row passes outweigh the wider cluster
    // barrier (d = 288: 1.93 -> 1.84 ms per syev; 16 is slower again).
    // BK_TRI_CLUSTER overrides the minimum (tuning runs only).
    static const int c0 = [] {
        const char* e = getenv("BK_TRI_CLUSTER");
        return e ? max(1, atoi(e)) : 8;
    }();
    for (int c = c0; c <= 16; c *= 2) {
        const size_t nloc = static_cast<size_t>((d + c - 1) / c);
        // + 3 d: the one-barrier kernel's second p buffer and two row buffers
        const size_t bytes = sizeof(double) * (nloc * d + 8 * static_cast<size_t>(d) + 8);
        if (bytes <= 200 * 1024) {
            *smem = bytes;
            return c;
        }
    }
    return 0;
}

// ------------------------------------------------------------------ 2. bisection
// Number of eigenvalues of T below x: sign changes of the leading principal
// minors p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} (Wilkinson's continuant
// form of the Sturm sequence; two dependent FMAs per step instead of the
// LDL^T form's division, whose ~60-cycle latency bounded the chain).  The
// pair (p_{i-1}, p_i) is rescaled by exact powers of two to stay in range; a
// zero minor takes the sign opposite to its predecessor (the LDL^T form's
// "q = -pivmin" convention).
__device__ __forceinline__ int sturm_count(int d, const double* __restrict__ dg, const double* __restrict__ off,
                                           double x, double pivmin, bool fast4) {
    (void)pivmin;
    constexpr double kBig = 0x1p+500, kScale = 0x1p-500;
    int cnt = 0;
    double pm = 1.0;       // p_{i-1}
    double p = dg[0] - x;  // p_i
    bool neg_prev = false;  // sign of p_{i-1} (p_0 = 1 > 0)
    bool neg = p < 0.0 || (p == 0.0 && !neg_prev);
    cnt += neg != neg_prev;
    auto step = [&](int i) {  // off holds the SQUARED off-diagonal here
        const double pn = fma(dg[i] - x, p, -off[i - 1] * pm);
        pm = p;
        p = pn;
        neg_prev = neg;
        neg = p < 0.0 || (p == 0.0 && !neg_prev);
        cnt += neg != neg_prev;
    };
    auto rescale = [&]() {  // branchless: the lanes' probes diverge in magnitude
        const double ap = fmax(fabs(p), fabs(pm));
        const double f = ap > kBig ? kScale : (ap < kScale ? kBig : 1.0);
        p *= f;
        pm *= f;
    };
    int i = 1;
    if (fast4) {  // ||T|| < 2^25: four steps grow |p| by < 2^204, so rescale every fourth
        for (; i + 3 < d; i += 4) {
            step(i);
            step(i + 1);
            step(i + 2);
            step(i + 3);
            rescale();
        }
    }
    for (; i < d; ++i) {
        step(i);
        rescale();
    }
    return cnt;
}

// one warp per eigenvalue index j < n_need; 32-way multisection
__global__ void __launch_bounds__(256) bisect_kernel(int d, const double* __restrict__ dg,
                                                      const double* __restrict__ off, int n_need,
                                                      double* __restrict__ lam, double* __restrict__ e2buf) {
    const int lane = threadIdx.x & 31;
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    (void)e2buf;
    // T (diagonal, squared off-diagonal) in shared memory: the Sturm chain's
    // operand loads are LDS (~30 cycles) instead of L1/L2 round trips
    extern __shared__ double bsm_t[];
    double* sdg = bsm_t;
    double* se2 = bsm_t + d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        sdg[i] = dg[i];
        se2[i] = i + 1 < d ? off[i] * off[i] : 0.0;
    }
    __syncthreads();
    if (j >= n_need) return;
    // Gershgorin interval and pivmin (every warp, O(d))
    double lo = INFINITY, hi = -INFINITY, emax2 = 0.0;
    for (int i = lane; i < d; i += 32) {
        const double r = (i > 0 ? fabs(off[i - 1]) : 0.0) + (i + 1 < d ? fabs(off[i]) : 0.0);
        lo = fmin(lo, dg[i] - r);
        hi = fmax(hi, dg[i] + r);
        if (i + 1 < d) emax2 = fmax(emax2, off[i] * off[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pivmin = DBL_MIN * fmax(1.0, emax2);
    const double slack = 2.0 * DBL_EPSILON * tnorm + pivmin;
    lo -= slack;
    hi += slack;
    // invariant: count(lo) <= j < count(hi)
    for (int it = 0; it < 40; ++it) {
        const double width = hi - lo;
        if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
        const double x = lo + width * (lane + 1) / 33.0;
        const int c = sturm_count(d, sdg, se2, x, pivmin, tnorm < 0x1p+25);
        // first lane whose probe has more than j eigenvalues below it
        const unsigned above = __ballot_sync(0xffffffffu, c > j);
        const int first = above ? __ffs(above) - 1 : 32;
        const double new_lo = first == 0 ? lo : __shfl_sync(0xffffffffu, x, max(first - 1, 0));
        const double new_hi = first == 32 ? hi : __shfl_sync(0xffffffffu, x, min(first, 31));
        if (new_lo == lo && new_hi == hi) break;
        lo = new_lo;
        hi = new_hi;
    }
    if (lane == 0) lam[j] = 0.5 * (lo + hi);
}

// One CTA of W warps per eigenvalue index j: (32W + 1)-way multisection, so a
// round shrinks the bracket 257-fold at W = 8 (8 rounds to full precision
// instead of 12-13 at 33-fold) and the eigenvalues' CTAs fill the SMs' sub-
// partitions instead of one warp each.  Probe t sits at lo + width (t+1)/(N+1),
// a formula every thread evaluates identically, so the new bracket needs no
// exchange of probe values — only the first probe index above j (ballot per
// warp, minimum over warps).
template <int W>
__global__ void __launch_bounds__(32 * W) bisect_multi_kernel(int d, const double* __restrict__ dg,
                                                              const double* __restrict__ off, int n_need,
                                                              double* __restrict__ lam) {
    constexpr int N = 32 * W;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int j = blockIdx.x;
    extern __shared__ double bsm_t[];
    __shared__ int s_first[2][W];
    double* sdg = bsm_t;
    double* se2 = bsm_t + d;
    for (int i = tid; i < d; i += N) {
        sdg[i] = dg[i];
        se2[i] = i + 1 < d ? off[i] * off[i] : 0.0;
    }
    __syncthreads();
    if (j >= n_need) return;
    double lo = INFINITY, hi = -INFINITY, emax2 = 0.0;
    for (int i = lane; i < d; i += 32) {
        const double r = (i > 0 ? fabs(off[i - 1]) : 0.0) + (i + 1 < d ? fabs(off[i]) : 0.0);
        lo = fmin(lo, dg[i] - r);
        hi = fmax(hi, dg[i] + r);
        if (i + 1 < d) emax2 = fmax(emax2, off[i] * off[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pivmin = DBL_MIN * fmax(1.0, emax2);
    const double slack = 2.0 * DBL_EPSILON * tnorm + pivmin;
    lo -= slack;
    hi += slack;
    const bool fast4 = tnorm < 0x1p+25;
    for (int it = 0; it < 40; ++it) {
        const double width = hi - lo;
        if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
        const double x = lo + width * (tid + 1) / static_cast<double>(N + 1);
        const int c = sturm_count(d, sdg, se2, x, pivmin, fast4);
        const unsigned above = __ballot_sync(0xffffffffu, c > j);
        if (lane == 0) s_first[it & 1][wid] = above ? wid * 32 + __ffs(above) - 1 : N;
        __syncthreads();
        int first = N;
#pragma unroll
        for (int w = 0; w < W; ++w) first = min(first, s_first[it & 1][w]);
        const double new_lo = first == 0 ? lo : lo + width * first / static_cast<double>(N + 1);
        const double new_hi = first == N ? hi : lo + width * (first + 1) / static_cast<double>(N + 1);
        if (new_lo == lo && new_hi == hi) break;
        lo = new_lo;
        hi = new_hi;
    }
    if (tid == 0) lam[j] = 0.5 * (lo + hi);
}

// ------------------------------------------------------------------ 3. inverse iteration
constexpr int kSmallCluster = 8;  // clusters up to this size are orthonormalised by one fused kernel
// groups of consecutive eigenvalues closer than gap_rel * ||T||; gstart[g], ngroups
__global__ void group_kernel(int n_need, const double* __restrict__ lam, const double* __restrict__ dg,
                             const double* __restrict__ off, int d, int* __restrict__ gstart,
                             int* __restrict__ ngroups) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double tnorm = 0.0;
    for (int i = 0; i < d; ++i)
        tnorm = fmax(tnorm, fabs(dg[i]) + (i > 0 ? fabs(off[i - 1]) : 0.0) + (i + 1 < d ? fabs(off[i]) : 0.0));
    const double thr = 1e-7 * fmax(tnorm, DBL_MIN);
    int g = 0;
    for (int j = 0; j < n_need; ++j)
        if (j == 0 || lam[j] - lam[j - 1] > thr) gstart[g++] = j;
    gstart[g] = n_need;
    ngroups[0] = g;
    ngroups[1] = g < n_need ? 1 : 0;  // some cluster has several members
    int big = 0;
    for (int c = 0; c < g; ++c) big |= gstart[c + 1] - gstart[c] > kSmallCluster;
    ngroups[2] = big;  // some cluster is too large for cluster_orth_small_kernel
}

// LU of T - lam I by Gaussian elimination with partial pivoting on the
// tridiagonal (rows i, i+1 may swap; fill-in in u2), stored for repeated
// solves: multipliers, swap flags, the two super-diagonals of U and the
// reciprocal pivots (tiny pivots replaced by +-eps*||T||: inverse iteration on
// an intentionally singular shift).  Factor once, then each inverse-iteration
// step is division-free.
__device__ void tri_factor(int d, const double* __restrict__ dg, const double* __restrict__ off, double lam,
                           double tiny, double* __restrict__ mult, double* __restrict__ rinv,
                           double* __restrict__ u1, double* __restrict__ u2, unsigned char* __restrict__ swp) {
    auto guard = [&](double p) { return fabs(p) < tiny ? copysign(tiny, p == 0.0 ? 1.0 : p) : p; };
    double diag_cur = dg[0] - lam;
    double sup_cur = d > 1 ? off[0] : 0.0;
    double sup2_cur = 0.0;
    for (int i = 0; i + 1 < d; ++i) {
        const double sub = off[i];  // A(i+1, i)
        const double nd = dg[i + 1] - lam;
        const double ns = i + 2 < d ? off[i + 1] : 0.0;
        // one reciprocal per step on the dependent chain, the multiplier from it
        // (two IEEE divisions per step bounded the factorisation)
        if (fabs(sub) > fabs(diag_cur)) {  // swap rows i and i+1
            const double r = __drcp_rn(sub);
            const double m = diag_cur * r;
            mult[i] = m;
            swp[i] = 1;
            rinv[i] = r;
            u1[i] = nd;
            u2[i] = ns;
            diag_cur = sup_cur - m * nd;
            sup_cur = sup2_cur - m * ns;
            sup2_cur = 0.0;
        } else {
            const double p0 = guard(diag_cur);
            const double r = __drcp_rn(p0);
            const double m = sub * r;
            mult[i] = m;
            swp[i] = 0;
            rinv[i] = r;
            u1[i] = sup_cur;
            u2[i] = sup2_cur;
            diag_cur = nd - m * sup_cur;
            sup_cur = ns;
            sup2_cur = 0.0;
        }
    }
    rinv[d - 1] = 1.0 / guard(diag_cur);
}

// b <- (T - lam I)^{-1} b with the stored factors
__device__ void tri_apply(int d, const double* __restrict__ mult, const double* __restrict__ rinv,
                          const double* __restrict__ u1, const double* __restrict__ u2,
                          const unsigned char* __restrict__ swp, double* __restrict__ b) {
    for (int i = 0; i + 1 < d; ++i) {
        if (swp[i]) {
            const double bi = b[i];
            b[i] = b[i + 1];
            b[i + 1] = bi - mult[i] * b[i];
        } else {
            b[i + 1] -= mult[i] * b[i];
        }
    }
    for (int i = d - 1; i >= 0; --i) {
        double s = b[i];
        if (i + 1 < d) s -= u1[i] * b[i + 1];
        if (i + 2 < d) s -= u2[i] * b[i + 2];
        b[i] = s * rinv[i];
    }
}

// one warp per wanted eigenvalue j; u column-major (ldu = d): column j = the
// inverse-iteration vector of T for lam[j].  Vectors are iterated independently
// (no Gram-Schmidt inside a cluster: that serialised a whole cluster on one
// warp); clusters are orthonormalised afterwards as blocks (group_chol_kernel).
__global__ void __launch_bounds__(128) invit_kernel(int d, const double* __restrict__ dg,
                                                     const double* __restrict__ off,
                                                     const double* __restrict__ lam, int n_need,
                                                     double* __restrict__ u, int steps, int from_u,
                                                     const double* __restrict__ src_rm,
                                                     const int* __restrict__ use_rm, double* __restrict__ out_rm) {
    extern __shared__ double ism[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // T staged in shared memory (the solve walks it sequentially), plus a
    // private 4*d workspace per warp: no global round trips on the serial path
    double* sdg = ism;
    double* soff = ism + d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        sdg[i] = dg[i];
        soff[i] = off[i];
    }
    __syncthreads();
    dg = sdg;
    off = soff;
    if (j >= n_need) return;
    // per warp: b, mult, rinv, u1, u2 (5d doubles) + swap flags (d bytes)
    double* b = ism + 2 * d + static_cast<size_t>(wib) * (5 * d + (d + 7) / 8);
    double* mult = b + d;
    double* rinv = mult + d;
    double* u1 = rinv + d;
    double* u2 = u1 + d;
    unsigned char* swp = reinterpret_cast<unsigned char*>(u2 + d);
    double tnorm = 0.0;
    for (int i = lane; i < d; i += 32)
        tnorm = fmax(tnorm, fabs(dg[i]) + (i > 0 ? fabs(off[i - 1]) : 0.0) + (i + 1 < d ? fabs(off[i]) : 0.0));
    for (int o = 16; o > 0; o >>= 1) tnorm = fmax(tnorm, __shfl_xor_sync(0xffffffffu, tnorm, o));
    const double tiny = DBL_EPSILON * fmax(tnorm, DBL_MIN);
    double* uj = u + static_cast<size_t>(j) * d;
    // deterministic pseudo-random start (splitmix64 of (j, i)): distinct starts
    // make the vectors of a degenerate cluster independent; from_u: continue from
    // the vector already in u (the second step, after the clusters of the first
    // step's vectors were orthonormalised as blocks)
    // (src_rm: the block-orthonormalised vectors, row-major d x n_need, when the
    // device flag use_rm says the cluster step ran; out_rm: a row-major copy of the
    // result for the Gram / update kernels — no separate transposition launches)
    if (from_u) {
        if (src_rm && *use_rm) {
            for (int i = lane; i < d; i += 32) b[i] = src_rm[static_cast<size_t>(i) * n_need + j];
        } else {
            for (int i = lane; i < d; i += 32) b[i] = uj[i];
        }
    } else
    for (int i = lane; i < d; i += 32) {
        unsigned long long z = (static_cast<unsigned long long>(j) << 32) + static_cast<unsigned long long>(i) +
                               0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        b[i] = static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
    __syncwarp();
    const double shift = lam[j];
    // two steps in all (one per launch): with the shift accurate to ~eps ||T|| and
    // clusters (gap < 1e-7 ||T||) treated as blocks, each step shrinks foreign
    // components by <= eps/1e-7.  Inside a cluster a step weights the cluster's
    // eigenvectors by 1/(lam_i - shift), differences of rounding size, so all
    // members lean towards the same vector; two unbroken steps square that ratio
    // and once in ~1e4 cluster solves left members parallel to 1e-7 — beyond what
    // the block Cholesky recovers (config 2 `none`@64, iteration 549: a Ritz
    // vector of norm^2 1 + 5e-6, the solve stagnated at 2 tol).  The caller
    // therefore orthonormalises the clusters between the steps.
    if (lane == 0) tri_factor(d, dg, off, shift, tiny, mult, rinv, u1, u2, swp);
    __syncwarp();
    for (int it = 0; it < steps; ++it) {
        if (lane == 0) tri_apply(d, mult, rinv, u1, u2, swp, b);
        __syncwarp();
        double nn = 0.0;
        for (int i = lane; i < d; i += 32) nn = fma(b[i], b[i], nn);
        nn = warp_sum(nn);
        const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
        for (int i = lane; i < d; i += 32) b[i] *= inv;
        __syncwarp();
    }
    for (int i = lane; i < d; i += 32) uj[i] = b[i];
    if (out_rm)
        for (int i = lane; i < d; i += 32) out_rm[static_cast<size_t>(i) * n_need + j] = b[i];
}

// Small clusters (<= kSmallCluster members: the degenerate pairs, triples and
// sextuples of lattice operators) in one launch: CTA b loads its cluster's columns of
// U (column-major, contiguous) into shared memory, forms their Gram matrix with
// fixed-order warp reductions, takes its Cholesky factor R in one thread and writes
// U R^{-1} back in place (and, when asked, a row-major copy of every column it owns,
// singletons included).  A pivot that lost more than 1e-12 of its diagonal, or a
// larger cluster, raises *big, which runs the general path (Gram, per-cluster
// skip-pivot Cholesky, update) after this kernel.
__global__ void __launch_bounds__(128) cluster_orth_small_kernel(int d, int n_need, const int* __restrict__ gstart,
                                                                  const int* __restrict__ ngroups,
                                                                  double* __restrict__ u, double* __restrict__ out_rm,
                                                                  int* __restrict__ big, const int* __restrict__ run_if) {
    extern __shared__ double cols[];  // d x g, column c at cols + c * d
    __shared__ double G[kSmallCluster][kSmallCluster], Ri[kSmallCluster][kSmallCluster];
    __shared__ int ok;
    if (run_if && *run_if == 0) return;
    const int b = blockIdx.x;
    if (b >= ngroups[0]) return;
    const int g0 = gstart[b], g = gstart[b + 1] - g0;
    if (g > kSmallCluster) return;  // ngroups[2] is already set by group_kernel
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* uc = u + static_cast<size_t>(g0) * d;
    if (g == 1) {
        if (out_rm)
            for (int i = tid; i < d; i += blockDim.x) out_rm[static_cast<size_t>(i) * n_need + g0] = uc[i];
        return;
    }
    for (int e = tid; e < d * g; e += blockDim.x) cols[e] = uc[e];
    __syncthreads();
    for (int p = warp; p < g * g; p += 4) {  // upper triangle, one warp per entry, fixed order
        const int a = p / g, c = p - a * g;
        if (a > c) continue;
        double sum = 0.0;
        for (int i = lane; i < d; i += 32) sum = fma(cols[a * d + i], cols[c * d + i], sum);
        sum = warp_sum(sum);
        if (lane == 0) G[a][c] = sum;
    }
    __syncthreads();
    if (tid == 0) {
        int good = 1;
        // R upper triangular, G = R^T R; Ri = R^{-1}
        double R[kSmallCluster][kSmallCluster];
        for (int j = 0; j < g && good; ++j) {
            double p = G[j][j];
            for (int l = 0; l < j; ++l) p -= R[l][j] * R[l][j];
            if (!(p > 1e-12 * G[j][j])) {
                good = 0;
                break;
            }
            const double r = sqrt(p);
            R[j][j] = r;
            for (int c = j + 1; c < g; ++c) {
                double v = G[j][c];
                for (int l = 0; l < j; ++l) v -= R[l][j] * R[l][c];
                R[j][c] = v / r;
            }
        }
        if (good)
            for (int c = 0; c < g; ++c) {  // column c of R^{-1} by back substitution
                for (int a = g - 1; a >= 0; --a) {
                    if (a > c) {
                        Ri[a][c] = 0.0;
                        continue;
                    }
                    double v = a == c ? 1.0 : 0.0;
                    for (int l = a + 1; l <= c; ++l) v -= R[a][l] * Ri[l][c];
                    Ri[a][c] = v / R[a][a];
                }
            }
        ok = good;
        if (!good) *big = 1;
    }
    __syncthreads();
    if (!ok) return;
    for (int i = tid; i < d; i += blockDim.x) {
        double xr[kSmallCluster];
#pragma unroll
        for (int a = 0; a < kSmallCluster; ++a) xr[a] = a < g ? cols[a * d + i] : 0.0;
#pragma unroll
        for (int c = 0; c < kSmallCluster; ++c) {
            if (c >= g) break;
            double v = 0.0;
#pragma unroll
            for (int a = 0; a < kSmallCluster; ++a)
                if (a <= c) v = fma(xr[a], Ri[a][c], v);
            uc[static_cast<size_t>(c) * d + i] = v;
            if (out_rm) out_rm[static_cast<size_t>(i) * n_need + g0 + c] = v;
        }
    }
}

// One CTA per cluster g (gstart[g] .. gstart[g+1]): Cholesky of the cluster's
// diagonal block of the Gram U^T U (row-major n_need x n_need), written as the
// block R^{-1} of the block-diagonal m (zeroed by the caller), so U m has each
// cluster orthonormal; inter-cluster products are O(eps ||T|| / gap) and the
// Newton-Schulz steps that follow remove them.
__global__ void __launch_bounds__(1024) group_chol_kernel(int n_need, const double* __restrict__ gram,
                                                           const int* __restrict__ gstart,
                                                           const int* __restrict__ ngroups, double* __restrict__ m,
                                                           double* __restrict__ gwork, int* __restrict__ ginfo,
                                                           int smem_max_a, const int* __restrict__ run_if) {
    extern __shared__ double dyn_s[];
    const int b = blockIdx.x;
    if (run_if && *run_if == 0) return;
    if (b >= *ngroups) return;
    const int g0 = gstart[b], g = gstart[b + 1] - g0;
    const size_t o = static_cast<size_t>(g0) * n_need + g0;
    chol_drop_body(g, gram + o, n_need, nullptr, 0.0, m + o, n_need, ginfo + 4 * b,
                   gwork + static_cast<size_t>(g0) * n_need, smem_max_a, dyn_s);
}

// ------------------------------------------------------------------ 5. back-transformation
// z (row-major, ldz): z[:, c] = H_0 H_1 ... H_{d-3} u[:, c]; one warp per column.
__global__ void __launch_bounds__(128) backtr_kernel(int d, int n_need, const double* __restrict__ vref,
                                                      const double* __restrict__ tau, double* __restrict__ u,
                                                      double* __restrict__ z, int ldz) {
    const int lane = threadIdx.x & 31;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= n_need) return;
    double* x = u + static_cast<size_t>(c) * d;
    for (int k = d - 3; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const int m = d - k - 1;
        const double* vk = vref + static_cast<size_t>(k) * d;
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s = fma(vk[i], x[k + 1 + i], s);
        s = warp_sum(s) * t;
        for (int i = lane; i < m; i += 32) x[k + 1 + i] -= s * vk[i];
        __syncwarp();
    }
    for (int i = lane; i < d; i += 32) z[static_cast<size_t>(i) * ldz + c] = x[i];
}

// Register-resident variant (d <= 32*NPL): each warp keeps its eigenvector
// column in registers (NPL values per lane); the CTA stages KC reflectors at a
// time in shared memory, so every reflector is read from L2 once per CTA.
template <int NPL>
__global__ void __launch_bounds__(256) backtr_reg_kernel(int d, int n_need, const double* __restrict__ vref,
                                                          const double* __restrict__ tau,
                                                          const double* __restrict__ u, double* __restrict__ z,
                                                          int ldz) {
    constexpr int KC = 8;
    extern __shared__ double bsm[];  // KC x d reflector slab
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int c = blockIdx.x * nwb + wib;
    const bool live = c < n_need;
    double x[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int r = lane + 32 * q;
        x[q] = live && r < d ? u[static_cast<size_t>(c) * d + r] : 0.0;
    }
    for (int kk = d - 3; kk >= 0; kk -= KC) {
        const int k_lo = max(0, kk - KC + 1);
        // stage reflectors k_lo..kk: slot (kk - k) holds v_k[0 .. d-k-2]
        for (int e = threadIdx.x; e < KC * d; e += blockDim.x) {
            const int sidx = e / d, i = e - sidx * d;
            const int k = kk - sidx;
            if (k >= k_lo && i < d - k - 1) bsm[e] = vref[static_cast<size_t>(k) * d + i];
        }
        __syncthreads();
        if (live)
            for (int k = kk; k >= k_lo; --k) {
                const double t = tau[k];
                if (t == 0.0) continue;
                const double* vk = bsm + (kk - k) * d;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const int r = lane + 32 * q;
                    if (r > k && r < d) s = fma(vk[r - k - 1], x[q], s);
                }
                s = warp_sum(s) * t;
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const int r = lane + 32 * q;
                    if (r > k && r < d) x[q] = fma(-s, vk[r - k - 1], x[q]);
                }
            }
        __syncthreads();
    }
    if (live)
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int r = lane + 32 * q;
            if (r < d) z[static_cast<size_t>(r) * ldz + c] = x[q];
        }
}

// Variant without shared-memory staging: each warp streams the reflectors
// from L1/L2 itself (the CTA's warps share them through L1), prefetching
// reflector k-1 while applying k, so there is no CTA barrier on the chain.
template <int NPL>
__global__ void __launch_bounds__(256) backtr_g_kernel(int d, int n_need, const double* __restrict__ vref,
                                                        const double* __restrict__ tau,
                                                        const double* __restrict__ u, double* __restrict__ z,
                                                        int ldz) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int c = blockIdx.x * nwb + wib;
    if (c >= n_need) return;
    double x[NPL], vn[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int r = lane + 32 * q;
        x[q] = r < d ? u[static_cast<size_t>(c) * d + r] : 0.0;
    }
    auto load_v = [&](int k, double (&v)[NPL]) {
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int r = lane + 32 * q;
            v[q] = (k >= 0 && r > k && r < d) ? __ldg(vref + static_cast<size_t>(k) * d + (r - k - 1)) : 0.0;
        }
    };
    load_v(d - 3, vn);
    double tn = d >= 3 ? __ldg(tau + d - 3) : 0.0;
    for (int k = d - 3; k >= 0; --k) {
        double vc[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) vc[q] = vn[q];
        const double t = tn;
        load_v(k - 1, vn);
        tn = k > 0 ? __ldg(tau + k - 1) : 0.0;
        if (t == 0.0) continue;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NPL; ++q) s = fma(vc[q], x[q], s);
        s = warp_sum(s) * t;
#pragma unroll
        for (int q = 0; q < NPL; ++q) x[q] = fma(-s, vc[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int r = lane + 32 * q;
        if (r < d) z[static_cast<size_t>(r) * ldz + c] = x[q];
    }
}

// u (column-major d x k) -> row-major scratch, and back
__global__ void rm_to_cm_small(int d, int k, const double* __restrict__ rm, int ldr, double* __restrict__ cm,
                               const int* __restrict__ run_if = nullptr) {
    if (run_if && *run_if == 0) return;
    const int64_t total = static_cast<int64_t>(d) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(e / d), i = static_cast<int>(e % d);
        cm[e] = rm[static_cast<size_t>(i) * ldr + c];
    }
}

// ------------------------------------------------------------------ grid-cooperative path
// Real and complex Hermitian reduction over an L2-resident copy of H, for the
// projected problems too large for one cluster's shared memory (real d > ~640)
// and for every complex one (config 5: d up to 3*384 = 1152).  LAPACK
// zhetd2/zlarfg conventions: H_j = I - tau_j v_j v_j^H with v_j[0] = 1 and
// H_j^H x = beta e_1, beta REAL, so T = Q^H A Q is a real symmetric tridiagonal
// even for complex A and the real bisection / inverse iteration above apply
// unchanged; Z = Q U is complex.
//
// One grid.sync() per column: the rank-2 update of step j-1 is applied lazily
// inside step j's single pass over the trailing rows (each warp owns rows
// r = j+1+gw, gw + #warps, ...), which also accumulates p_j = tau_j A v_j.
// Every CTA rebuilds the reflector redundantly from row j (deterministic
// reductions, so all CTAs hold bit-identical v_j), P and the p^H v partials
// are double-buffered across steps.
__device__ __forceinline__ double re_(double a) { return a; }
__device__ __forceinline__ double re_(double2 a) { return a.x; }
__device__ __forceinline__ double im_(double) { return 0.0; }
__device__ __forceinline__ double im_(double2 a) { return a.y; }
__device__ __forceinline__ double cj(double a) { return a; }
__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 operator-(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 scal(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double scal(double s, double a) { return s * a; }
template <class E>
__device__ __forceinline__ E mk(double r, double i);
template <>
__device__ __forceinline__ double mk<double>(double r, double) { return r; }
template <>
__device__ __forceinline__ double2 mk<double2>(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ double wsum(double v) { return warp_sum(v); }
__device__ __forceinline__ double2 wsum(double2 v) { return make_double2(warp_sum(v.x), warp_sum(v.y)); }
__device__ __forceinline__ double abs2(double a) { return a * a; }
__device__ __forceinline__ double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
// 1 / z
__device__ __forceinline__ double inv_(double a) { return 1.0 / a; }
__device__ __forceinline__ double2 inv_(double2 a) {
    const double s = 1.0 / (a.x * a.x + a.y * a.y);
    return make_double2(a.x * s, -a.y * s);
}

constexpr int kCoopThreads = 512;

// A <- (H + H^H)/2, full storage (lda = d)
template <class E>
__global__ void sym_copy_kernel(int d, const E* __restrict__ h, int ldh, E* __restrict__ a) {
    const int total = d * d;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int i = e / d, j = e - i * d;
        const E x = h[static_cast<size_t>(i) * ldh + j], y = cj(h[static_cast<size_t>(j) * ldh + i]);
        a[e] = scal(0.5, x + y);
    }
}

template <class E>
__global__ void __launch_bounds__(kCoopThreads) tridiag_coop_kernel(int d, E* __restrict__ a, E* __restrict__ vref,
                                                                     E* __restrict__ tau, double* __restrict__ dg,
                                                                     double* __restrict__ off, E* __restrict__ pbuf,
                                                                     E* __restrict__ part) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ unsigned char coop_sm[];
    E* vprev = reinterpret_cast<E*>(coop_sm);
    E* wprev = vprev + d;
    E* vcur = wprev + d;
    __shared__ double red_d[kCoopThreads / 32];
    __shared__ E red_e[kCoopThreads / 32];
    __shared__ double s_diag;
    __shared__ E s_pv;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int gwarps = gridDim.x * nw, gw = blockIdx.x * nw + wid;
    bool hp = false;
    for (int j = 0; j + 1 < d; ++j) {
        const int buf = j & 1;
        // ---- A: row j (pending update applied), reflector of x = conj(row j)[j+1:]
        double xn2 = 0.0;
        for (int c = j + tid; c < d; c += blockDim.x) {
            E av = a[static_cast<size_t>(j) * d + c];
            if (hp) av = av - (mul(vprev[j], cj(wprev[c])) + mul(wprev[j], cj(vprev[c])));
            if (c == j) {
                s_diag = re_(av);
            } else {
                const E x = cj(av);
                vcur[c] = x;
                if (c >= j + 2) xn2 += abs2(x);
            }
        }
        xn2 = warp_sum(xn2);
        if (lane == 0) red_d[wid] = xn2;
        __syncthreads();
        xn2 = warp_sum(lane < nw ? red_d[lane] : 0.0);
        const E alpha = vcur[j + 1];
        E t = mk<E>(0.0, 0.0);
        double beta = re_(alpha);
        E sc = mk<E>(0.0, 0.0);
        const bool refl = !(xn2 == 0.0 && im_(alpha) == 0.0);
        if (refl) {
            const double ar = re_(alpha), ai = im_(alpha);
            beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
            t = mk<E>((beta - ar) / beta, -ai / beta);
            sc = inv_(alpha - mk<E>(beta, 0.0));
        }
        __syncthreads();  // every thread has read alpha before v overwrites vcur[j+1]
        for (int c = j + 1 + tid; c < d; c += blockDim.x) {
            const E v = c == j + 1 ? mk<E>(1.0, 0.0) : (refl ? mul(sc, vcur[c]) : mk<E>(0.0, 0.0));
            vcur[c] = v;
            if (blockIdx.x == 0) vref[static_cast<size_t>(j) * d + (c - j - 1)] = v;
        }
        if (blockIdx.x == 0 && tid == 0) {
            tau[j] = t;
            dg[j] = s_diag;
            off[j] = beta;
        }
        __syncthreads();
        // ---- B: owned trailing rows: apply update j-1, p_j = tau_j A v_j
        E pv = mk<E>(0.0, 0.0);
        for (int r = j + 1 + gw; r < d; r += gwarps) {
            E s = mk<E>(0.0, 0.0);
            E* row = a + static_cast<size_t>(r) * d;
            const E vr = hp ? vprev[r] : mk<E>(0.0, 0.0), wr = hp ? wprev[r] : mk<E>(0.0, 0.0);
            // 4 row elements per lane in flight: the pass is L2-latency bound
            // (a step's trailing block is spread over every warp of the grid)
            int c = j + 1 + lane;
            for (; c + 96 < d; c += 128) {
                E av[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) av[u] = row[c + 32 * u];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = c + 32 * u;
                    if (hp) {
                        av[u] = av[u] - (mul(vr, cj(wprev[cc])) + mul(wr, cj(vprev[cc])));
                        row[cc] = av[u];
                    }
                    s = s + mul(av[u], vcur[cc]);
                }
            }
            for (; c < d; c += 32) {
                E av = row[c];
                if (hp) {
                    av = av - (mul(vr, cj(wprev[c])) + mul(wr, cj(vprev[c])));
                    row[c] = av;
                }
                s = s + mul(av, vcur[c]);
            }
            s = wsum(s);
            const E p = mul(t, s);
            if (lane == 0) pbuf[static_cast<size_t>(buf) * d + r] = p;
            pv = pv + mul(cj(p), vcur[r]);
        }
        if (lane == 0) red_e[wid] = pv;
        __syncthreads();
        if (tid == 0) {
            E acc = mk<E>(0.0, 0.0);
            for (int w = 0; w < nw; ++w) acc = acc + red_e[w];
            part[static_cast<size_t>(buf) * gridDim.x + blockIdx.x] = acc;
        }
        grid.sync();
        // ---- C: w_j = p_j - (tau_j / 2)(p_j^H v_j) v_j
        if (wid == 0) {  // the grid's partials, lane-strided then a fixed shuffle tree
            E acc = mk<E>(0.0, 0.0);
            for (int g = lane; g < static_cast<int>(gridDim.x); g += 32)
                acc = acc + part[static_cast<size_t>(buf) * gridDim.x + g];
            acc = wsum(acc);
            if (lane == 0) s_pv = acc;
        }
        __syncthreads();
        const E aw = scal(-0.5, mul(t, s_pv));
        E* tmp = vprev;
        vprev = vcur;
        vcur = tmp;
        for (int c = j + 1 + tid; c < d; c += blockDim.x)
            wprev[c] = pbuf[static_cast<size_t>(buf) * d + c] + mul(aw, vprev[c]);
        hp = true;
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) {
        E av = a[static_cast<size_t>(d - 1) * d + d - 1];
        if (hp) av = av - (mul(vprev[d - 1], cj(wprev[d - 1])) + mul(wprev[d - 1], cj(vprev[d - 1])));
        dg[d - 1] = re_(av);
    }
}

// Z = Q U (U real, column-major d x n_need) applying H_{d-2} ... H_0; CB
// columns per CTA held in registers (R rows per thread), one CTA barrier per
// reflector; z row-major (ldz elements).
template <class E, int R>
__global__ void __launch_bounds__(256) backtr_cta_kernel(int d, int n_need, const E* __restrict__ vref,
                                                          const E* __restrict__ tau, const double* __restrict__ u,
                                                          E* __restrict__ z, int ldz) {
    constexpr int CB = 4;
    __shared__ E red[2][8][CB];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int col0 = blockIdx.x * CB;
    E x[CB][R];
#pragma unroll
    for (int c = 0; c < CB; ++c)
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int i = tid + 256 * q;
            x[c][q] = mk<E>(i < d && col0 + c < n_need ? u[static_cast<size_t>(col0 + c) * d + i] : 0.0, 0.0);
        }
    int b = 0;
    for (int j = d - 2; j >= 0; --j) {
        const E t = tau[j];
        if (re_(t) == 0.0 && im_(t) == 0.0) continue;
        const E* v = vref + static_cast<size_t>(j) * d - (j + 1);  // v[i] for i in [j+1, d)
        E vv[R];
        E s[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) s[c] = mk<E>(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int i = tid + 256 * q;
            vv[q] = i > j && i < d ? v[i] : mk<E>(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < CB; ++c) s[c] = s[c] + mul(cj(vv[q]), x[c][q]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            s[c] = wsum(s[c]);
            if (lane == 0) red[b][wid][c] = s[c];
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            E tot = mk<E>(0.0, 0.0);
            for (int w = 0; w < 8; ++w) tot = tot + red[b][w][c];
            s[c] = mul(t, tot);
        }
        b ^= 1;
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < CB; ++c) x[c][q] = x[c][q] - mul(vv[q], s[c]);
    }
#pragma unroll
    for (int c = 0; c < CB; ++c)
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int i = tid + 256 * q;
            if (i < d && col0 + c < n_need) z[static_cast<size_t>(i) * ldz + col0 + c] = x[c][q];
        }
}

struct SyevWs {
    double *a, *vref, *tau, *dg, *off, *e2, *u, *urm, *u2rm, *gram, *m, *chol, *scratch;
    int *gstart, *ngroups, *cinfo, *ginfo;
    double *za, *zv, *ztau, *zp, *zpart;  // grid-cooperative / complex path (interleaved complex)
};

size_t carve(SyevWs* w, void* base, int d) {
    const size_t dd = static_cast<size_t>(d) * d;
    char* p = static_cast<char*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* r = p ? p + off : nullptr;
        off += (bytes + 255) & ~size_t(255);
        return r;
    };
    SyevWs t{};
    t.a = reinterpret_cast<double*>(take(dd * 8));
    t.vref = reinterpret_cast<double*>(take(dd * 8));
    t.tau = reinterpret_cast<double*>(take(d * 8 + 8));
    t.dg = reinterpret_cast<double*>(take(d * 8 + 8));
    t.off = reinterpret_cast<double*>(take(d * 8 + 8));
    t.e2 = reinterpret_cast<double*>(take(d * 8 + 8));
    t.u = reinterpret_cast<double*>(take(dd * 8));
    t.urm = reinterpret_cast<double*>(take(dd * 8));
    t.u2rm = reinterpret_cast<double*>(take(dd * 8));
    t.gram = reinterpret_cast<double*>(take(dd * 8));
    t.m = reinterpret_cast<double*>(take(dd * 8));
    t.chol = reinterpret_cast<double*>(take(bk_chol_work_bytes(d)));
    t.scratch = reinterpret_cast<double*>(take(static_cast<size_t>(d) * (6 * d + 8) * 8));
    t.gstart = reinterpret_cast<int*>(take((d + 2) * 4));
    t.ngroups = reinterpret_cast<int*>(take(64));
    t.cinfo = reinterpret_cast<int*>(take(64));
    t.ginfo = reinterpret_cast<int*>(take(static_cast<size_t>(d) * 16 + 64));
    t.za = reinterpret_cast<double*>(take(2 * dd * 8));
    t.zv = reinterpret_cast<double*>(take(2 * dd * 8));
    t.ztau = reinterpret_cast<double*>(take(2 * static_cast<size_t>(d) * 8 + 16));
    t.zp = reinterpret_cast<double*>(take(4 * static_cast<size_t>(d) * 8 + 32));
    t.zpart = reinterpret_cast<double*>(take(4 * static_cast<size_t>(kSMs) * 8 + 32));
    const size_t gram_ws = bk_gram_work_bytes(d, d, d);
    double* gw = reinterpret_cast<double*>(take(gram_ws));
    (void)gw;
    if (w) *w = t;
    return off;
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" size_t bk_syev_tri_work_bytes(int d) { return carve(nullptr, nullptr, d > 0 ? d : 1); }

namespace bk {
namespace {
// eigenvalues (bisection) and orthonormal eigenvectors U (column-major d x
// n_need in w.u) of the tridiagonal T in (w.dg, w.off)
int tri_vectors(int d, int n_need, double* values, SyevWs& w, void* gram_work, void* stream) {
    const cudaStream_t s = as_stream(stream);
    // latency-bound chains: two warps per CTA so the n_need warps spread over the
    // SMs instead of queueing 8 to an SM (12 SMs busy at n_need = 96 before)
    // one CTA of 8 warps per eigenvalue (257-way multisection); BK_BISECT_W = 0
    // selects the warp-per-eigenvalue kernel, 4 a 129-way CTA (tuning runs)
    static const int bw = [] {
        const char* e = getenv("BK_BISECT_W");
        return e ? atoi(e) : 8;
    }();
    const size_t bsm = 2 * sizeof(double) * d;
    if (bw == 4)
        bisect_multi_kernel<4><<<n_need, 128, bsm, s>>>(d, w.dg, w.off, n_need, values);
    else if (bw == 8)
        bisect_multi_kernel<8><<<n_need, 256, bsm, s>>>(d, w.dg, w.off, n_need, values);
    else
        bisect_kernel<<<ceil_div(n_need * 32, 64), 64, bsm, s>>>(d, w.dg, w.off, n_need, values, w.e2);
    group_kernel<<<1, 32, 0, s>>>(n_need, values, w.dg, w.off, d, w.gstart, w.ngroups);
    const int* has_clusters = w.ngroups + 1;  // device flag: some cluster has several members
    // Schur complement in shared memory for clusters up to smax columns
    int smax = n_need < 160 ? n_need : 160;
    while (smax > 0 && static_cast<size_t>(smax) * smax + 4 * static_cast<size_t>(n_need) + 8 > 28800) --smax;
    const size_t gsm = sizeof(double) * (static_cast<size_t>(smax) * smax + 4 * static_cast<size_t>(n_need) + 8);
    BK_RET(BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(group_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   226 * 1024)));
    const size_t ism = sizeof(double) * (2 * static_cast<size_t>(d) + 2 * (5 * static_cast<size_t>(d) + (d + 7) / 8));
    BK_RET(BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(sizeof(double) * 14 * kSyevMaxD))));
    // clusters -> orthonormal blocks: Gram, per-cluster Cholesky (block-diagonal
    // R^{-1}), update; run_if: only when some cluster has several members
    auto cluster_step = [&](const int* run_if) -> int {  // w.urm (written by invit_kernel) -> w.u2rm
        int rc = run_if ? bk_gram_if_d(d, w.urm, n_need, n_need, w.urm, n_need, n_need, w.gram, n_need, gram_work,
                                       run_if, stream)
                        : bk_gram_d(d, w.urm, n_need, n_need, w.urm, n_need, n_need, w.gram, n_need, gram_work, stream);
        if (rc) return rc;
        BK_RET(cudaMemsetAsync(w.m, 0, sizeof(double) * n_need * n_need, s));
        group_chol_kernel<<<n_need, 1024, gsm, s>>>(n_need, w.gram, w.gstart, w.ngroups, w.m, w.scratch, w.ginfo,
                                                    smax, run_if);
        return run_if ? bk_gemm_if_d(d, w.urm, n_need, n_need, w.m, n_need, n_need, 1.0, 0.0, w.u2rm, n_need, run_if,
                                     stream)
                      : bk_gemm_d(d, w.urm, n_need, n_need, w.m, n_need, n_need, 1.0, 0.0, w.u2rm, n_need, stream);
    };
    // inverse iteration, two steps; the clusters of the first step's vectors are
    // orthonormalised before the second (see invit_kernel), skipped on the device
    // when every wanted eigenvalue is isolated
    int* big = w.ngroups + 2;  // device flag: the general cluster path is needed (set by group_kernel / the small kernel)
    const size_t csm = sizeof(double) * static_cast<size_t>(d) * kSmallCluster;
    BK_RET(BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(cluster_orth_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(sizeof(double) * kSyevMaxD * kSmallCluster))));
    invit_kernel<<<ceil_div(n_need * 32, 64), 64, ism, s>>>(d, w.dg, w.off, values, n_need, w.u, 1, 0, nullptr,
                                                            nullptr, w.urm);
    // clusters between the steps: small ones in place in w.u by one fused kernel; the
    // general path (w.urm -> w.u2rm) only when a cluster is large or a pivot was poor
    cluster_orth_small_kernel<<<n_need, 128, csm, s>>>(d, n_need, w.gstart, w.ngroups, w.u, nullptr, big, has_clusters);
    {
        const int rc = cluster_step(big);
        if (rc) return rc;
    }
    invit_kernel<<<ceil_div(n_need * 32, 64), 64, ism, s>>>(d, w.dg, w.off, values, n_need, w.u, 1, 1, w.u2rm, big,
                                                            w.urm);
    cluster_orth_small_kernel<<<n_need, 128, csm, s>>>(d, n_need, w.gstart, w.ngroups, w.u, w.u2rm, big, nullptr);
    {
        const int rc = cluster_step(big);
        if (rc) return rc;
    }
    // three Newton-Schulz steps U <- U (3I - U^T U)/2: after the cluster step the
    // columns are orthonormal to O(eps ||T|| / gap) (gap >= 1e-7 ||T|| between
    // clusters) and a cluster's members to eps cond(G_cluster); the error squares
    // per step (0.02 -> 3e-4 -> 7e-8 -> 4e-15) — GEMM-only
    for (int pass = 0; pass < 3; ++pass) {
        double* src = pass == 1 ? w.urm : w.u2rm;
        double* dst = pass == 1 ? w.u2rm : w.urm;
        int rc = bk_gram_d(d, src, n_need, n_need, src, n_need, n_need, w.gram, n_need, gram_work, stream);
        if (rc) return rc;
        rc = bk_ns_coeff_d(n_need, w.gram, n_need, w.m, n_need, stream);
        if (rc) return rc;
        rc = bk_gemm_d(d, src, n_need, n_need, w.m, n_need, n_need, 1.0, 0.0, dst, n_need, stream);
        if (rc) return rc;
    }
    rm_to_cm_small<<<ceil_div(d * n_need, 256), 256, 0, s>>>(d, n_need, w.urm, n_need, w.u);
    BK_LAUNCHED();
}

// grid-cooperative tridiagonalisation (E = double or double2) of the sym/Hermitian
// part of h into w.dg, w.off and reflectors (w.zv, w.ztau)
template <class E>
int coop_tridiag(int d, const double* h, int ldh, SyevWs& w, cudaStream_t s) {
    sym_copy_kernel<E><<<max(1, min(ceil_div(d * d, 256), 8 * kSMs)), 256, 0, s>>>(
        d, reinterpret_cast<const E*>(h), ldh, reinterpret_cast<E*>(w.za));
    const size_t smem = 3 * static_cast<size_t>(d) * sizeof(E);
    const cudaError_t attr = BK_ONCE_PER_DEVICE(prep_smem(tridiag_coop_kernel<E>, 3 * sizeof(E) * kSyevMaxD));
    BK_RET(attr);
    static int per_sm_dev[kMaxDevices];  // occupancy is per device
    int dev = 0;
    BK_RET(cudaGetDevice(&dev));
    dev = dev < kMaxDevices ? dev : 0;
    BK_RET(BK_ONCE_PER_DEVICE(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm_dev[dev], tridiag_coop_kernel<E>, kCoopThreads, 3 * sizeof(E) * kSyevMaxD)));
    const int per_sm = per_sm_dev[dev];
    if (per_sm < 1) return static_cast<int>(cudaErrorLaunchOutOfResources);
    int grid = max(1, min(ceil_div(d, kCoopThreads / 32), kSMs));
    grid = min(grid, per_sm * kSMs);
    int dd = d;
    E* a = reinterpret_cast<E*>(w.za);
    E* v = reinterpret_cast<E*>(w.zv);
    E* t = reinterpret_cast<E*>(w.ztau);
    E* pb = reinterpret_cast<E*>(w.zp);
    E* pt = reinterpret_cast<E*>(w.zpart);
    double* dg = w.dg;
    double* off = w.off;
    void* args[] = {&dd, &a, &v, &t, &dg, &off, &pb, &pt};
    BK_RET(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tridiag_coop_kernel<E>), dim3(grid),
                                       dim3(kCoopThreads), args, smem, s));
    return 0;
}

template <class E>
int backtr_cta(int d, int n_need, const SyevWs& w, E* z, int ldz, cudaStream_t s) {
    const int blocks = ceil_div(n_need, 4);
    const E* v = reinterpret_cast<const E*>(w.zv);
    const E* t = reinterpret_cast<const E*>(w.ztau);
    if (d <= 256)
        backtr_cta_kernel<E, 1><<<blocks, 256, 0, s>>>(d, n_need, v, t, w.u, z, ldz);
    else if (d <= 512)
        backtr_cta_kernel<E, 2><<<blocks, 256, 0, s>>>(d, n_need, v, t, w.u, z, ldz);
    else if (d <= 768)
        backtr_cta_kernel<E, 3><<<blocks, 256, 0, s>>>(d, n_need, v, t, w.u, z, ldz);
    else if (d <= 1024)
        backtr_cta_kernel<E, 4><<<blocks, 256, 0, s>>>(d, n_need, v, t, w.u, z, ldz);
    else
        backtr_cta_kernel<E, 5><<<blocks, 256, 0, s>>>(d, n_need, v, t, w.u, z, ldz);
    BK_LAUNCHED();
}
}  // namespace
}  // namespace bk

extern "C" int bk_syev_tri_d(int d, const double* h, int ldh, int n_need, double* values, double* z, int ldz,
                             void* work, int* info, void* stream) {
    if (d <= 0) return 0;
    if (n_need <= 0 || n_need > d) n_need = d;
    const cudaStream_t s = as_stream(stream);
    SyevWs w;
    const size_t total = carve(&w, work, d);
    void* gram_work = static_cast<char*>(work) + total - ((bk_gram_work_bytes(d, d, d) + 255) & ~size_t(255));
    const int mm = d < kTriSmemMaxM + 1 ? d : kTriSmemMaxM + 1;
    const size_t smem = sizeof(double) * (4 * static_cast<size_t>(d) + static_cast<size_t>(mm) * mm);
    const cudaError_t attr = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(
        tridiag_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(sizeof(double) * (4 * kSyevMaxD + (kTriSmemMaxM + 1) * (kTriSmemMaxM + 1)))));
    BK_RET(attr);
    if (d > kSyevMaxD) return static_cast<int>(cudaErrorInvalidValue);
    if (d == 1) {
        // 1x1: value and unit vector
        BK_RET(cudaMemcpyAsync(values, h, sizeof(double), cudaMemcpyDeviceToDevice, s));
        const double one = 1.0;
        BK_RET(cudaMemcpyAsync(z, &one, sizeof(double), cudaMemcpyHostToDevice, s));
        BK_RET(cudaMemsetAsync(info, 0, 2 * sizeof(int), s));
        return 0;
    }
    size_t csmem = 0;
    const int C = tridiag_cluster_size(d, &csmem);
    bool launched = false;
    static const bool force_coop = getenv("BK_SYEV_COOP") != nullptr;  // tuning runs only
    static const bool no_packed = getenv("BK_TRI_NO_PACKED") != nullptr;  // tuning runs only
    static const bool no_small_packed = getenv("BK_TRI_NO_SMALL_PACKED") != nullptr;  // A/B runs
    if (d <= 65 && !force_coop && !no_packed && !no_small_packed) {
        // small projected problems (config 1's SI, d <= 40): 4 warps of <= 16 rows
        // and 2 column chunks — a 16-warp CTA's barriers cost more than the work
        auto kern = tridiag_packed_kernel<128, 2, 16>;
        const cudaError_t ap = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(
            kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(packed_smem_bytes(65))));
        BK_RET(ap);
        kern<<<1, 128, packed_smem_bytes(d), s>>>(d, h, ldh, w.vref, w.tau, w.dg, w.off);
        BK_RET(cudaGetLastError());
        launched = true;
    }
    if (!launched && d <= kPackedUseMaxD && !force_coop && !no_packed) {
        auto kern = tridiag_packed_kernel<kPkThreads, kPkM, kPkR>;
        const cudaError_t ap = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(kern,
                                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            static_cast<int>(packed_smem_bytes(kPackedMaxD))));
        BK_RET(ap);
        kern<<<1, kPkThreads, packed_smem_bytes(d), s>>>(d, h, ldh, w.vref, w.tau, w.dg, w.off);
        BK_RET(cudaGetLastError());
        launched = true;
    }
    if (!launched && C > 0 && !force_coop) {
        // CTA size of the cluster kernel: 256 threads (fewer warps repeat the
        // replicated reflector / reduction work; syev d = 207 1076 -> 1009 us,
        // d = 288 1563 -> 1508 us); BK_TRI_THREADS = 128 / 512 for tuning runs
        static const int tthreads = [] {
            const char* e = getenv("BK_TRI_THREADS");
            const int v = e ? atoi(e) : 256;
            return v == 128 || v == 512 ? v : 256;
        }();
        // one cluster barrier per step (BK_TRI_2BAR: the two-barrier kernel, tuning runs)
        static const bool two_bar = getenv("BK_TRI_2BAR") != nullptr;
        auto kern = two_bar ? (tthreads == 256   ? tridiag_cluster_kernel<256>
                               : tthreads == 128 ? tridiag_cluster_kernel<128>
                                                 : tridiag_cluster_kernel<kClThreads>)
                            : (tthreads == 256   ? tridiag_cluster1_kernel<256>
                               : tthreads == 128 ? tridiag_cluster1_kernel<128>
                                                 : tridiag_cluster1_kernel<kClThreads>);
        const cudaError_t a1 = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            200 * 1024 + 8192));
        const cudaError_t a2 = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        BK_RET(a1);
        BK_RET(a2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C, 1, 1);
        cfg.blockDim = dim3(tthreads, 1, 1);
        cfg.dynamicSmemBytes = csmem;
        cfg.stream = s;
        cudaLaunchAttribute attr_c[1];
        attr_c[0].id = cudaLaunchAttributeClusterDimension;
        attr_c[0].val.clusterDim.x = C;
        attr_c[0].val.clusterDim.y = 1;
        attr_c[0].val.clusterDim.z = 1;
        cfg.attrs = attr_c;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, d, h, ldh, w.vref, w.tau, w.dg, w.off);
        if (e == cudaSuccess) launched = true;
        else (void)cudaGetLastError();  // cluster not schedulable: fall back below
    }
    bool coop = false;
    if (!launched) {
        if (d > 256 || force_coop) {
            // large d: the grid-cooperative reduction (one grid sync per column)
            const int rc = coop_tridiag<double>(d, h, ldh, w, s);
            if (rc) return rc;
            coop = true;
        } else {
            tridiag_fused_kernel<<<1, kTriThreads, smem, s>>>(d, h, ldh, w.a, w.vref, w.tau, w.dg, w.off);
        }
    }
    {
        const int rc = tri_vectors(d, n_need, values, w, gram_work, stream);
        if (rc) return rc;
    }
    if (coop) {
        const int rc = backtr_cta<double>(d, n_need, w, z, ldz, s);
        if (rc) return rc;
    } else {
        const size_t bs = sizeof(double) * 8 * static_cast<size_t>(d);
        const int blocks = ceil_div(n_need, 8);
        const cudaError_t ab4 = BK_ONCE_PER_DEVICE(prep_smem(backtr_reg_kernel<4>, sizeof(double) * 8 * kSyevMaxD));
        const cudaError_t ab8 = BK_ONCE_PER_DEVICE(prep_smem(backtr_reg_kernel<8>, sizeof(double) * 8 * kSyevMaxD));
        const cudaError_t ab12 = BK_ONCE_PER_DEVICE(prep_smem(backtr_reg_kernel<12>, sizeof(double) * 8 * kSyevMaxD));
        const cudaError_t ab16 = BK_ONCE_PER_DEVICE(prep_smem(backtr_reg_kernel<16>, sizeof(double) * 8 * kSyevMaxD));
        BK_RET(ab4);
        BK_RET(ab8);
        BK_RET(ab12);
        BK_RET(ab16);
        // streaming variant (no staging barrier): d = 288 syev 1.89 -> 1.79 ms.
        // BK_BACKTR_STAGED=1 selects the staged kernel, BK_BACKTR_WARPS the warps
        // (columns) per CTA (tuning runs)
        static const bool staged = getenv("BK_BACKTR_STAGED") != nullptr;
        static const int bw = [] {
            const char* e = getenv("BK_BACKTR_WARPS");
            return e ? max(1, min(8, atoi(e))) : 2;
        }();
        const int gblocks = ceil_div(n_need, bw);
        if (!staged && d <= 512) {
            if (d <= 128)
                backtr_g_kernel<4><<<gblocks, 32 * bw, 0, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
            else if (d <= 256)
                backtr_g_kernel<8><<<gblocks, 32 * bw, 0, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
            else if (d <= 384)
                backtr_g_kernel<12><<<gblocks, 32 * bw, 0, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
            else
                backtr_g_kernel<16><<<gblocks, 32 * bw, 0, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
        } else if (d <= 128)
            backtr_reg_kernel<4><<<blocks, 256, bs, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
        else if (d <= 256)
            backtr_reg_kernel<8><<<blocks, 256, bs, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
        else if (d <= 384)
            backtr_reg_kernel<12><<<blocks, 256, bs, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
        else if (d <= 512)
            backtr_reg_kernel<16><<<blocks, 256, bs, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
        else
            backtr_kernel<<<ceil_div(n_need * 32, 128), 128, 0, s>>>(d, n_need, w.vref, w.tau, w.u, z, ldz);
    }
    BK_RET(cudaMemsetAsync(info, 0, 2 * sizeof(int), s));
    BK_LAUNCHED();
}

// Complex Hermitian projected problem (config 5): h, z interleaved complex
// row-major (ldh, ldz in complex elements); values real ascending.
extern "C" size_t bk_syev_z_work_bytes(int d) { return carve(nullptr, nullptr, d > 0 ? d : 1); }

extern "C" int bk_syev_z(int d, const double* h, int ldh, int n_need, double* values, double* z, int ldz, void* work,
                         int* info, void* stream) {
    if (d <= 0) return 0;
    if (d > kSyevMaxD) return static_cast<int>(cudaErrorInvalidValue);
    if (n_need <= 0 || n_need > d) n_need = d;
    const cudaStream_t s = as_stream(stream);
    SyevWs w;
    const size_t total = carve(&w, work, d);
    void* gram_work = static_cast<char*>(work) + total - ((bk_gram_work_bytes(d, d, d) + 255) & ~size_t(255));
    if (d == 1) {
        // 1x1: value = Re h, vector = 1
        const double zero_one[2] = {1.0, 0.0};
        BK_RET(cudaMemcpyAsync(values, h, sizeof(double), cudaMemcpyDeviceToDevice, s));
        BK_RET(cudaMemcpyAsync(z, zero_one, 2 * sizeof(double), cudaMemcpyHostToDevice, s));
        BK_RET(cudaMemsetAsync(info, 0, 2 * sizeof(int), s));
        return 0;
    }
    int rc = coop_tridiag<double2>(d, h, ldh, w, s);
    if (rc) return rc;
    rc = tri_vectors(d, n_need, values, w, gram_work, stream);
    if (rc) return rc;
    rc = backtr_cta<double2>(d, n_need, w, reinterpret_cast<double2*>(z), ldz, s);
    if (rc) return rc;
    BK_RET(cudaMemsetAsync(info, 0, 2 * sizeof(int), s));
    BK_LAUNCHED();
}

// Dispatch: tridiagonalisation + bisection + inverse iteration; the one-CTA
// cyclic Jacobi (bk_small.cu) only on request (BK_SYEV_JACOBI_MAX).
extern "C" size_t bk_syev_work_bytes(int d) {
    const size_t a = bk_syev_jacobi_work_bytes(d), b = bk_syev_tri_work_bytes(d);
    return a > b ? a : b;
}

extern "C" int bk_syev_d(int d, double* h, int ldh, int n_need, double* values, double* z, int ldz, void* work,
                         int* info, void* stream) {
    static const int jmax = [] {  // BK_SYEV_JACOBI_MAX: Jacobi/tridiagonal switch (tuning runs)
        const char* e = getenv("BK_SYEV_JACOBI_MAX");
        return e ? atoi(e) : kSyevJacobiMaxD;
    }();
    if (d <= jmax) return bk_syev_jacobi_d(d, h, ldh, values, z, ldz, work, info, stream);
    return bk_syev_tri_d(d, h, ldh, n_need, values, z, ldz, work, info, stream);
}
