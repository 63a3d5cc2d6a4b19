// Skip-pivot Cholesky with the CGS2 drop rule, as a CTA-wide device routine
// shared by K4 (bk_small.cu: one CTA per projected block) and K5 (bk_syev.cu:
// one CTA per eigenvalue cluster when orthonormalising inverse-iteration
// vectors).  See bk_small.cu for the algorithm and its reference mapping
// (proj/src/kernel.cpp:65-89).
//
// pairs: g is the real 2c x 2c embedding of a complex Hermitian Gram (bk_complex.cu);
// odd indices follow the decision of their even twin.
// dyn_s: dynamic shared memory of (3a + (a+1)/2) doubles, plus a*a doubles when
// a <= smem_max_a (the Schur complement then lives in shared memory; otherwise
// in the global scratch s, a*a doubles).
#pragma once
#include "bk_common.cuh"

namespace bk {

// one-CTA launch of the routine below (bk_small.cu); pairs: see above
int chol_launch(int a, const double* g, int ldg, const double* ref2, double drop, double* m, int ldm, int* info,
                void* work, cudaStream_t st, bool pairs);

__device__ __forceinline__ void chol_drop_body(int a, const double* __restrict__ g, int ldg,
                                               const double* __restrict__ ref2, double drop,
                                               double* __restrict__ m, int ldm, int* __restrict__ info,
                                               double* __restrict__ s, int smem_max_a, double* dyn_s,
                                               bool pairs = false) {
    __shared__ int s_unsure, s_bad;
    __shared__ double s_recip[2];  // 1 / next pivot, computed by thread 0 during the previous step
    __shared__ int s_recip_ok[2];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    // shared layout: gd[a] r2[a] piv[a] slot[a] (ints) | Schur complement s (a <= kCholSmemMaxA)
    double* gd = dyn_s;
    double* r2 = dyn_s + a;
    double* piv = dyn_s + 2 * a;
    int* slot = reinterpret_cast<int*>(dyn_s + 3 * a);
    if (a <= smem_max_a) s = dyn_s + 3 * a + (a + 1) / 2;  // working Schur complement in shared memory
    for (int e = tid; e < a * a; e += nt) s[e] = g[static_cast<size_t>(e / a) * ldg + e % a];
    for (int j = tid; j < a; j += nt) {
        gd[j] = g[static_cast<size_t>(j) * ldg + j];
        r2[j] = ref2 ? ref2[j] : 0.0;
    }
    if (tid == 0) {
        s_unsure = 0;
        s_bad = 0;
        s_recip_ok[0] = s_recip_ok[1] = 0;
    }
    __syncthreads();
    const double drop2 = drop * drop;
    constexpr double kLo2 = (1.0 - 1e-4) * (1.0 - 1e-4), kHi2 = (1.0 + 1e-4) * (1.0 + 1e-4);
    // right-looking skip-pivot Cholesky with ONE barrier per pivot: every thread
    // evaluates the (identical) keep decision itself; row j stays unscaled
    // during the step and R is formed in a final pass.
    int kept = 0;
    for (int j = 0; j < a; ++j) {
        const double p = s[j * a + j];
        const double gjj = gd[j];
        int keep;
        bool unsure = false, bad = false;
        if (!isfinite(p) || !isfinite(gjj)) {
            bad = true;
            keep = 0;
        } else if (pairs && (j & 1)) {
            // real embedding of a complex Gram: index 2c+1 is the imaginary twin
            // of 2c (same pivot in exact arithmetic) and follows its decision
            keep = slot[j - 1] >= 0 && p > 0.0;
            unsure = (slot[j - 1] >= 0) != (p > 0.0);
        } else if (ref2 == nullptr) {
            keep = p > 0.0;
            unsure = p <= 1e-8 * gjj;  // pass 2 of CholQR2: basis lost rank
        } else {
            // squared form of "remaining norm >= drop * original norm" (no sqrt on
            // the sequential path); the uncertainty band |sqrt(p) - thr| < 1e-4 thr
            // becomes p in ((1-1e-4)^2 thr^2, (1+1e-4)^2 thr^2)
            const double thr2 = drop2 * r2[j];
            if (r2[j] == 0.0 || gjj < thr2) {
                keep = 0;  // certain: the pivot can never exceed the projected norm
            } else {
                keep = p >= thr2;
                unsure = p < 1e-8 * gjj || (p > kLo2 * thr2 && p < kHi2 * thr2);
            }
        }
        const int par = j & 1;
        const double invp = keep ? (s_recip_ok[par] ? s_recip[par] : 1.0 / p) : 0.0;
        __syncwarp();
        if (tid == 0) {
            if (unsure) s_unsure = 1;
            if (bad) s_bad = 1;
            slot[j] = keep ? kept : -1;
            piv[j] = p;
            s_recip_ok[par ^ 1] = 0;
        }
        if (keep) {
            ++kept;
            for (int k = j + 1 + wid; k < a; k += nw) {
                const double rk = s[j * a + k] * invp;
                for (int l = k + lane; l < a; l += 32) s[k * a + l] -= rk * s[j * a + l];
                // thread 0 owns the next pivot s[j+1][j+1] (first row of warp 0,
                // first element of lane 0): its reciprocal, off the other warps' path
                if (tid == 0 && k == j + 1) {
                    s_recip[par ^ 1] = 1.0 / s[k * a + k];
                    s_recip_ok[par ^ 1] = 1;
                }
            }
        }
        __syncthreads();
    }
    // R rows: R[j][l] = s[j][l] / sqrt(p_j), R[j][j] = sqrt(p_j)
    for (int e = tid; e < a * a; e += nt) {
        const int j = e / a, l = e % a;
        if (l < j || slot[j] < 0) continue;
        const double rj = sqrt(piv[j]);
        s[e] = l == j ? rj : s[e] / rj;
    }
    __syncthreads();
    // R^{-1} = M (upper triangular over the kept indices), computed row by row
    // from the bottom: for each kept i (descending, one barrier per row) all
    // kept c > i in parallel:  M[i][c] = -(sum_{i<l<=c} R[i][l] M[l][c]) / R[i][i].
    // R lives in the upper triangle of s; M is stored transposed in the strict
    // lower triangle (M[l][c] at s[c*a + l]) and its diagonal in m's diagonal
    // slot, so both stay in shared memory.
    // dropped indices hold no R entries: zero their row of R (upper part) so the
    // dot products below need no per-element test
    for (int e = tid; e < a * a; e += nt) {
        const int j = e / a, l = e % a;
        if (l > j && (slot[j] < 0 || slot[l] < 0)) s[e] = 0.0;
    }
    __syncthreads();
    // 1/R[i][i] once (piv[] no longer needed)
    for (int i = tid; i < a; i += nt) piv[i] = slot[i] >= 0 ? 1.0 / s[i * a + i] : 0.0;
    __syncthreads();
    // Column c of M depends only on itself: one warp per column walks i
    // downward (lanes split each dot product), no CTA barrier needed.
    for (int c = wid; c < a; c += nw) {
        if (slot[c] < 0) continue;
        for (int i = c - 1; i >= 0; --i) {
            if (slot[i] < 0) continue;
            double acc = 0.0;
            for (int l = i + 1 + lane; l < c; l += 32) acc = fma(s[i * a + l], s[c * a + l], acc);
            acc = warp_sum(acc);
            if (lane == 0) s[c * a + i] = -(acc + s[i * a + c] * piv[c]) * piv[i];  // M[i][c]
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = tid; e < a * a; e += nt) {
        const int j = e / a, c = e % a;  // output row j (original column), column c (slot)
        m[static_cast<size_t>(j) * ldm + c] = 0.0;
    }
    __syncthreads();
    for (int e = tid; e < a * a; e += nt) {
        const int i = e / a, c = e % a;  // M[i][c], original indices i <= c
        if (i > c || slot[i] < 0 || slot[c] < 0) continue;
        const double val = i == c ? piv[c] : s[c * a + i];
        m[static_cast<size_t>(i) * ldm + slot[c]] = val;
    }
    if (tid == 0) {
        info[0] = kept;
        info[1] = s_unsure;
        info[2] = s_bad;
    }
}

}  // namespace bk
