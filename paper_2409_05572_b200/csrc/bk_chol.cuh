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

// indexable view of the extern shared array: S[i] stays in the shared window
struct SmemRef {
    double* base;
    __device__ __forceinline__ double& operator[](int i) const { return base[i]; }
};

// one-CTA launch of the routine below (bk_small.cu); pairs: see above
// cond (optional, 2 ints): [0] = 1 when some kept pivot lost more than kCondFused
// of its projected norm squared (g_jj / p_j > kCondFused: the block is
// ill-conditioned, so the caller orthonormalises the tall product explicitly),
// [1] = 1 when a nonempty block is well-conditioned; predicates of bk_*_if_*
int chol_launch(int a, const double* g, int ldg, const double* ref2, double drop, double* m, int ldm, int* info,
                void* work, cudaStream_t st, bool pairs, int* cond = nullptr);
constexpr double kCondFused = 1e3;

// Shared-memory layout (dyn_s): gd[a] thr2[a] piv[a] slot[a] (ints) | S (a x a, a <= smem_max_a).
// S holds the Schur complement in its upper triangle and, in its strict lower
// triangle, the unit-lower elimination matrix E (E G = D L^T), so R^{-1} =
// E^T D^{-1/2} comes out of the same sweep: no separate triangular inversion
// (whose per-column warp walks cost half the kernel).  One barrier per pivot;
// the keep decision of pivot j+1 is taken by thread 0 right after its warp
// (warp 0, which owns row j+1 alone) has updated S[j+1][j+1], and published
// through shared memory — the other warps never run the decision logic.
template <class Ptr>
__device__ __forceinline__ void chol_drop_core(int a, const double* __restrict__ g, int ldg,
                                               const double* __restrict__ ref2, double drop,
                                               double* __restrict__ m, int ldm, int* __restrict__ info, Ptr S,
                                               double* gd, double* thr2, double* piv, int* slot, bool pairs,
                                               int* __restrict__ cond = nullptr) {
    __shared__ int s_keep[2];
    __shared__ double s_invp[2];
    __shared__ int s_kept, s_flags;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    for (int e = tid; e < a * a; e += nt) {
        const int k = e / a, l = e - k * a;
        S[e] = l >= k ? g[static_cast<size_t>(k) * ldg + l] : 0.0;
    }
    const double drop2 = drop * drop;
    for (int j = tid; j < a; j += nt) {
        const double d = g[static_cast<size_t>(j) * ldg + j];
        gd[j] = d;
        // thr2 < 0: no reference norm (pass 2 of CholQR2); +inf: certain drop
        double t = -1.0;
        if (ref2) {
            const double r = ref2[j], t2 = drop2 * r;
            t = (r == 0.0 || d < t2) ? INFINITY : t2;
        }
        thr2[j] = t;
    }
    __syncthreads();
    constexpr double kLo2 = (1.0 - 1e-4) * (1.0 - 1e-4), kHi2 = (1.0 + 1e-4) * (1.0 + 1e-4);
    // thread 0's running state: decisions, flags, kept count
    int kept = 0, flags = 0;  // flags: 1 unsure, 2 bad
    double worst = 0.0;       // max g_jj / p_j over kept pivots (cond)
    auto decide = [&](int j, double p) {
        const double gjj = gd[j], t2 = thr2[j];
        int keep;
        if (!isfinite(p) || !isfinite(gjj)) {
            flags |= 2;
            keep = 0;
        } else if (pairs && (j & 1)) {
            // real embedding of a complex Gram: index 2c+1 is the imaginary twin
            // of 2c (same pivot in exact arithmetic) and follows its decision
            keep = slot[j - 1] >= 0 && p > 0.0;
            if ((slot[j - 1] >= 0) != (p > 0.0)) flags |= 1;
        } else if (t2 < 0.0) {
            keep = p > 0.0;
            if (p <= 1e-8 * gjj) flags |= 1;  // pass 2 of CholQR2: basis lost rank
        } else if (t2 == INFINITY) {
            keep = 0;  // certain: the pivot can never exceed the projected norm
        } else {
            // squared form of "remaining norm >= drop * original norm"; the
            // uncertainty band |sqrt(p) - thr| < 1e-4 thr in squared form
            keep = p >= t2;
            if (p < 1e-8 * gjj || (p > kLo2 * t2 && p < kHi2 * t2)) flags |= 1;
        }
        slot[j] = keep ? kept : -1;
        piv[j] = p;
        kept += keep;
        if (keep) worst = fmax(worst, gjj / p);
        s_keep[j & 1] = keep;
        s_invp[j & 1] = keep ? __drcp_rn(p) : 0.0;  // reciprocal without the division routine
    };
    if (tid == 0) decide(0, S[0]);
    __syncthreads();
    for (int j = 0; j < a; ++j) {
        const int par = j & 1;
        if (s_keep[par]) {
            const double invp = s_invp[par];
            const int e_len = j + 1;  // E part of a row: l in [0, j]
            // warp 0: row j+1 alone (its diagonal is the next pivot); other warps: rows j+2..
            // (a single warp takes every row)
            const int k_begin = j + 1 + wid;
            const int k_step = nw == 1 ? 1 : (wid == 0 ? a : nw - 1);
            for (int k = k_begin; k < a; k += k_step) {
                const double f = S[j * a + k] * invp;
                const int up = a - k;  // Schur part: l in [k, a)
                for (int q = lane; q < up + e_len; q += 32) {
                    if (q < up) {
                        const int l = k + q;
                        S[k * a + l] -= f * S[j * a + l];
                    } else {
                        const int l = q - up;
                        S[k * a + l] = l == j ? -f : S[k * a + l] - f * S[j * a + l];
                    }
                }
            }
        }
        if (tid == 0 && j + 1 < a) decide(j + 1, S[(j + 1) * a + j + 1]);
        __syncthreads();
    }
    if (tid == 0) {
        s_kept = kept;
        s_flags = flags;
    }
    // slot^{-1} (column of M -> original index), reusing gd
    int* inv = reinterpret_cast<int*>(gd);
    for (int j = tid; j < a; j += nt)
        if (slot[j] >= 0) inv[slot[j]] = j;
    __syncthreads();
    // M[i][slot[c]] = E[c][i] / sqrt(p_c) for kept i <= c (E[c][c] = 1); zero elsewhere
    const int nk = s_kept;
    for (int e = tid; e < a * a; e += nt) {
        const int i = e / a, col = e - i * a;
        double v = 0.0;
        if (col < nk && slot[i] >= 0) {
            const int c = inv[col];
            if (i <= c) v = (i == c ? 1.0 : S[c * a + i]) / sqrt(piv[c]);
        }
        m[static_cast<size_t>(i) * ldm + col] = v;
    }
    if (tid == 0) {
        info[0] = nk;
        info[1] = s_flags & 1;
        info[2] = (s_flags >> 1) & 1;
        if (cond) {
            const int ill = nk > 0 && !(worst <= kCondFused);
            cond[0] = ill;
            cond[1] = nk > 0 && !ill;
        }
    }
}

__device__ __forceinline__ void chol_drop_body(int a, const double* __restrict__ g, int ldg,
                                               const double* __restrict__ ref2, double drop,
                                               double* __restrict__ m, int ldm, int* __restrict__ info,
                                               double* __restrict__ s, int smem_max_a, double* dyn_s,
                                               bool pairs = false, int* __restrict__ cond = nullptr) {
    double* gd = dyn_s;
    double* thr2 = dyn_s + a;
    double* piv = dyn_s + 2 * a;
    int* slot = reinterpret_cast<int*>(dyn_s + 3 * a);
    if (a <= smem_max_a) {
        // the Schur complement in shared memory: the specialised instantiation
        // keeps every access an LDS/STS (a generic pointer compiles to LD/ST)
        extern __shared__ double chol_smem[];
        SmemRef S{chol_smem + 3 * a + (a + 1) / 2};
        chol_drop_core(a, g, ldg, ref2, drop, m, ldm, info, S, gd, thr2, piv, slot, pairs, cond);
    } else {
        chol_drop_core(a, g, ldg, ref2, drop, m, ldm, info, s, gd, thr2, piv, slot, pairs, cond);
    }
}

}  // namespace bk
