// K4 (Cholesky with the CGS2 drop rule) and K5 (projected eigenproblem) —
// single-CTA kernels on the small dense side of the iteration.
//
// K4: the reference orthonormalises column by column with classical
// Gram-Schmidt applied twice and drops a column whose remaining norm is below
// 1e-8 of its original norm (proj/src/kernel.cpp:65-89).  Here the block is
// projected against the external basis with two K2/K3 passes and then
// orthonormalised by CholQR2; the keep/drop decision is the Cholesky pivot of
// the column against the columns kept before it, which in exact arithmetic is
// the same remaining norm CGS2 measures.  Pivots computed with heavy
// cancellation (remaining norm < 1e-4 of the projected norm) are reported as
// uncertain and the caller redoes that block with exact column CGS2.
//
// K5: eigendecomposition of 0.5(H + H^T) (sym_eig_small, kernel.cpp:95-100) by
// two-sided cyclic Jacobi in round-robin parallel order: every round rotates
// d/2 disjoint pairs at once, each 2x2 block of H is updated by one thread
// (rows and columns in one pass), and V accumulates the rotations.  H lives in
// shared memory up to d = 160 and in global memory (L2-resident) above.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>

#include "bk_chol.cuh"

namespace bk {
namespace {

// ------------------------------------------------------------------ K4
constexpr int kCholSmemMaxA = 160;

__global__ void __launch_bounds__(1024) chol_drop_kernel(int a, const double* __restrict__ g, int ldg,
                                                          const double* __restrict__ ref2, double drop,
                                                          double* __restrict__ m, int ldm,
                                                          int* __restrict__ info, double* __restrict__ s,
                                                          int pairs, int* __restrict__ cond) {
    extern __shared__ double dyn_s[];
    chol_drop_body(a, g, ldg, ref2, drop, m, ldm, info, s, kCholSmemMaxA, dyn_s, pairs != 0, cond);
}

// Grid-cooperative variant for blocks beyond shared memory (a > kCholSmemMaxA:
// config 5's 768-wide real embedding of a 384-wide complex Gram, config 3's SI
// block of 200): the same decisions, operation order and output as
// chol_drop_body, with the Schur complement in global memory (L2-resident), its
// rows dealt over every warp of the grid and one grid barrier per pivot.  One
// CTA walking a 768 x 768 complement through L2 took 40 ms; the grid takes ~2.
// work layout: s (a x a) | gd, r2, piv (a each) | slot (a ints) | flags (4 ints)
__global__ void __launch_bounds__(1024) chol_coop_kernel(int a, const double* __restrict__ g, int ldg,
                                                          const double* __restrict__ ref2, double drop,
                                                          double* __restrict__ m, int ldm, int* __restrict__ info,
                                                          double* __restrict__ s, int pairs, int* __restrict__ cond) {
    namespace cgr = cooperative_groups;
    cgr::grid_group grid = cgr::this_grid();
    double* gd = s + static_cast<size_t>(a) * a;
    double* r2 = gd + a;
    double* piv = r2 + a;
    int* slot = reinterpret_cast<int*>(piv + a);
    int* flags = slot + a;  // [0] unsure, [1] bad
    const int tid = threadIdx.x, lane = tid & 31;
    const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
    const int gw = gtid >> 5, gwarps = gthreads >> 5;
    const bool lead = gtid == 0;
    for (size_t e = gtid; e < static_cast<size_t>(a) * a; e += gthreads)
        s[e] = g[(e / a) * ldg + e % a];
    for (int j = gtid; j < a; j += gthreads) {
        gd[j] = g[static_cast<size_t>(j) * ldg + j];
        r2[j] = ref2 ? ref2[j] : 0.0;
    }
    if (lead) flags[0] = flags[1] = 0;
    grid.sync();
    const double drop2 = drop * drop;
    constexpr double kLo2 = (1.0 - 1e-4) * (1.0 - 1e-4), kHi2 = (1.0 + 1e-4) * (1.0 + 1e-4);
    int kept = 0;
    double worst = 0.0;  // max g_jj / p_j over kept pivots (cond)
    // keep decision of a non-odd-twin pivot (the reference's drop rule)
    auto decide_even = [&](int j, double p, bool& unsure, bool& bad) -> int {
        const double gjj = gd[j];
        if (!isfinite(p) || !isfinite(gjj)) {
            bad = true;
            return 0;
        }
        if (ref2 == nullptr) {
            unsure = p <= 1e-8 * gjj;
            return p > 0.0;
        }
        const double thr2 = drop2 * r2[j];
        if (r2[j] == 0.0 || gjj < thr2) return 0;
        unsure = p < 1e-8 * gjj || (p > kLo2 * thr2 && p < kHi2 * thr2);
        return p >= thr2;
    };
    if (pairs == 2 && (a & 1) == 0) {
        // Real embedding of a complex Gram: pivots 2c and 2c + 1 in one grid step
        // (half the grid barriers).  Bit-identical to the pivot-by-pivot loop
        // below: every thread forms row 2c + 1's update by pivot 2c on the fly,
        // f = s[2c][2c+1] / p0, s'[2c+1][l] = s[2c+1][l] - f s[2c][l], with the
        // same expressions that loop evaluates, and each trailing row receives
        // the two rank-1 updates in the same order; row 2c + 1 itself is written
        // back in the next step (nobody reads it there).
        for (int j = 0; j < a; j += 2) {
            if (j >= 2 && slot[j - 2] >= 0) {  // deferred write-back of row j - 1
                const double* rowe = s + static_cast<size_t>(j - 2) * a;
                double* rowo = s + static_cast<size_t>(j - 1) * a;
                const double fo = rowe[j - 1] * (1.0 / piv[j - 2]);
                for (int l = j - 1 + gtid; l < a; l += gthreads) rowo[l] -= fo * rowe[l];
            }
            const double* row0 = s + static_cast<size_t>(j) * a;
            const double* row1 = row0 + a;
            const double p0 = row0[j];
            bool unsure0 = false, bad0 = false, bad1 = false;
            const int keep0 = decide_even(j, p0, unsure0, bad0);
            const double invp0 = keep0 ? 1.0 / p0 : 0.0;
            const double f01 = keep0 ? row0[j + 1] * invp0 : 0.0;
            const double p1 = keep0 ? row1[j + 1] - f01 * row0[j + 1] : row1[j + 1];
            int keep1;
            bool unsure1 = false;
            if (!isfinite(p1) || !isfinite(gd[j + 1])) {
                bad1 = true;
                keep1 = 0;
            } else {
                keep1 = keep0 && p1 > 0.0;
                unsure1 = (keep0 != 0) != (p1 > 0.0);
            }
            if (lead) {
                if (unsure0 || unsure1) flags[0] = 1;
                if (bad0 || bad1) flags[1] = 1;
                slot[j] = keep0 ? kept : -1;
                slot[j + 1] = keep1 ? kept + keep0 : -1;
                piv[j] = p0;
                piv[j + 1] = p1;
            }
            if (keep0) worst = fmax(worst, gd[j] / p0);
            if (keep1) worst = fmax(worst, gd[j + 1] / p1);
            kept += keep0 + keep1;
            if (keep0) {
                const double invp1 = keep1 ? 1.0 / p1 : 0.0;
                for (int k = j + 2 + gw; k < a; k += gwarps) {
                    const double rk0 = row0[k] * invp0;
                    const double s1k = row1[k] - f01 * row0[k];
                    const double rk1 = s1k * invp1;
                    double* rowk = s + static_cast<size_t>(k) * a;
                    for (int l = k + lane; l < a; l += 32) {
                        double v = rowk[l];
                        v -= rk0 * row0[l];
                        if (keep1) v -= rk1 * (row1[l] - f01 * row0[l]);
                        rowk[l] = v;
                    }
                }
            }
            grid.sync();
        }
        if (a >= 2 && slot[a - 2] >= 0) {  // the last odd row
            const double* rowe = s + static_cast<size_t>(a - 2) * a;
            double* rowo = s + static_cast<size_t>(a - 1) * a;
            const double fo = rowe[a - 1] * (1.0 / piv[a - 2]);
            for (int l = a - 1 + gtid; l < a; l += gthreads) rowo[l] -= fo * rowe[l];
        }
        grid.sync();
    } else {
        for (int j = 0; j < a; ++j) {
            const double p = s[static_cast<size_t>(j) * a + j];
            const double gjj = gd[j];
            int keep;
            bool unsure = false, bad = false;
            if (pairs && (j & 1)) {
                if (!isfinite(p) || !isfinite(gjj)) {
                    bad = true;
                    keep = 0;
                } else {
                    keep = slot[j - 1] >= 0 && p > 0.0;
                    unsure = (slot[j - 1] >= 0) != (p > 0.0);
                }
            } else {
                keep = decide_even(j, p, unsure, bad);
            }
            if (lead) {
                if (unsure) flags[0] = 1;
                if (bad) flags[1] = 1;
                slot[j] = keep ? kept : -1;
                piv[j] = p;
            }
            if (keep) {
                ++kept;
                worst = fmax(worst, gjj / p);
                const double invp = 1.0 / p;
                const double* rowj = s + static_cast<size_t>(j) * a;
                for (int k = j + 1 + gw; k < a; k += gwarps) {
                    const double rk = rowj[k] * invp;
                    double* rowk = s + static_cast<size_t>(k) * a;
                    for (int l = k + lane; l < a; l += 32) rowk[l] -= rk * rowj[l];
                }
            }
            grid.sync();
        }
    }
    for (size_t e = gtid; e < static_cast<size_t>(a) * a; e += gthreads) {
        const int j = static_cast<int>(e / a), l = static_cast<int>(e % a);
        if (l < j || slot[j] < 0) continue;
        const double rj = sqrt(piv[j]);
        s[e] = l == j ? rj : s[e] / rj;
    }
    grid.sync();
    for (size_t e = gtid; e < static_cast<size_t>(a) * a; e += gthreads) {
        const int j = static_cast<int>(e / a), l = static_cast<int>(e % a);
        if (l > j && (slot[j] < 0 || slot[l] < 0)) s[e] = 0.0;
    }
    grid.sync();
    for (int i = gtid; i < a; i += gthreads) piv[i] = slot[i] >= 0 ? 1.0 / s[static_cast<size_t>(i) * a + i] : 0.0;
    grid.sync();
    for (int c = gw; c < a; c += gwarps) {
        if (slot[c] < 0) continue;
        const double* rowc = s + static_cast<size_t>(c) * a;
        for (int i = c - 1; i >= 0; --i) {
            if (slot[i] < 0) continue;
            const double* rowi = s + static_cast<size_t>(i) * a;
            double acc = 0.0;
            for (int l = i + 1 + lane; l < c; l += 32) acc = fma(rowi[l], rowc[l], acc);
            acc = warp_sum(acc);
            if (lane == 0) s[static_cast<size_t>(c) * a + i] = -(acc + rowi[c] * piv[c]) * piv[i];
            __syncwarp();
        }
    }
    grid.sync();
    for (size_t e = gtid; e < static_cast<size_t>(a) * a; e += gthreads)
        m[(e / a) * ldm + e % a] = 0.0;
    grid.sync();
    for (size_t e = gtid; e < static_cast<size_t>(a) * a; e += gthreads) {
        const int i = static_cast<int>(e / a), c = static_cast<int>(e % a);
        if (i > c || slot[i] < 0 || slot[c] < 0) continue;
        const double val = i == c ? piv[c] : s[static_cast<size_t>(c) * a + i];
        m[static_cast<size_t>(i) * ldm + slot[c]] = val;
    }
    if (lead) {
        info[0] = kept;
        info[1] = flags[0];
        info[2] = flags[1];
        if (cond) {
            const int ill = kept > 0 && !(worst <= kCondFused);
            cond[0] = ill;
            cond[1] = kept > 0 && !ill;
        }
    }
}

// ------------------------------------------------------------------ K5
constexpr int kJacobiSmemMaxD = 160;
constexpr int kJacobiThreads = 1024;
constexpr int kMaxPairs = 1024;  // pairs per round: d <= 2048

__device__ __forceinline__ int rr_index(int r, int i, int m) { return i == 0 ? 0 : 1 + (i - 1 + r) % (m - 1); }

__global__ void __launch_bounds__(kJacobiThreads) jacobi_kernel(int d, const double* __restrict__ hin, int ldh,
                                                                 double* __restrict__ hg, double* __restrict__ v,
                                                                 double* __restrict__ values,
                                                                 double* __restrict__ z, int ldz,
                                                                 int* __restrict__ info, int use_smem) {
    extern __shared__ double dyn[];
    __shared__ int pp[kMaxPairs / 2 + 1], pq[kMaxPairs / 2 + 1];
    __shared__ double pc[kMaxPairs / 2 + 1], ps[kMaxPairs / 2 + 1], pt[kMaxPairs / 2 + 1];
    __shared__ double red[kJacobiThreads / 32];
    __shared__ double s_fro, s_sweep_max;
    double* h = use_smem ? dyn : hg;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const int m = d + (d & 1);
    const int np = m / 2;

    // symmetrise, V = I, ||H||_F
    double f2 = 0.0;
    for (int e = tid; e < d * d; e += nt) {
        const int i = e / d, j = e % d;
        const double hv = 0.5 * (hin[static_cast<size_t>(i) * ldh + j] + hin[static_cast<size_t>(j) * ldh + i]);
        h[e] = hv;
        v[e] = i == j ? 1.0 : 0.0;
        f2 = fma(hv, hv, f2);
    }
    f2 = warp_sum(f2);
    if (lane == 0) red[wid] = f2;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < nt / 32; ++w) s += red[w];
        s_fro = sqrt(s);
    }
    __syncthreads();
    const double fro = s_fro;
    const double skip = 1e-18 * fro;
    const double stop = 1e-16 * fro;
    int sweep = 0;
    bool converged = fro == 0.0 || d < 2;
    for (; sweep < 60 && !converged; ++sweep) {
        double my_max = 0.0;
        for (int r = 0; r < m - 1; ++r) {
            for (int k = tid; k < np; k += nt) {
                int p = rr_index(r, k, m), q = rr_index(r, m - 1 - k, m);
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                pp[k] = p;
                pq[k] = q;
                double c = 1.0, s = 0.0, t = 0.0;
                if (q < d) {
                    const double apq = h[p * d + q];
                    my_max = fmax(my_max, fabs(apq));
                    if (fabs(apq) > skip) {
                        const double theta = (h[q * d + q] - h[p * d + p]) / (2.0 * apq);
                        t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
                        c = 1.0 / sqrt(fma(t, t, 1.0));
                        s = t * c;
                    }
                }
                pc[k] = c;
                ps[k] = s;
                pt[k] = t;
            }
            __syncthreads();
            // H <- J^T H J, one thread per 2x2 block (k1 <= k2), mirrored
            const int nblk = np * (np + 1) / 2;
            for (int e = tid; e < nblk; e += nt) {
                int k1 = static_cast<int>((2.0 * np + 1.0 - sqrt((2.0 * np + 1.0) * (2.0 * np + 1.0) - 8.0 * e)) / 2.0);
                while (k1 > 0 && k1 * np - k1 * (k1 - 1) / 2 > e) --k1;
                while ((k1 + 1) * np - (k1 + 1) * k1 / 2 <= e) ++k1;
                const int k2 = k1 + (e - (k1 * np - k1 * (k1 - 1) / 2));
                const int p1 = pp[k1], q1 = pq[k1], p2 = pp[k2], q2 = pq[k2];
                const double c1 = pc[k1], s1 = ps[k1], c2 = pc[k2], s2 = ps[k2];
                if (k1 == k2) {
                    if (q1 < d && s1 != 0.0) {
                        const double apq = h[p1 * d + q1];
                        h[p1 * d + p1] -= pt[k1] * apq;
                        h[q1 * d + q1] += pt[k1] * apq;
                        h[p1 * d + q1] = 0.0;
                        h[q1 * d + p1] = 0.0;
                    }
                    continue;
                }
                const bool q1ok = q1 < d, q2ok = q2 < d;
                double a00 = h[p1 * d + p2];
                double a01 = q2ok ? h[p1 * d + q2] : 0.0;
                double a10 = q1ok ? h[q1 * d + p2] : 0.0;
                double a11 = (q1ok && q2ok) ? h[q1 * d + q2] : 0.0;
                // rows: [x_p; x_q] -> [c x_p - s x_q; s x_p + c x_q]
                double b00 = c1 * a00 - s1 * a10, b10 = s1 * a00 + c1 * a10;
                double b01 = c1 * a01 - s1 * a11, b11 = s1 * a01 + c1 * a11;
                // columns likewise
                a00 = c2 * b00 - s2 * b01;
                a01 = s2 * b00 + c2 * b01;
                a10 = c2 * b10 - s2 * b11;
                a11 = s2 * b10 + c2 * b11;
                h[p1 * d + p2] = a00;
                h[p2 * d + p1] = a00;
                if (q2ok) {
                    h[p1 * d + q2] = a01;
                    h[q2 * d + p1] = a01;
                }
                if (q1ok) {
                    h[q1 * d + p2] = a10;
                    h[p2 * d + q1] = a10;
                }
                if (q1ok && q2ok) {
                    h[q1 * d + q2] = a11;
                    h[q2 * d + q1] = a11;
                }
            }
            // V <- V J (rows independent)
            for (int e = tid; e < d * np; e += nt) {
                const int i = e / np, k = e % np;
                const int p = pp[k], q = pq[k];
                if (q >= d || ps[k] == 0.0) continue;
                const double c = pc[k], s = ps[k];
                const double vp = v[i * d + p], vq = v[i * d + q];
                v[i * d + p] = c * vp - s * vq;
                v[i * d + q] = s * vp + c * vq;
            }
            __syncthreads();
        }
        for (int o = 16; o > 0; o >>= 1) my_max = fmax(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
        if (lane == 0) red[wid] = my_max;
        __syncthreads();
        if (tid == 0) {
            double mx = 0.0;
            for (int w = 0; w < nt / 32; ++w) mx = fmax(mx, red[w]);
            s_sweep_max = mx;
        }
        __syncthreads();
        converged = s_sweep_max <= stop;
    }
    // ascending stable order: rank_j = #{i : h_i < h_j or (h_i == h_j and i < j)}
    for (int j = tid; j < d; j += nt) {
        const double hj = h[j * d + j];
        int rank = 0;
        for (int i = 0; i < d; ++i) {
            const double hi = h[i * d + i];
            rank += (hi < hj) || (hi == hj && i < j);
        }
        values[rank] = hj;
        for (int i = 0; i < d; ++i) z[static_cast<size_t>(i) * ldz + rank] = v[i * d + j];
    }
    if (tid == 0) {
        info[0] = sweep;
        info[1] = converged ? 0 : 1;
    }
}

}  // namespace
}  // namespace bk

using namespace bk;

extern "C" size_t bk_chol_work_bytes(int a) {
    const size_t aa = static_cast<size_t>(a > 0 ? a : 1);
    return (aa * aa + 3 * aa) * sizeof(double) + aa * sizeof(int) + 64;
}

namespace bk {
int chol_launch(int a, const double* g, int ldg, const double* ref2, double drop, double* m, int ldm, int* info,
                void* work, cudaStream_t st, bool pairs, int* cond) {
    if (a <= 0) {
        BK_RET(cudaMemsetAsync(info, 0, 3 * sizeof(int), st));
        if (cond) BK_RET(cudaMemsetAsync(cond, 0, 2 * sizeof(int), st));
        return 0;
    }
    auto s = static_cast<double*>(work);  // a x a (used when a > kCholSmemMaxA)
    if (a > 4096) return static_cast<int>(cudaErrorInvalidValue);
    const cudaError_t attr = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(
        chol_drop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>((kCholSmemMaxA * kCholSmemMaxA + 4 * kCholSmemMaxA) * sizeof(double))));
    BK_RET(attr);
    const size_t small = (3 * static_cast<size_t>(a) + (a + 1) / 2) * sizeof(double);
    const size_t smem = small + (a <= kCholSmemMaxA ? static_cast<size_t>(a) * a * sizeof(double) : 0);
    if (a > kCholSmemMaxA) {
        // grid-cooperative: one warp per trailing row at most, one CTA per SM at most
        int per_sm = 0;
        BK_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_coop_kernel, 1024, 0));
        const int grid = max(1, min(min(ceil_div(a, 32), kSMs), max(per_sm, 1) * kSMs));
        // pairs: 2 = the paired-pivot grid step (default), 1 = pivot by pivot
        // (BK_CHOL_PAIRSTEP=0, read per call: the bit-identity test)
        const char* ps = getenv("BK_CHOL_PAIRSTEP");
        int aa = a, l1 = ldg, l2 = ldm, pr = pairs ? ((ps && ps[0] == '0') ? 1 : 2) : 0;
        void* args[] = {&aa, const_cast<double**>(&g), &l1, const_cast<double**>(&ref2), &drop, &m, &l2, &info, &s,
                        &pr, &cond};
        BK_RET(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(chol_coop_kernel), dim3(grid), dim3(1024),
                                           args, 0, st));
        return 0;
    }
    // 1024 threads: the per-pivot rank-1 updates are the work (fewer warps measured
    // 1.3-4x slower at a = 96..288)
    static const int threads = [] {  // BK_CHOL_THREADS: CTA size (tuning runs only)
        const char* e = getenv("BK_CHOL_THREADS");
        return e ? max(32, min(1024, atoi(e) / 32 * 32)) : 1024;
    }();
    chol_drop_kernel<<<1, threads, smem, st>>>(a, g, ldg, ref2, drop, m, ldm, info, s, pairs ? 1 : 0, cond);
    BK_LAUNCHED();
}
}  // namespace bk

extern "C" int bk_chol_drop_d(int a, const double* g, int ldg, const double* ref2, double drop, double* m,
                              int ldm, int* info, void* work, void* stream) {
    return chol_launch(a, g, ldg, ref2, drop, m, ldm, info, work, as_stream(stream), false);
}

extern "C" int bk_chol_drop_cond_d(int a, const double* g, int ldg, const double* ref2, double drop, double* m,
                                   int ldm, int* info, int* cond, void* work, void* stream) {
    return chol_launch(a, g, ldg, ref2, drop, m, ldm, info, work, as_stream(stream), false, cond);
}

extern "C" size_t bk_syev_jacobi_work_bytes(int d) {
    const size_t dd = static_cast<size_t>(d > 0 ? d : 1);
    return 2 * dd * dd * sizeof(double);
}

extern "C" int bk_syev_jacobi_d(int d, double* h, int ldh, double* values, double* z, int ldz, void* work,
                         int* info, void* stream) {
    if (d <= 0) return 0;
    if (d > kMaxPairs * 2) return static_cast<int>(cudaErrorInvalidValue);
    const cudaStream_t s = as_stream(stream);
    auto hg = static_cast<double*>(work);
    double* v = hg + static_cast<size_t>(d) * d;
    const int use_smem = d <= kJacobiSmemMaxD ? 1 : 0;
    const size_t smem = use_smem ? static_cast<size_t>(d) * d * sizeof(double) : 0;
    const cudaError_t attr = BK_ONCE_PER_DEVICE(cudaFuncSetAttribute(
        jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(kJacobiSmemMaxD * kJacobiSmemMaxD * sizeof(double))));
    BK_RET(attr);
    jacobi_kernel<<<1, kJacobiThreads, smem, s>>>(d, h, ldh, hg, v, values, z, ldz, info, use_smem);
    BK_LAUNCHED();
}
