// Helpers shared by the real (bk_dense.cu) and complex 3M (bk_zdense.cu) DMMA
// contraction kernels: cp.async tile staging, the split-K plan of the Grams.
#pragma once
#include <algorithm>

#include "bk_common.cuh"

namespace bk {
namespace {

template <bool V16>
__device__ __forceinline__ void load_rows(double* dst, int pitch, const double* __restrict__ src, int ld, int r0,
                                          int r_end, int c0, int c_end, int rows, int cols, int tid, int nthreads) {
    // copy src[r0 + r][c0 + c] for r < rows, c < cols into dst[r*pitch + c], zero outside
    if constexpr (V16) {
        const int cpr = cols / 2;  // 16-byte chunks per row (cols even)
        for (int e = tid; e < rows * cpr; e += nthreads) {
            const int r = e / cpr, c = 2 * (e - r * cpr);
            const int row = r0 + r, col = c0 + c;
            int bytes = 0;
            if (row < r_end && col < c_end) bytes = col + 1 < c_end ? 16 : 8;
            const double* g = bytes ? src + static_cast<size_t>(row) * ld + col : src;
            cp_async16(dst + r * pitch + c, g, bytes);
        }
    } else {
        for (int e = tid; e < rows * cols; e += nthreads) {
            const int r = e / cols, c = e - r * cols;
            const int row = r0 + r, col = c0 + c;
            const bool ok = row < r_end && col < c_end;
            cp_async8(dst + r * pitch + c, ok ? src + static_cast<size_t>(row) * ld + col : src, ok);
        }
    }
}

// 16-byte cp.async tile copy with the shape fixed at compile time (ROWS rows of
// CPR 16-byte chunks, NT threads): src[r0 + r][c0 + 2c'] -> dst[r * pitch + 2c'],
// zero-filled outside rows < r_end, columns < c_end (c_end even: complex views)
template <int ROWS, int CPR, int NT>
__device__ __forceinline__ void load_tile16(double* dst, int pitch, const double* __restrict__ src, int ld, int r0,
                                            int r_end, int c0, int c_end, int tid) {
    constexpr int TOTAL = ROWS * CPR;
#pragma unroll
    for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
        const int e = tid + it * NT;
        if (TOTAL % NT != 0 && e >= TOTAL) break;
        const int r = e / CPR, c = 2 * (e % CPR);
        const int row = r0 + r, col = c0 + c;
        const bool ok = row < r_end && col < c_end;
        cp_async16(dst + r * pitch + c, ok ? src + static_cast<size_t>(row) * ld + col : src, ok);
    }
}

// The same with the real kernels' shapes: V16 copies 16-byte chunks (an odd
// width's last chunk copies 8 bytes and zero-fills the rest), else 8-byte
// elements; ROWS x COLS doubles, NT threads, all fixed at compile time
template <bool V16, int ROWS, int COLS, int NT>
__device__ __forceinline__ void load_tile(double* dst, int pitch, const double* __restrict__ src, int ld, int r0,
                                          int r_end, int c0, int c_end, int tid) {
    if constexpr (V16) {
        constexpr int CPR = COLS / 2, TOTAL = ROWS * CPR;
#pragma unroll
        for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
            const int e = tid + it * NT;
            if (TOTAL % NT != 0 && e >= TOTAL) break;
            const int r = e / CPR, c = 2 * (e % CPR);
            const int row = r0 + r, col = c0 + c;
            int bytes = 0;
            if (row < r_end && col < c_end) bytes = col + 1 < c_end ? 16 : 8;
            cp_async16(dst + r * pitch + c, bytes ? src + static_cast<size_t>(row) * ld + col : src, bytes);
        }
    } else {
        constexpr int TOTAL = ROWS * COLS;
#pragma unroll
        for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
            const int e = tid + it * NT;
            if (TOTAL % NT != 0 && e >= TOTAL) break;
            const int r = e / COLS, c = e % COLS;
            const int row = r0 + r, col = c0 + c;
            const bool ok = row < r_end && col < c_end;
            cp_async8(dst + r * pitch + c, ok ? src + static_cast<size_t>(row) * ld + col : src, ok);
        }
    }
}

struct GramPlan {
    int splits, rows_per_split;
};

// Split-K partials budget (doubles) for an a x b Gram over n rows: the partial
// tiles may add at most 1/40 of the input traffic, but never less than two
// full waves of 96 x 96 tiles' worth (small outputs)
inline size_t gram_budget(int n, int a, int b) {
    const size_t floor_elems = 2 * (2 * static_cast<size_t>(kSMs) + 8) * 96 * 96;
    const size_t traffic = static_cast<size_t>(max(n, 1)) * (max(a, 1) + max(b, 1)) / 40;
    return std::max(floor_elems, traffic);
}

// Split count for `tiles` output tiles (partial size a*b per split): enough CTAs
// for whole waves of cps x 148 resident CTAs — a last wave with a handful of
// CTAs doubles the time (config 5's Hermitian Rayleigh-Ritz Gram has 300 upper
// tiles of the 2304-wide real view: one split is 300 CTAs on 296 slots) — within
// the partials budget and >= 256 rows per split.
inline GramPlan gram_plan(int n, int tiles, int a, int b, int cps = 2, int tk = 16) {
    const int slots = cps * kSMs;
    int max_split = max(1, ceil_div(n, 256));
    const size_t out_elems = static_cast<size_t>(max(a, 1)) * max(b, 1);
    const size_t by_budget = gram_budget(n, a, b) / out_elems;
    max_split = static_cast<int>(std::min<size_t>(static_cast<size_t>(max_split), std::max<size_t>(1, by_budget)));
    int splits = 1;
    double best = 0.0;
    for (int sp = 1; sp <= max_split; ++sp) {
        const int ctas = tiles * sp;
        const int waves = ceil_div(ctas, slots);
        const double eff = static_cast<double>(ctas) / (static_cast<double>(waves) * slots);
        if (eff > best + 0.01) {  // fewest splits within 1 % of the best wave efficiency
            best = eff;
            splits = sp;
        }
        if (ctas >= 64 * slots) break;
    }
    int rps = ceil_div(n, splits);
    rps = ceil_div(rps, tk) * tk;
    splits = max(1, ceil_div(n, rps));
    return {splits, rps};
}

inline bool aligned16(const double* p, int ld) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld & 1) == 0; }

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}


// contractions over a short axis (coefficient space) use the CUDA-core forms
constexpr int kSmallN = 512;

}  // namespace
}  // namespace bk
