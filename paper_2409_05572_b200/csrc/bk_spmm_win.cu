// K1w — window-staged CSR SpMM, Y = A X (sm_100a), bit-identical to K1.
//
// The plain K1 (bk_spmm.cu) gathers one X row per nonzero through L1/L2: on a
// 7-point stencil that is ~5 L2 row loads per matrix row after L1 hits, and the
// kernel waits on those register-landing gathers (config 2: 0.37 of HBM).
// Here a host plan (host/tiling.cpp) regroups the rows into tiles of graph-local
// rows and lists each tile's window: its own rows plus the halo columns its
// rows reference.  A CTA stages a window's X rows in shared memory — one column
// chunk of kc columns at a time, so the window fits beside the other resident
// CTAs — with one bulk copy per row (cp.async.bulk completing on an mbarrier),
// and the tile's index slice (row pointers, row ids, (slot, val) per nonzero)
// with cp.async one tile ahead; tile descriptors and the window's row ids are
// prefetched into registers.  Every nonzero then reads its X row from shared
// memory: an X row crosses L2 -> SM once per tile that touches it (64-row
// tiles of the 7-point stencil: 2.4 loads per matrix row).  Three CTAs per SM:
// one CTA's copies run while the others multiply.
//
// Products: LPR lanes per matrix row (32/LPR rows per warp), each lane V x
// double2 columns, four nonzeros' shared-memory reads in flight; a row's
// nonzeros are accumulated in their CSR order with one fma each, exactly as K1
// does, so Y is bit-identical (proj/src/kernel.cpp:8-33 is the reference loop).
// Algorithmic bytes as K1: 12 nnz + 4 (n + 1) + 16 n k; the on-chip gathers cost
// nnz * k * 8 bytes of shared-memory bandwidth (128 B/clk/SM), which bounds
// matrices with many nonzeros per row (config 4: 25 per row).  Measurements and
// the variants tried: profiles/r02_spmm_win.md.
#include <cstdlib>
#include <type_traits>

#include "bk_common.cuh"

namespace bk {
namespace {

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
// one row chunk, global -> shared, by the bulk-copy engine (SASS UBLKCP): no
// per-16-byte instructions and no LSU wavefronts; completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int LPR, int V>
__global__ void __launch_bounds__(256, 3) spmm_d_win_kernel(int n, int T, int ntiles, int wmax, int nzmax,
                                                          const int32_t* __restrict__ rp2,
                                                          const int32_t* __restrict__ code,
                                                          const double* __restrict__ val2,
                                                          const int32_t* __restrict__ wptr,
                                                          const int32_t* __restrict__ wrow,
                                                          const double* __restrict__ x, int ldx, int k, int kc,
                                                          int nch, double* __restrict__ y, int ldy, int skip) {
    // mbarrier | wmax x kc X rows | 2 x (nzmax vals | nzmax slots | T + 1 row pointers | T row ids)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    double* xs = reinterpret_cast<double*>(smem_raw + 16);
    unsigned char* ibase = reinterpret_cast<unsigned char*>(xs + static_cast<size_t>(wmax) * kc);
    const size_t ibytes = (12 * static_cast<size_t>(nzmax) + 4 * (2 * static_cast<size_t>(T) + 1) + 15) & ~size_t(15);
    // index slice of the tile being multiplied (set per tile)
    const double* sval = nullptr;
    const int* soff = nullptr;
    const int* srp = nullptr;
    const int* sid = nullptr;
    constexpr int RPW = 32 / LPR;  // matrix rows per warp
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hl = lane & (LPR - 1), sub = lane / LPR;
    const int grp = warp * RPW + sub, ngrp = (blockDim.x >> 5) * RPW;
    const int kr = (k + 1) & ~1;  // columns incl. the pad of an odd width (inside the row: ld is even)
    const int rowbytes = kc * 8;
    // this lane's first double2 of slot 0; lanes past the chunk read the next
    // slot's columns (or the index slice after the last slot) and never store
    const char* xlane = reinterpret_cast<const char*>(xs) + hl * 16;
    // N nonzeros of one row: all their X reads issued, then the fmas in CSR order
    // N nonzeros of one row over VL 16-byte column groups: all their X reads issued,
    // then the fmas in CSR order
    auto step = [&](auto nc, auto vl, int q, auto& acc) {
        constexpr int N = decltype(nc)::value;
        constexpr int VL = decltype(vl)::value;
        double2 xv[N][VL];
        double vv[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const char* xr = xlane + soff[q + i] * rowbytes;
            vv[i] = sval[q + i];
#pragma unroll
            for (int u = 0; u < VL; ++u) xv[i][u] = *reinterpret_cast<const double2*>(xr + u * (LPR * 16));
        }
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int u = 0; u < VL; ++u) {
                acc[u].x = fma(vv[i], xv[i][u].x, acc[u].x);
                acc[u].y = fma(vv[i], xv[i][u].y, acc[u].y);
            }
    };
    // Index loads are kept off the critical path: a tile's descriptor (window and
    // nonzero ranges) is loaded one tile ahead and the X-row ids of its window two
    // steps ahead of the copies that need them (8 per lane group, in registers,
    // reused by every column chunk of the tile), so the only exposed memory round
    // trip of a chunk is the X rows themselves.
    constexpr int MAXR = 8;
    struct Desc {
        int w0, ws, p0, p1;
    };
    auto load_desc = [&](int t) {
        Desc d{0, 0, 0, 0};
        if (t < ntiles) {
            const int r0 = t * T, nr = min(T, n - r0);
            d.w0 = __ldg(wptr + t);
            d.ws = __ldg(wptr + t + 1) - d.w0;
            d.p0 = __ldg(rp2 + r0);
            d.p1 = __ldg(rp2 + r0 + nr);
        }
        return d;
    };
    auto load_rows = [&](const Desc& d, int first, int (&rows)[MAXR]) {
#pragma unroll
        for (int j = 0; j < MAXR; ++j) {
            const int sl = first + grp + j * ngrp;
            rows[j] = sl < d.ws ? __ldg(wrow + d.w0 + sl) : 0;
        }
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    // a tile's index slice (row pointers, row ids, (slot, val) per nonzero) -> buffer ib
    auto stage_index = [&](int t, const Desc& d, int ib) {
        double* v = reinterpret_cast<double*>(ibase + ib * ibytes);
        int* o = reinterpret_cast<int*>(v + nzmax);
        int* rp = o + nzmax;
        int* id = rp + T + 1;
        const int r0 = t * T, nr = min(T, n - r0);
        for (int i = tid; i <= nr; i += blockDim.x) cp_async4(rp + i, rp2 + r0 + i);
        for (int i = tid; i < nr; i += blockDim.x) cp_async4(id + i, wrow + d.w0 + i);
        for (int q = tid; q < d.p1 - d.p0; q += blockDim.x) {
            cp_async8(v + q, val2 + d.p0 + q, true);
            cp_async4(o + q, code + d.p0 + q);
        }
        cp_async_commit();
    };
    Desc cur = load_desc(blockIdx.x), nxt = load_desc(blockIdx.x + gridDim.x);
    int rows[MAXR];
    load_rows(cur, 0, rows);
    int ib = 0;
    if (static_cast<int>(blockIdx.x) < ntiles) stage_index(blockIdx.x, cur, 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int nr = min(T, n - t * T);
        const int ws = cur.ws, p0 = cur.p0;
        const Desc nn = load_desc(t + 2 * gridDim.x);  // two tiles ahead: never waited for
        int nrows[MAXR];
        sval = reinterpret_cast<const double*>(ibase + ib * ibytes);
        soff = reinterpret_cast<const int*>(sval + nzmax);
        srp = soff + nzmax;
        sid = srp + T + 1;
        for (int ch = 0; ch < nch; ++ch) {
            const int c0 = ch * kc;
            const int kw2 = (min(kc, kr - c0) + 1) >> 1;  // live double2 per row in this chunk
            // the window's X rows: LPR lanes copy one row's chunk, 16 bytes each
            if (tid == 0) mbar_expect_tx(bar, static_cast<uint32_t>(ws) * kw2 * 16u);
#pragma unroll
            for (int j = 0; j < MAXR; ++j) {
                const int sl = grp + j * ngrp;
                if (sl < ws && hl == 0)
                    bulk_g2s(xs + static_cast<size_t>(sl) * kc, x + static_cast<size_t>(rows[j]) * ldx + c0, kw2 * 16u, bar);
            }
            for (int first = MAXR * ngrp; first < ws; first += MAXR * ngrp) {  // windows beyond 8 rows per group
                int more[MAXR];
                load_rows(cur, first, more);
#pragma unroll
                for (int j = 0; j < MAXR; ++j) {
                    const int sl = first + grp + j * ngrp;
                    if (sl < ws && hl == 0)
                        bulk_g2s(xs + static_cast<size_t>(sl) * kc, x + static_cast<size_t>(more[j]) * ldx + c0, kw2 * 16u,
                                 bar);
                }
            }
            // the next tile's row ids and index slice fly during the products below
            bool prefetched = false;
            if (ch == nch - 1) {
                load_rows(nxt, 0, nrows);
                if (t + static_cast<int>(gridDim.x) < ntiles) {
                    stage_index(t + gridDim.x, nxt, ib ^ 1);
                    prefetched = true;
                }
            }
            if (ch == 0) {  // this tile's index slice (staged one tile ago)
                if (prefetched) cp_async_wait<1>();
                else cp_async_wait<0>();
            }
            // one warp polls the window's mbarrier; the others sleep on the block
            // barrier instead of spinning on try_wait (the polls of the CTAs still
            // waiting took issue slots from the one multiplying)
            if (warp == 0) mbar_wait(bar, phase);
            phase ^= 1;
            __syncthreads();  // index slice and window visible to all
            // the products of the tile's rows over the chunk's VL live column groups
            // (a narrower last chunk skips the empty ones)
            auto rows_pass = [&](auto vl) {
                constexpr int VL = decltype(vl)::value;
                for (int sl = grp; sl < nr; sl += ngrp) {
                    const int e = srp[sl + 1] - p0;
                    int q = srp[sl] - p0;
                    double2 acc[VL];
#pragma unroll
                    for (int u = 0; u < VL; ++u) acc[u] = make_double2(0.0, 0.0);
                    for (; q + 4 <= e; q += 4) step(std::integral_constant<int, 4>{}, vl, q, acc);
                    const int rem = e - q;
                    if (rem == 3) step(std::integral_constant<int, 3>{}, vl, q, acc);
                    else if (rem == 2) step(std::integral_constant<int, 2>{}, vl, q, acc);
                    else if (rem == 1) step(std::integral_constant<int, 1>{}, vl, q, acc);
                    double* yr = y + static_cast<size_t>(sid[sl]) * ldy + c0;
#pragma unroll
                    for (int u = 0; u < VL; ++u) {
                        const int c = 2 * (hl + LPR * u);
                        if (hl + LPR * u < kw2) {
                            if (c0 + c < skip) {  // the pad column in front of an odd view: never written
                                if (c0 + c + 1 < k) yr[c + 1] = acc[u].y;
                            } else if (c0 + c + 1 < k) {
                                reinterpret_cast<double2*>(yr)[hl + LPR * u] = acc[u];
                            } else if (c0 + c < k) {
                                yr[c] = acc[u].x;
                            }
                        }
                    }
                }
            };
            const int vlive = (kw2 + LPR - 1) / LPR;
            if (vlive >= V) rows_pass(std::integral_constant<int, V>{});
            else if (V > 3 && vlive == 3) rows_pass(std::integral_constant<int, (V > 3 ? 3 : 1)>{});
            else if (V > 2 && vlive == 2) rows_pass(std::integral_constant<int, (V > 2 ? 2 : 1)>{});
            else rows_pass(std::integral_constant<int, 1>{});
            __syncthreads();  // the window is restaged for the next chunk / tile
        }
        cur = nxt;
        nxt = nn;
        ib ^= 1;
#pragma unroll
        for (int j = 0; j < MAXR; ++j) rows[j] = nrows[j];
    }
}




}  // namespace
}  // namespace bk

using namespace bk;

extern "C" int bk_spmm_win_d(int n, int tile, int ntiles, int wmax, int nzmax, const int32_t* rp2,
                             const int32_t* code, const double* val2, const int32_t* wptr, const int32_t* wrow,
                             const double* x, int ldx, int k, double* y, int ldy, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    if (tile <= 0 || ntiles <= 0 || wmax <= 0 || nzmax < 0) return static_cast<int>(cudaErrorInvalidValue);
    // 16-byte row chunks: even leading dimensions and 16-byte aligned bases (the
    // blocks of the solver have ld % 8 == 0).  Views of X and Y that both start at an
    // odd column of their block are taken one column earlier — that column is
    // multiplied along and never stored; other misalignments are the caller's
    // fallback to bk_spmm_d.
    if ((ldx & 1) || (ldy & 1)) return static_cast<int>(cudaErrorMisalignedAddress);
    const unsigned mx = static_cast<unsigned>(reinterpret_cast<uintptr_t>(x) & 15);
    const unsigned my = static_cast<unsigned>(reinterpret_cast<uintptr_t>(y) & 15);
    int skip = 0;
    if (mx == 8 && my == 8) {
        skip = 1;
        --x;
        --y;
        ++k;
    } else if (mx || my) {
        return static_cast<int>(cudaErrorMisalignedAddress);
    }
    const cudaStream_t s = as_stream(stream);
    const int kr = (k + 1) & ~1;
    // one index slice (16-byte multiple); + 1 KB at the end so lanes past the last
    // slot's chunk read inside the allocation
    const size_t idx_bytes = (12 * static_cast<size_t>(nzmax) + 4 * (2 * static_cast<size_t>(tile) + 1) + 15) & ~size_t(15);
    static const int cps_env = [] {
        const char* e = getenv("BK_SPMM_WIN_CPS");  // CTAs per SM (tuning runs)
        return e ? max(1, atoi(e)) : 0;
    }();
    // column chunk: the widest (<= 128 columns, even) that leaves `cps` CTAs per SM
    // their window buffers
    auto chunk_for = [&](int cps) -> int {
        const size_t budget = (227 * 1024) / static_cast<size_t>(cps) - 1024;
        const size_t fixed = 2 * idx_bytes + 1024 + 16;
        if (budget <= fixed + 64) return 0;
        const size_t kmax = (budget - fixed) / (8 * static_cast<size_t>(wmax));
        return static_cast<int>((kmax < 128 ? kmax : size_t(128)) & ~size_t(1));
    };
    // three CTAs per SM measured best on config 2 (tiles of 64 rows: 4.0 TB/s at
    // k = 96 against 3.3 with two CTAs of wider chunks); fewer when the windows
    // are too large for that
    int cps = cps_env ? cps_env : 3, kcmax = chunk_for(cps);
    while (kcmax < 8 && cps > 1) kcmax = chunk_for(--cps);
    if (kcmax < 8) return static_cast<int>(cudaErrorInvalidValue);  // window too large for shared memory
    int nch = ceil_div(kr, kcmax);
    int kc = (ceil_div(kr, nch) + 3) & ~3;  // balanced chunks, whole 32-byte sectors when they fit
    if (kc > kcmax) kc = kcmax;
    // whole 16-column lane groups instead when that costs no extra chunk: the last,
    // narrower chunk then skips its empty groups (k = 69: 48 + 22 columns read 5 groups
    // per nonzero where 36 + 34 read 6)
    const int kc16 = (kc + 15) & ~15;
    if (kc16 <= kcmax && kc16 <= 64 && ceil_div(kr, kc16) == nch) kc = kc16;
    nch = ceil_div(kr, kc);
    const size_t smem = 16 + 8 * static_cast<size_t>(wmax) * kc + 2 * idx_bytes + 1024;
    const int grid = max(1, min(ntiles, kSMs * cps));
    auto launch = [&](auto kern) -> int {
        BK_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<grid, 256, smem, s>>>(n, tile, ntiles, wmax, nzmax, rp2, code, val2, wptr, wrow, x, ldx, k, kc, nch, y,
                                     ldy, skip);
        BK_LAUNCHED();
    };
    // lanes per row: 8 (four rows per warp) when that wastes fewer lanes on the chunk
    const int w16 = 32 * ceil_div(kc, 32) - kc, w8 = 16 * ceil_div(kc, 16) - kc;
    const bool l8 = kc <= 64 && w8 < w16;
    const int v = l8 ? ceil_div(kc, 16) : ceil_div(kc, 32);
#define BK_WIN_CASE(L, VV)                                                 \
    if (l8 == (L == 8) && v == VV)                                         \
        return launch(spmm_d_win_kernel<L, VV>);
    BK_WIN_CASE(8, 1)
    BK_WIN_CASE(8, 2)
    BK_WIN_CASE(8, 3)
    BK_WIN_CASE(8, 4)
    BK_WIN_CASE(16, 1)
    BK_WIN_CASE(16, 2)
    BK_WIN_CASE(16, 3)
    BK_WIN_CASE(16, 4)
#undef BK_WIN_CASE
    return static_cast<int>(cudaErrorInvalidValue);
}
