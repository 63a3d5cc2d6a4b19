// Host-side plan for the window-staged SpMM (K1w, bk_spmm_win_d): the rows of the
// full CSR are regrouped into tiles of graph-local rows and every tile gets its
// *window* — the tile's own rows followed by the distinct out-of-tile columns its
// rows reference (the halo).  The kernel stages a window's X rows in shared
// memory once and every nonzero of the tile then reads its X row on chip, so an
// X row travels from L2 to an SM once per tile that touches it instead of once
// per nonzero (7-point stencil, 64-row tiles: 2.4 row loads per matrix row
// instead of 7).  Each row keeps its nonzeros in their original order, so the
// product is bit-identical to the plain K1 (proj/src/kernel.cpp:8-33 restated as
// one pass over a full CSR).
#include <algorithm>
#include <cstring>
#include <new>

#include "../../../include/bk_kernels.h"
#include "host.hpp"

namespace b2 {

// Graph-local row order: rows are grouped into tiles of `tile` rows grown
// greedily over the sparsity graph — each step takes the unplaced row with the
// most neighbours already in the tile (oldest first among equals), which grows
// compact, cube-like blobs (7-point stencil, tile 64: 80 % of the nonzeros
// in-tile, against 64 % for breadth-first balls); a tile is seeded from the
// oldest row the previous tiles reached, so consecutive tiles are neighbours.
// Returns the order (ordered index -> row) and the fraction of nonzeros whose
// column lies in the row's own tile.
double cluster_rows(int n, const int32_t* rp, const int32_t* col, int tile, std::vector<int32_t>& order) {
    order.clear();
    order.reserve(n);
    std::vector<int32_t> tile_of(static_cast<size_t>(n), -1), gain(static_cast<size_t>(n), 0);
    std::vector<int32_t> frontier;  // global FIFO of reached rows (may repeat)
    size_t fhead = 0;
    int next_seed = 0;
    constexpr int kB = 32;  // gain buckets (gains >= kB - 1 share the last)
    std::vector<int32_t> bucket[kB];
    size_t bhead[kB];
    std::vector<int32_t> touched;
    while (static_cast<int>(order.size()) < n) {
        const int t = static_cast<int>(order.size()) / tile;
        const size_t start = order.size();
        for (int g = 0; g < kB; ++g) {
            bucket[g].clear();
            bhead[g] = 0;
        }
        touched.clear();
        auto seed = [&]() {
            while (fhead < frontier.size() && tile_of[frontier[fhead]] >= 0) ++fhead;
            if (fhead < frontier.size()) return frontier[fhead++];
            while (next_seed < n && tile_of[next_seed] >= 0) ++next_seed;
            return next_seed < n ? next_seed : -1;
        };
        while (order.size() - start < static_cast<size_t>(tile)) {
            int u = -1;
            for (int g = kB - 1; g > 0 && u < 0; --g) {
                auto& b = bucket[g];
                while (bhead[g] < b.size() &&
                       (tile_of[b[bhead[g]]] >= 0 || std::min(gain[b[bhead[g]]], kB - 1) != g))
                    ++bhead[g];
                if (bhead[g] < b.size()) u = b[bhead[g]++];
            }
            if (u < 0 && (u = seed()) < 0) break;
            tile_of[u] = t;
            order.push_back(u);
            for (int32_t p = rp[u]; p < rp[u + 1]; ++p) {
                const int c = col[p];
                if (tile_of[c] >= 0) continue;
                if (gain[c]++ == 0) touched.push_back(c);
                bucket[std::min(gain[c], kB - 1)].push_back(c);
            }
        }
        for (int c : touched) {
            if (tile_of[c] < 0) frontier.push_back(c);
            gain[c] = 0;
        }
    }
    int64_t in = 0;
    for (int r = 0; r < n; ++r)
        for (int32_t p = rp[r]; p < rp[r + 1]; ++p) in += tile_of[col[p]] == tile_of[r];
    return rp[n] ? static_cast<double>(in) / rp[n] : 0.0;
}

// Windows over a given row order.  Slot s < rows(t) of tile t is the tile's own
// ordered row t*tile + s; the halo slots follow in ascending column order.
void build_windows(int n, const int32_t* rp, const int32_t* col, const double* val, int per, int tile,
                   const std::vector<int32_t>& order, WindowPlan& w) {
    const int64_t nnz = rp[n];
    w.n = n;
    w.tile = tile;
    w.ntiles = (n + tile - 1) / tile;
    w.rp2.assign(static_cast<size_t>(n) + 1, 0);
    w.code.resize(static_cast<size_t>(nnz));
    w.val2.resize(static_cast<size_t>(nnz) * per);
    w.wptr.assign(static_cast<size_t>(w.ntiles) + 1, 0);
    w.wrow.clear();
    w.wrow.reserve(static_cast<size_t>(n) * 2);
    std::vector<int32_t> pos(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) pos[order[i]] = i;
    std::vector<int32_t> slot_of(static_cast<size_t>(n), -1);  // column -> slot in the current window
    std::vector<int32_t> halo;
    int64_t q = 0;
    w.wmax = 0;
    w.nzmax = 0;
    for (int t = 0; t < w.ntiles; ++t) {
        const int i0 = t * tile, nr = std::min(tile, n - i0);
        halo.clear();
        for (int i = i0; i < i0 + nr; ++i) {
            const int r = order[i];
            for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
                const int c = col[p];
                if (pos[c] / tile != t && slot_of[c] < 0) {
                    slot_of[c] = 0;
                    halo.push_back(c);
                }
            }
        }
        std::sort(halo.begin(), halo.end());
        for (size_t h = 0; h < halo.size(); ++h) slot_of[halo[h]] = nr + static_cast<int>(h);
        for (int i = i0; i < i0 + nr; ++i) w.wrow.push_back(order[i]);
        w.wrow.insert(w.wrow.end(), halo.begin(), halo.end());
        w.wptr[t + 1] = static_cast<int32_t>(w.wrow.size());
        const int64_t q0 = q;
        for (int i = i0; i < i0 + nr; ++i) {
            const int r = order[i];
            for (int32_t p = rp[r]; p < rp[r + 1]; ++p, ++q) {
                const int c = col[p];
                w.code[q] = pos[c] / tile == t ? pos[c] - i0 : slot_of[c];
                for (int u = 0; u < per; ++u) w.val2[q * per + u] = val[static_cast<int64_t>(p) * per + u];
            }
            w.rp2[i + 1] = static_cast<int32_t>(q);
        }
        for (int c : halo) slot_of[c] = -1;
        w.wmax = std::max(w.wmax, nr + static_cast<int>(halo.size()));
        w.nzmax = std::max<int>(w.nzmax, static_cast<int>(q - q0));
    }
    w.loads_per_row = n ? static_cast<double>(w.wrow.size()) / n : 0.0;
}

// Plan with `tile_req` rows per tile (0: 64, the size measured best on the 7-point
// stencil) and decide whether K1w pays: the windows must load well under the X
// rows the nonzeros gather (else the graph has too little locality — config 3's
// random columns), and the largest window must leave three CTAs per SM a chunk
// of >= 32 columns (bk_spmm_win.cu; config 4's 25-point stencil of A^2 has
// windows of 300-800 rows and stays on the plain kernel).  wcap > 0 overrides
// the shared-memory rule with a plain slot cap (tests, tuning runs).
bool plan_windows(int n, const int32_t* rp, const int32_t* col, const double* val, int per, int tile_req,
                  int wcap, WindowPlan& w) {
    if (n <= 0 || rp[n] <= 0) return false;
    const double nnz_per_row = static_cast<double>(rp[n]) / n;
    const int tile = tile_req > 0 ? tile_req : 64;
    if (n < 4 * tile) return false;
    std::vector<int32_t> order;
    cluster_rows(n, rp, col, tile, order);
    build_windows(n, rp, col, val, per, tile, order, w);
    const size_t idx = (12 * static_cast<size_t>(w.nzmax) + 4 * (2 * static_cast<size_t>(tile) + 1) + 15) & ~size_t(15);
    const size_t need = 16 + 8 * static_cast<size_t>(w.wmax) * 32 + 2 * idx + 1024;
    const bool fits = wcap > 0 ? w.wmax <= wcap : need <= (227 * 1024) / 3 - 1024;
    return fits && w.loads_per_row <= 0.55 * nnz_per_row;
}

}  // namespace b2

// ---- C ABI (host side of K1w; tests and tools build a plan, upload its arrays
// and call bk_spmm_win_d) ----
using b2::WindowPlan;

extern "C" int bk_spmm_win_plan(int n, const int32_t* rp, const int32_t* col, const double* val, int tile,
                                int wcap, void** plan) {
    if (!plan || !rp || !col || !val || n <= 0 || wcap < 0 || tile < 0) return 1;
    *plan = nullptr;
    auto* w = new (std::nothrow) WindowPlan();
    if (!w) return 2;
    try {
        w->ok = b2::plan_windows(n, rp, col, val, 1, tile, wcap, *w);
    } catch (...) {
        delete w;
        return 2;
    }
    *plan = w;
    return 0;
}

extern "C" int bk_spmm_win_plan_info(const void* plan, int* ok, int* tile, int* ntiles, int* wmax, int* nzmax,
                                     double* loads_per_row) {
    if (!plan) return 1;
    const auto* w = static_cast<const WindowPlan*>(plan);
    if (ok) *ok = w->ok ? 1 : 0;
    if (tile) *tile = w->tile;
    if (ntiles) *ntiles = w->ntiles;
    if (wmax) *wmax = w->wmax;
    if (nzmax) *nzmax = w->nzmax;
    if (loads_per_row) *loads_per_row = w->loads_per_row;
    return 0;
}

extern "C" int bk_spmm_win_plan_arrays(const void* plan, const int32_t** rp2, const int32_t** code,
                                       const double** val2, const int32_t** wptr, const int32_t** wrow,
                                       int64_t* wrow_len) {
    if (!plan) return 1;
    const auto* w = static_cast<const WindowPlan*>(plan);
    if (rp2) *rp2 = w->rp2.data();
    if (code) *code = w->code.data();
    if (val2) *val2 = w->val2.data();
    if (wptr) *wptr = w->wptr.data();
    if (wrow) *wrow = w->wrow.data();
    if (wrow_len) *wrow_len = static_cast<int64_t>(w->wrow.size());
    return 0;
}

extern "C" void bk_spmm_win_plan_free(void* plan) { delete static_cast<WindowPlan*>(plan); }
