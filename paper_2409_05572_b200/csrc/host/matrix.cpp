// Matrix handle: lower-CSR storage, generators, norm estimate, Matrix Market
// ingest/export and the cached device copy (full CSR) used by the SpMM kernel.
// Reference: proj/src/matio.{hpp,cpp}, proj/src/kernel.cpp:166-196.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <future>
#include <mutex>
#include <thread>
#include <vector>
#include <fstream>
#include <sstream>
#include <unordered_map>

#include "host.hpp"

namespace b2 {

void cuda_check(int code, const char* what) {
    if (code != 0)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(code)));
}

// ---------------------------------------------------------------- device block cache
// Solves allocate their S / AS / work blocks (GBs) on entry and release them on
// exit; cudaMalloc/cudaFree of that much costs 0.05-0.25 s per solve and
// cudaFree synchronises the device.  Released blocks are kept per device and
// reused best-fit (within 2x) by the next solve; on an allocation failure the
// cache is emptied and the allocation retried.  BLOCKEIG_NO_CACHE=1 disables it;
// beig_release_device_cache() empties it.  A block is only returned after its
// owner synchronised its stream (Engine's destructor), so reuse is race-free.
namespace {
struct CachedBlock {
    void* p;
    size_t bytes;
    int dev;
};
// never destroyed: handles released during process exit still return blocks safely
std::mutex& g_cache_mu = *new std::mutex;
std::vector<CachedBlock>& g_cache = *new std::vector<CachedBlock>;
const bool g_cache_off = std::getenv("BLOCKEIG_NO_CACHE") != nullptr;

void* cache_take(size_t bytes, size_t* got, int dev) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t best = g_cache.size();
    for (size_t i = 0; i < g_cache.size(); ++i) {
        const auto& b = g_cache[i];
        if (b.dev == dev && b.bytes >= bytes && b.bytes <= 2 * bytes &&
            (best == g_cache.size() || b.bytes < g_cache[best].bytes))
            best = i;
    }
    if (best == g_cache.size()) return nullptr;
    void* p = g_cache[best].p;
    *got = g_cache[best].bytes;
    g_cache.erase(g_cache.begin() + static_cast<std::ptrdiff_t>(best));
    return p;
}

void cache_drop_all() {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& b : g_cache) {
        cudaSetDevice(b.dev);
        cudaFree(b.p);
    }
    cudaSetDevice(cur);
    g_cache.clear();
}
}  // namespace

void release_device_cache() { cache_drop_all(); }

DevMem::~DevMem() {
    if (!p_) return;
    if (g_cache_off) {
        cudaFree(p_);
        return;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.push_back({p_, bytes_, dev_});
}

void DevMem::alloc(size_t bytes) {
    if (p_) {
        DevMem old;
        old.p_ = p_;
        old.bytes_ = bytes_;
        old.dev_ = dev_;
        p_ = nullptr;
        bytes_ = 0;
    }
    if (bytes == 0) return;
    cuda_check(cudaGetDevice(&dev_), "cudaGetDevice");
    if (!g_cache_off) {
        size_t got = 0;
        if (void* p = cache_take(bytes, &got, dev_)) {
            p_ = p;
            bytes_ = got;
            return;
        }
    }
    cudaError_t e = cudaMalloc(&p_, bytes);
    if (e == cudaErrorMemoryAllocation && !g_cache_off) {
        (void)cudaGetLastError();
        cache_drop_all();
        e = cudaMalloc(&p_, bytes);
    }
    cuda_check(e, "cudaMalloc");
    bytes_ = bytes;
}

// ---------------------------------------------------------------- SparseSym

SparseSym::SparseSym()
    : n_(0), complex_(false), rp_(1, 0),
      norm_cache_(std::make_shared<std::atomic<double>>(-1.0)), dev_(std::make_shared<DevCache>()) {}

SparseSym::SparseSym(int n, std::vector<int64_t> rp, std::vector<int> col, std::vector<double> val,
                     bool complex_values)
    : n_(n), complex_(complex_values), rp_(std::move(rp)), col_(std::move(col)), val_(std::move(val)),
      norm_cache_(std::make_shared<std::atomic<double>>(-1.0)), dev_(std::make_shared<DevCache>()) {
    const size_t per = complex_ ? 2 : 1;
    if (n_ < 0 || rp_.size() != static_cast<size_t>(n_) + 1 || val_.size() != per * col_.size() ||
        rp_.front() != 0 || rp_.back() != static_cast<int64_t>(col_.size()))
        throw std::invalid_argument("SparseSym: inconsistent CSR arrays");
    for (int r = 0; r < n_; ++r) {
        if (rp_[r + 1] < rp_[r]) throw std::invalid_argument("SparseSym: inconsistent CSR arrays");
        int prev = -1;
        for (int64_t p = rp_[r]; p < rp_[r + 1]; ++p) {
            const int c = col_[p];
            if (c < 0 || c > r || c <= prev)
                throw std::invalid_argument("SparseSym: columns must be strictly increasing and <= row");
            prev = c;
            if (complex_ && c == r && val_[2 * p + 1] != 0.0)
                throw std::invalid_argument("Hermitian matrix needs a real diagonal");
        }
    }
    if (static_cast<int64_t>(col_.size()) * 2 >= (int64_t{1} << 31))
        throw std::invalid_argument("matrix too large for int32 device indices");
}

double SparseSym::diagonal(int i) const {
    for (int64_t p = rp_[i + 1] - 1; p >= rp_[i]; --p) {
        if (col_[p] == i) return complex_ ? val_[2 * p] : val_[p];
        if (col_[p] < i) break;
    }
    return 0.0;
}

namespace {

// reference spmv (kernel.cpp:8-26): lower CSR, mirrored scatter, fixed order
void host_spmv(const SparseSym& a, const std::vector<double>& x, std::vector<double>& y) {
    const int n = a.rows();
    const auto& rp = a.row_ptr();
    const auto& col = a.col();
    const auto& val = a.val();
    y.assign(x.size(), 0.0);
    if (!a.is_complex()) {
        for (int r = 0; r < n; ++r) {
            double acc = 0.0;
            const double xr = x[r];
            for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
                const int c = col[p];
                const double v = val[p];
                acc += v * x[c];
                if (c != r) y[c] += v * xr;
            }
            y[r] += acc;
        }
        return;
    }
    for (int r = 0; r < n; ++r) {
        double ar = 0.0, ai = 0.0;
        const double xr = x[2 * r], xi = x[2 * r + 1];
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
            const int c = col[p];
            const double vr = val[2 * p], vi = val[2 * p + 1];
            ar += vr * x[2 * c] - vi * x[2 * c + 1];
            ai += vr * x[2 * c + 1] + vi * x[2 * c];
            if (c != r) {  // conj(v) * x[r]
                y[2 * c] += vr * xr + vi * xi;
                y[2 * c + 1] += vr * xi - vi * xr;
            }
        }
        y[2 * r] += ar;
        y[2 * r + 1] += ai;
    }
}

// complex: |z|^2 = re^2 + im^2 formed per element, then accumulated (the
// oracle's nrm2 over std::complex entries), so the estimate is bit-identical
double host_nrm2(const std::vector<double>& v, bool cplx) {
    double s = 0.0;
    if (!cplx) {
        for (double x : v) s += x * x;
    } else {
        for (size_t i = 0; i + 1 < v.size(); i += 2) s += v[i] * v[i] + v[i + 1] * v[i + 1];
    }
    return std::sqrt(s);
}

}  // namespace

// kernel.cpp:174-196 — computed once per handle on the host with the
// reference's seeded start and loop order, shared by every solve on the
// handle (and bit-identical to the CPU oracle's value).
double SparseSym::norm_est() const {
    const double cached = norm_cache_->load(std::memory_order_relaxed);
    if (cached >= 0.0) return cached;
    if (n_ == 0) return 0.0;
    std::mt19937_64 rng(0x9e3779b97f4a7c15ULL);
    std::normal_distribution<double> dist(0.0, 1.0);
    std::vector<double> v(static_cast<size_t>(n_) * (complex_ ? 2 : 1));
    for (auto& x : v) x = dist(rng);
    double nrm = host_nrm2(v, complex_);
    if (nrm == 0.0) return 0.0;
    for (auto& x : v) x /= nrm;
    std::vector<double> w, t;
    // real: the full (both triangles) CSR, each row [lower entries, then the
    // mirrored upper ones, columns ascending] summed left to right from 0 —
    // exactly the order in which host_spmv's row scan and scatter build y[r]
    // (acc over the lower row, then y[r] += v x[r'] for each later row r'), so
    // the rows can be split over threads and the estimate stays bit-identical
    const bool par = !complex_ && n_ >= 65536;
    if (par) {
        // one team of host threads for the whole estimate (spin barrier between
        // phases, instead of threads spawned per product: 63 -> 48 ms at config 2); the
        // squared norm stays a serial sum on thread 0 and the normalisation an
        // exact division per entry: the reference loop's values
        const FullCsr& fc = full_csr();
        const int nthr = std::max(1, std::min(8, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<double> tt(v.size()), ww(v.size());
        std::atomic<int> arrived{0}, phase{0};
        auto barrier = [&]() {
            const int ph = phase.load(std::memory_order_acquire);
            if (arrived.fetch_add(1, std::memory_order_acq_rel) == nthr - 1) {
                arrived.store(0, std::memory_order_relaxed);
                phase.store(ph + 1, std::memory_order_release);
            } else {
                while (phase.load(std::memory_order_acquire) == ph) std::this_thread::yield();
            }
        };
        double shared_nrm = 0.0, est_t = 0.0;
        auto team = [&](int id) {
            const int r0 = static_cast<int>(static_cast<int64_t>(n_) * id / nthr);
            const int r1 = static_cast<int>(static_cast<int64_t>(n_) * (id + 1) / nthr);
            auto rows = [&](const std::vector<double>& x, std::vector<double>& y) {
                for (int r = r0; r < r1; ++r) {
                    double acc = 0.0;
                    for (int32_t p = fc.rp[r]; p < fc.rp[r + 1]; ++p) acc += fc.val[p] * x[fc.col[p]];
                    y[r] = acc;
                }
            };
            for (int it = 0; it < 30; ++it) {
                rows(v, tt);
                barrier();
                rows(tt, ww);
                barrier();
                if (id == 0) shared_nrm = host_nrm2(ww, false);
                barrier();
                const double nr = shared_nrm;
                if (nr == 0.0) return;
                for (int r = r0; r < r1; ++r) v[r] = ww[r] / nr;
                barrier();
            }
            rows(v, tt);
            barrier();
            if (id == 0) est_t = host_nrm2(tt, false);
        };
        std::vector<std::thread> th;
        for (int i = 1; i < nthr; ++i) th.emplace_back(team, i);
        team(0);
        for (auto& x : th) x.join();
        const double res = shared_nrm == 0.0 ? 0.0 : est_t;
        norm_cache_->store(res, std::memory_order_relaxed);
        return res;
    }
    for (int it = 0; it < 30; ++it) {
        host_spmv(*this, v, t);
        host_spmv(*this, t, w);
        nrm = host_nrm2(w, complex_);
        if (nrm == 0.0) {
            norm_cache_->store(0.0, std::memory_order_relaxed);
            return 0.0;
        }
        for (size_t i = 0; i < v.size(); ++i) v[i] = w[i] / nrm;
    }
    host_spmv(*this, v, t);
    const double est = host_nrm2(t, complex_);
    norm_cache_->store(est, std::memory_order_relaxed);
    return est;
}

// Expand the lower triangle to full CSR (int32) and upload once per
// (device, sign); the upper entries are the mirrored (conjugated) lower ones.
const SparseSym::FullCsr& SparseSym::full_csr() const {
    std::lock_guard<std::mutex> lk(dev_->full_mu);
    if (dev_->full_ready) return dev_->full;
    auto& frp = dev_->full.rp;
    auto& fcol = dev_->full.col;
    auto& fval = dev_->full.val;
    const double sgn = 1.0;
    const int per = complex_ ? 2 : 1;
    std::vector<int32_t> cnt(static_cast<size_t>(n_) + 1, 0);
    for (int r = 0; r < n_; ++r)
        for (int64_t p = rp_[r]; p < rp_[r + 1]; ++p) {
            cnt[r + 1]++;
            if (col_[p] != r) cnt[col_[p] + 1]++;
        }
    for (int r = 0; r < n_; ++r) cnt[r + 1] += cnt[r];
    const int64_t nnz = cnt[n_];
    frp = cnt;
    fcol.assign(static_cast<size_t>(nnz), 0);
    fval.assign(static_cast<size_t>(nnz) * per, 0.0);
    // rows in order: a row's lower entries, then its upper entries (c > r), which
    // are later rows' lower entries — gathered by a counting-sort transpose
    // (scanning rows in increasing order keeps each row's upper part sorted)
    std::vector<int64_t> uptr(static_cast<size_t>(n_) + 1, 0);
    for (int r = 0; r < n_; ++r)
        for (int64_t p = rp_[r]; p < rp_[r + 1]; ++p)
            if (col_[p] != r) uptr[col_[p] + 1]++;
    for (int r = 0; r < n_; ++r) uptr[r + 1] += uptr[r];
    std::vector<int64_t> usrc(static_cast<size_t>(uptr[n_]));  // source entry p of each upper entry
    std::vector<int32_t> urow(static_cast<size_t>(uptr[n_]));
    {
        std::vector<int64_t> fill(uptr.begin(), uptr.end() - 1);
        for (int r = 0; r < n_; ++r)
            for (int64_t p = rp_[r]; p < rp_[r + 1]; ++p)
                if (col_[p] != r) {
                    const int64_t q = fill[col_[p]]++;
                    usrc[q] = p;
                    urow[q] = r;
                }
    }
    for (int r = 0; r < n_; ++r) {
        int32_t q = cnt[r];
        for (int64_t p = rp_[r]; p < rp_[r + 1]; ++p) {
            fcol[q] = col_[p];
            for (int t = 0; t < per; ++t) fval[static_cast<size_t>(q) * per + t] = sgn * val_[p * per + t];
            ++q;
        }
        for (int64_t u = uptr[r]; u < uptr[r + 1]; ++u) {  // entry (r, c) = conj(A(c, r)), c > r
            const int64_t p = usrc[u];
            fcol[q] = urow[u];
            fval[static_cast<size_t>(q) * per] = sgn * val_[p * per];
            if (complex_) fval[static_cast<size_t>(q) * per + 1] = -sgn * val_[p * per + 1];
            ++q;
        }
    }
    dev_->full_ready = true;
    return dev_->full;
}

const DeviceCsr& SparseSym::device_csr(int device, bool negate) const {
    std::lock_guard<std::mutex> lk(dev_->mu);
    for (auto& e : dev_->entries)
        if (e->device == device && e->negated == negate) return *e;
    const FullCsr& full = full_csr();
    const std::vector<int32_t>& frp = full.rp;
    const std::vector<int32_t>& fcol = full.col;
    std::vector<double> neg;
    if (negate) {  // M = -A (largest eigenpairs)
        neg.resize(full.val.size());
        for (size_t i = 0; i < neg.size(); ++i) neg[i] = -full.val[i];
    }
    const std::vector<double>& fval = negate ? neg : full.val;
    const int64_t nnz = frp[n_];
    auto e = std::make_unique<DeviceCsr>();
    e->device = device;
    e->n = n_;
    e->nnz_full = nnz;
    e->negated = negate;
    int prev = 0;
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    e->row_ptr.alloc(sizeof(int32_t) * frp.size());
    e->col.alloc(sizeof(int32_t) * std::max<size_t>(fcol.size(), 1));
    e->val.alloc(sizeof(double) * std::max<size_t>(fval.size(), 1));
    cuda_check(cudaMemcpy(e->row_ptr.as<void>(), frp.data(), sizeof(int32_t) * frp.size(), cudaMemcpyHostToDevice), "upload");
    if (nnz) {
        cuda_check(cudaMemcpy(e->col.as<void>(), fcol.data(), sizeof(int32_t) * fcol.size(), cudaMemcpyHostToDevice), "upload");
        cuda_check(cudaMemcpy(e->val.as<void>(), fval.data(), sizeof(double) * fval.size(), cudaMemcpyHostToDevice), "upload");
    }
    // window-staged SpMM plan (K1w): clustering, windows and their upload run on a
    // host thread so a fresh handle's first solve starts at once on the plain
    // kernel and switches over when the plan is ready (bit-identical products).
    // Real matrices of >= 65536 rows; BLOCKEIG_SPMM_WIN=0 keeps the plain kernel.
    // (BLOCKEIG_SPMM_WIN=2: wait for the plan here — tests and kernel timing runs)
    static const int win_mode = [] {
        const char* v = std::getenv("BLOCKEIG_SPMM_WIN");
        return v ? std::atoi(v) : 1;
    }();
    const bool win_off = win_mode == 0;
    if (!complex_ && !win_off && n_ >= 65536 && nnz) {
        DeviceCsr* ep = e.get();
        const FullCsr* fp = &full;  // owned by dev_, which outlives the entry
        const bool neg_vals = negate;
        ep->win_state.store(1, std::memory_order_release);
        ep->win_job = std::async(std::launch::async, [ep, fp, neg_vals, device] {
            try {
                const auto t0 = std::chrono::steady_clock::now();
                WindowPlan w;
                const int n = static_cast<int>(fp->rp.size()) - 1;
                std::vector<double> nv;
                if (neg_vals) {
                    nv.resize(fp->val.size());
                    for (size_t i = 0; i < nv.size(); ++i) nv[i] = -fp->val[i];
                }
                const bool ok = plan_windows(n, fp->rp.data(), fp->col.data(), neg_vals ? nv.data() : fp->val.data(), 1,
                                             0, 0, w);
                if (!ok) {
                    ep->win_state.store(3, std::memory_order_release);
                    return;
                }
                cuda_check(cudaSetDevice(device), "cudaSetDevice");
                cudaStream_t st = nullptr;
                cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
                auto up = [&](DevMem& d, const void* src, size_t bytes) {
                    d.alloc(bytes);
                    cuda_check(cudaMemcpyAsync(d.p(), src, bytes, cudaMemcpyHostToDevice, st), "upload");
                };
                DeviceCsr::Win& o = ep->win;
                up(o.rp2, w.rp2.data(), sizeof(int32_t) * w.rp2.size());
                up(o.code, w.code.data(), sizeof(int32_t) * w.code.size());
                up(o.val2, w.val2.data(), sizeof(double) * w.val2.size());
                up(o.wptr, w.wptr.data(), sizeof(int32_t) * w.wptr.size());
                up(o.wrow, w.wrow.data(), sizeof(int32_t) * w.wrow.size());
                const cudaError_t se = cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
                cuda_check(se, "upload");
                o.tile = w.tile;
                o.ntiles = w.ntiles;
                o.wmax = w.wmax;
                o.nzmax = w.nzmax;
                o.loads_per_row = w.loads_per_row;
                o.plan_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                ep->win_state.store(2, std::memory_order_release);
            } catch (...) {  // no plan: the plain kernel stays in use
                ep->win_state.store(3, std::memory_order_release);
            }
        });
        if (win_mode == 2) ep->win_job.wait();
    }
    cudaSetDevice(prev);
    dev_->entries.push_back(std::move(e));
    return *dev_->entries.back();
}

// ---------------------------------------------------------------- generators

namespace {
struct Entry {
    int r, c;
    double v;
};
SparseSym from_entries(int n, std::vector<Entry>& es) {
    std::sort(es.begin(), es.end(), [](const Entry& a, const Entry& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
    std::vector<int> col(es.size());
    std::vector<double> val(es.size());
    for (size_t i = 0; i < es.size(); ++i) {
        rp[es[i].r + 1]++;
        col[i] = es[i].c;
        val[i] = es[i].v;
    }
    for (int r = 0; r < n; ++r) rp[r + 1] += rp[r];
    return SparseSym(n, std::move(rp), std::move(col), std::move(val));
}

std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> out(1);
    for (char ch : s) {
        if (ch == ',') out.emplace_back();
        else out.back() += ch;
    }
    return out;
}

int to_int(const std::string& s) {
    size_t pos = 0;
    const int v = std::stoi(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("bad integer '" + s + "' in spec");
    return v;
}
double to_double(const std::string& s) {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("bad number '" + s + "' in spec");
    return v;
}

SparseSym diag_from(const std::vector<double>& v) {
    const int n = static_cast<int>(v.size());
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1);
    std::vector<int> col(static_cast<size_t>(n));
    for (int i = 0; i <= n; ++i) rp[i] = i;
    for (int i = 0; i < n; ++i) col[i] = i;
    return SparseSym(n, std::move(rp), std::move(col), v);
}
}  // namespace

// matio.cpp:246-290: "laplacian1d:N", "diag:v1,...", "diag-geom:N,RATIO"
SparseSym gen_from_spec(const std::string& spec) {
    const size_t colon = spec.find(':');
    if (colon == std::string::npos)
        throw std::invalid_argument("generator spec needs 'name:args', got '" + spec + "'");
    const std::string name = spec.substr(0, colon), args = spec.substr(colon + 1);
    if (name == "laplacian1d") {
        const int n = to_int(args);
        if (n < 1) throw std::invalid_argument("gen_laplacian_1d: n must be positive");
        std::vector<Entry> es;
        for (int i = 0; i < n; ++i) {
            if (i > 0) es.push_back({i, i - 1, -1.0});
            es.push_back({i, i, 2.0});
        }
        return from_entries(n, es);
    }
    if (name == "diag") {
        std::vector<double> v;
        for (const auto& t : split_commas(args)) v.push_back(to_double(t));
        return diag_from(v);
    }
    if (name == "diag-geom") {
        const auto parts = split_commas(args);
        if (parts.size() != 2) throw std::invalid_argument("diag-geom needs 'diag-geom:n,ratio'");
        const int n = to_int(parts[0]);
        const double ratio = to_double(parts[1]);
        if (n < 1) throw std::invalid_argument("gen_diag_geometric: n must be positive");
        if (!(ratio > 0)) throw std::invalid_argument("gen_diag_geometric: ratio must be positive");
        std::vector<double> v(static_cast<size_t>(n));
        double x = 1.0;
        for (int i = 0; i < n; ++i, x *= ratio) v[i] = x;
        return diag_from(v);
    }
    throw std::invalid_argument("unknown generator '" + name + "'");
}

double spd_shift_value(double lambda1) { return lambda1 <= 0.0 ? 1.05 * lambda1 : 0.0; }

SparseSym apply_spd_shift(const SparseSym& a, double lambda1) {
    if (a.is_complex()) throw std::invalid_argument("spd_shift: real matrices only");
    const double shift = spd_shift_value(lambda1);
    if (shift == 0.0) return a;
    std::vector<Entry> es;
    for (int r = 0; r < a.rows(); ++r) {
        bool has = false;
        for (int64_t p = a.row_ptr()[r]; p < a.row_ptr()[r + 1]; ++p) {
            double v = a.val()[p];
            if (a.col()[p] == r) {
                v -= shift;
                has = true;
            }
            es.push_back({r, a.col()[p], v});
        }
        if (!has) es.push_back({r, r, -shift});
    }
    return from_entries(a.rows(), es);
}

// ---------------------------------------------------------------- Matrix Market
// Same acceptance rules as proj/src/matio.cpp:89-184: 'matrix coordinate',
// real|integer, symmetric (lower triangle) | general (numerically symmetric
// within 1e-12 relative); ParseError carries the offending line.

namespace {
std::string lowered(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}
bool content_line(std::istream& in, std::string& line, long& no) {
    while (std::getline(in, line)) {
        ++no;
        const size_t i = line.find_first_not_of(" \t\r\n");
        if (i == std::string::npos || line[i] == '%') continue;
        return true;
    }
    return false;
}
}  // namespace

SparseSym parse_matrix_market_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open '" + path + "'");
    std::string line;
    long no = 0;
    if (!std::getline(in, line)) throw ParseError("empty input", 1);
    ++no;
    std::istringstream hs(line);
    std::string banner, object, format, field, sym;
    hs >> banner >> object >> format >> field >> sym;
    if (banner != "%%MatrixMarket") throw ParseError("missing %%MatrixMarket banner", no);
    if (lowered(object) != "matrix" || lowered(format) != "coordinate")
        throw ParseError("only 'matrix coordinate' inputs are supported", no);
    field = lowered(field);
    sym = lowered(sym);
    // extension: "complex hermitian" (lower triangle, real diagonal) and
    // "complex general" (must be Hermitian) build a complex Hermitian matrix
    const bool cplx = field == "complex";
    if (field != "real" && field != "integer" && !cplx) throw ParseError("unsupported field '" + field + "'", no);
    if (cplx ? (sym != "hermitian" && sym != "general") : (sym != "symmetric" && sym != "general"))
        throw ParseError("unsupported symmetry '" + sym + "'", no);
    const bool general = sym == "general";
    if (!content_line(in, line, no)) throw ParseError("missing size line", no + 1);
    long rows = 0, cols = 0, nnz = 0;
    {
        std::istringstream ss(line);
        std::string rest;
        if (!(ss >> rows >> cols >> nnz)) throw ParseError("malformed size line", no);
        if (ss >> rest) throw ParseError("trailing tokens on size line", no);
    }
    if (rows != cols) throw ParseError("matrix is not square", no);
    if (rows < 0 || nnz < 0) throw ParseError("negative dimensions", no);
    struct Pair {
        double lo = 0, up = 0, lo_im = 0, up_im = 0;
        bool has_lo = false, has_up = false;
        long ln_lo = 0, ln_up = 0;
    };
    std::unordered_map<int64_t, Pair> slots;
    std::vector<int64_t> order;
    for (long e = 0; e < nnz; ++e) {
        if (!content_line(in, line, no))
            throw ParseError("unexpected end of input, expected " + std::to_string(nnz) + " entries, got " +
                                 std::to_string(e),
                             no + 1);
        std::istringstream ss(line);
        long i, j;
        double v, vi = 0.0;
        std::string rest;
        if (!(ss >> i >> j >> v) || (cplx && !(ss >> vi)))
            throw ParseError(cplx ? "malformed entry (need 'i j re im')" : "malformed entry (need 'i j value')", no);
        if (ss >> rest) throw ParseError("trailing tokens on entry line", no);
        if (i < 1 || i > rows || j < 1 || j > cols) throw ParseError("index out of range", no);
        if (!std::isfinite(v) || !std::isfinite(vi)) throw ParseError("non-finite value", no);
        const bool low = i >= j;
        if (!general && !low)
            throw ParseError(cplx ? "hermitian input must store the lower triangle"
                                  : "symmetric input must store the lower triangle", no);
        if (cplx && i == j && vi != 0.0) throw ParseError("hermitian diagonal must be real", no);
        const int64_t r = (low ? i : j) - 1, c = (low ? j : i) - 1;
        const int64_t key = r * rows + c;
        auto it = slots.find(key);
        if (it == slots.end()) {
            it = slots.emplace(key, Pair{}).first;
            order.push_back(key);
        }
        Pair& s = it->second;
        if (low) {
            if (s.has_lo) throw ParseError("duplicate entry", no);
            s.lo = v, s.lo_im = vi, s.has_lo = true, s.ln_lo = no;
        } else {
            if (s.has_up) throw ParseError("duplicate entry", no);
            s.up = v, s.up_im = vi, s.has_up = true, s.ln_up = no;
        }
    }
    std::sort(order.begin(), order.end());
    if (cplx) {  // Hermitian: the mirror of (r, c) holds conj(a_rc)
        std::vector<int64_t> rp(static_cast<size_t>(rows) + 1, 0);
        std::vector<int> col;
        std::vector<double> val;
        col.reserve(order.size());
        val.reserve(2 * order.size());
        for (int64_t key : order) {
            const Pair& s = slots[key];
            const int r = static_cast<int>(key / rows), c = static_cast<int>(key % rows);
            if (r != c && general) {
                const std::string where = "(" + std::to_string(r + 1) + "," + std::to_string(c + 1) + ")";
                if (!s.has_lo || !s.has_up)
                    throw ParseError("general input is not hermitian: entry " + where + " lacks its mirror",
                                     s.has_lo ? s.ln_lo : s.ln_up);
                const double scale = std::max({std::hypot(s.lo, s.lo_im), std::hypot(s.up, s.up_im), 1e-300});
                if (std::hypot(s.lo - s.up, s.lo_im + s.up_im) > 1e-12 * scale)
                    throw ParseError("general input is not hermitian: entry " + where + " mismatches its mirror",
                                     s.ln_up);
            }
            if (r == c && general && s.lo_im != 0.0) throw ParseError("hermitian diagonal must be real", s.ln_lo);
            rp[r + 1]++;
            col.push_back(c);
            val.push_back(s.lo);
            val.push_back(s.lo_im);
        }
        for (long r = 0; r < rows; ++r) rp[r + 1] += rp[r];
        return SparseSym(static_cast<int>(rows), std::move(rp), std::move(col), std::move(val), true);
    }
    std::vector<Entry> es;
    es.reserve(order.size());
    for (int64_t key : order) {
        const Pair& s = slots[key];
        const int r = static_cast<int>(key / rows), c = static_cast<int>(key % rows);
        if (r != c && general) {
            const std::string where = "(" + std::to_string(r + 1) + "," + std::to_string(c + 1) + ")";
            if (!s.has_lo || !s.has_up)
                throw ParseError("general input is not symmetric: entry " + where + " lacks its mirror",
                                 s.has_lo ? s.ln_lo : s.ln_up);
            const double scale = std::max({std::fabs(s.lo), std::fabs(s.up), 1e-300});
            if (std::fabs(s.lo - s.up) > 1e-12 * scale)
                throw ParseError("general input is not symmetric: entry " + where + " mismatches its mirror", s.ln_up);
        }
        es.push_back({r, c, s.lo});
    }
    return from_entries(static_cast<int>(rows), es);
}

void write_matrix_market_file(const SparseSym& a, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    const bool cplx = a.is_complex();  // extension: "complex hermitian", lower triangle
    out << (cplx ? "%%MatrixMarket matrix coordinate complex hermitian\n"
                 : "%%MatrixMarket matrix coordinate real symmetric\n");
    out << a.rows() << " " << a.rows() << " " << a.nnz_lower() << "\n";
    char buf[120];
    for (int r = 0; r < a.rows(); ++r)
        for (int64_t p = a.row_ptr()[r]; p < a.row_ptr()[r + 1]; ++p) {
            if (cplx)
                std::snprintf(buf, sizeof buf, "%d %d %.17g %.17g\n", r + 1, a.col()[p] + 1, a.val()[2 * p],
                              a.val()[2 * p + 1]);
            else
                std::snprintf(buf, sizeof buf, "%d %d %.17g\n", r + 1, a.col()[p] + 1, a.val()[p]);
            out << buf;
        }
    if (!out.flush()) throw IoError("write failed for '" + path + "'");
}

}  // namespace b2
