// Solver loops over device-resident blocks (single B200).
//
// This file restates the control flow of the reference's four solvers
// (proj/src/solvers.cpp:204-463) — the same decisions, events, lock handling,
// work-meter formulas and history records — while every O(n) operation runs
// as a bk_* kernel on one CUDA stream.  Blocks are row-major n x ld buffers;
// X (Ritz vectors), P (LOBPCG momentum) and W (preconditioned residual) are
// adjacent column ranges of one buffer S, so the reference's hcat / leftCols /
// rightCols become column offsets, and shrink/expand is a width change plus a
// strided compaction copy (K7).  The host reads back one small record per
// iteration (r_overall, converged prefix, non-finite flag) plus the kept count
// of each orthonormalisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <limits>
#include <thread>
#include <vector>

#include "host.hpp"
#include "rng.hpp"

namespace b2 {

namespace {

constexpr double kDropTol = 1e-8;  // kDropTolDefault, proj/src/kernel.hpp:17
constexpr int kMaxRitzDim = 1200;
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();  // K5 (bk_syev_d / _z) limit, kSyevMaxD in bk_syev.cu

int round8(int x) { return (x + 7) & ~7; }

// A block view: ld and column offsets count scalar elements; cw = 2 for
// complex128 (interleaved (re, im) doubles), so column c starts at p + c*cw.
struct Blk {
    double* p;
    int ld;
    int cw;
    Blk at(int c) const { return {p + static_cast<size_t>(c) * cw, ld, cw}; }
};

thread_local double g_host_call_s = 0.0;  // BLOCKEIG_TIMING: host time inside CUDA / bk_* calls
#define BKC(call)                                                                                          \
    do {                                                                                                   \
        const auto _h0 = std::chrono::steady_clock::now();                                                 \
        cuda_check((call), #call);                                                                         \
        g_host_call_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - _h0).count(); \
    } while (0)
// launch + (when profiling) time it as an "other" kernel class
// small bookkeeping launches ("other"): not bracketed by timing events — two
// event records per launch cost ~6 % of a profiled solve; the class's time is
// the step time minus the timed classes
#define BKO(call) BKC(call)

// pinned host staging for the per-iteration record and small infos
struct Pinned {
    double* rec = nullptr;  // 8 doubles
    int* info = nullptr;    // 64 ints: [0..15] synchronous infos, [16..] speculative K4 slots,
                            // [48..] K4 conditioning flags (2 per call slot)
    Pinned() {
        BKC(cudaMallocHost(reinterpret_cast<void**>(&rec), 8 * sizeof(double)));
        BKC(cudaMallocHost(reinterpret_cast<void**>(&info), 64 * sizeof(int)));
    }
    ~Pinned() {
        cudaFreeHost(rec);
        cudaFreeHost(info);
    }
};

// Work counters with the reference formulas (proj/src/solvers.cpp:26-60).
struct Meter {
    Work w;
    int64_t rr_flops = 0;
    int iter_rr_dim = 0;
    void begin_iteration() { iter_rr_dim = 0; }
    void ortho(int64_t n, int64_t k) { w.ortho_flops += n * k * k; }
    void proj_ortho(int64_t n, int64_t k, int64_t m) { w.ortho_flops += n * k * (2 * m + k); }
    void rr(int64_t n, int64_t d) {
        w.spmv_cols += d;
        rr_flops += 2 * n * d * d + d * d * d;
        iter_rr_dim = static_cast<int>(d);
    }
};

// reference StagnationGuard (solvers.cpp:128-143)
struct Stagnation {
    double mark = std::numeric_limits<double>::infinity();
    int mark_iter = 0;
    bool update(int j, double overall) {
        const double lg = std::log10(std::max(overall, 1e-300));
        if (lg <= mark - 0.01) {
            mark = lg;
            mark_iter = j;
            return false;
        }
        return j - mark_iter >= 50;
    }
};

class Engine {
    // first member: the device is current before any member that creates
    // device objects (the event pool) is initialised
    int cfg_dev_;
    static int set_device(int dev) {
        BKC(cudaSetDevice(dev));
        return dev;
    }

public:
    Engine(const SparseSym& a, const SolverConfig& cfg, SolverKind kind)
        : cfg_dev_(set_device(cfg.device)), a_(a), cfg_(cfg), kind_(kind), n_(a.rows()), cw_(a.is_complex() ? 2 : 1),
          rng_(cfg.seed) {
        csr_ = &a.device_csr(cfg.device, cfg.largest);
        BKC(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        const int n_ex = cfg.n_ex, n_es = cfg.n_es;
        const int xd = std::max(1, 2 * (n_ex - n_es));
        tcap_ = std::max(n_ex, xd);
        dcap_ = 3 * n_ex + xd;
        dcap_ = std::min(dcap_, std::max(n_, 1));
        dcap_ = std::max(dcap_, n_ex);
        ldS_ = round8(std::max(dcap_ + tcap_, 8));
        ldT_ = round8(std::max(tcap_, 8));
        const size_t n = static_cast<size_t>(std::max(n_, 1));
        const size_t es = sizeof(double) * cw_;  // bytes per scalar element
        for (auto& s : S_) s.alloc(n * ldS_ * es);
        AS_.alloc(n * ldS_ * es);
        R_.alloc(n * ldT_ * es);
        XD_.alloc(n * ldT_ * es);
        T1_.alloc(n * ldT_ * es);
        T2_.alloc(n * ldT_ * es);
        PT_.alloc(n * ldT_ * es);
        VEC_.alloc(n * es);
        // coefficient blocks: 64-byte rows (16-byte copies of update coefficients)
        const size_t dc = static_cast<size_t>(round8(dcap_ + tcap_));
        ldH_ = static_cast<int>(dc);
        H_.alloc(dc * dc * es);
        Z_.alloc(dc * dc * es);
        ZC_.alloc(dc * dc * es);
        CZ_.alloc(dc * dc * es);
        VALS_.alloc(dc * sizeof(double));
        VALS_BAK_.alloc(dc * sizeof(double));
        COEF_.alloc(dc * static_cast<size_t>(tcap_) * es + 64);
        GB_.alloc(static_cast<size_t>(tcap_) * tcap_ * es);
        M1_.alloc(static_cast<size_t>(tcap_) * tcap_ * es);
        M2_.alloc(static_cast<size_t>(tcap_) * tcap_ * es);
        SMALL_.alloc(8 * dc * sizeof(double));
        INFO_.alloc(96 * sizeof(int));
        const int idc = static_cast<int>(dc);
        size_t work;
        if (cw_ == 1) {
            work = bk_gram_work_bytes(n_, idc, idc);
            work = std::max(work, bk_chol_work_bytes(std::max(tcap_, 1)));
            work = std::max(work, bk_syev_work_bytes(idc));
            work = std::max(work, bk_residual_work_bytes(n_, idc));
            work = std::max(work, bk_colnorm2_work_bytes(n_, idc));
        } else {
            work = bk_gram_z_work_bytes(n_, idc, idc);
            work = std::max(work, bk_chol_z_work_bytes(std::max(tcap_, 1)));
            work = std::max(work, bk_syev_z_work_bytes(idc));
            work = std::max(work, bk_residual_z_work_bytes(n_, idc));
            work = std::max(work, bk_colnorm2_z_work_bytes(n_, idc));
            CEXP_.alloc(bk_gemm_z_work_bytes(idc, idc));
        }
        WORK_.alloc(work);
        if (cfg.precond == Precond::diagonal) {
            std::vector<double> t(n);
            for (int i = 0; i < n_; ++i) t[i] = 1.0 / std::max(std::fabs(a.diagonal(i)), 1e-12);
            TD_.alloc(n * sizeof(double));
            BKC(cudaMemcpyAsync(TD_.d(), t.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream_));
        }
        // estimate_norm2 (host, reference loop order) is first needed by the
        // first convergence test: a fresh handle computes it on a host thread
        // while the device uploads x0 and runs the initial orthonormalisation
        // and Rayleigh-Ritz step (config 5: 0.8 s hidden)
        if (a.norm_cached() || n_ < 65536) norm_a_ = a.norm_est();
        else norm_job_ = std::async(std::launch::async, [&a] { return a.norm_est(); });
    }
    ~Engine() {
        if (norm_job_.valid()) norm_job_.wait();
        if (stream_) {
            cudaStreamSynchronize(stream_);
            cudaStreamDestroy(stream_);
        }
        for (auto& p : pending_) {  // unresolved (solve aborted): back to the pool
            ev_pool_.push_back(p.a);
            ev_pool_.push_back(p.b);
        }
    }

    SolveOutput run(const double* x0, int x0_cols);
    void set_strategy(const StrategyConfig& s) { strategy_ = s; }

    // ---- test harness (bk_harness_*): one K4 or HL-trick call through the
    // solvers' own code, on host column-major blocks
    int harness_proj_ortho(const double* w, int a, const double* q, int m, double* out) {
        upload_colmajor(w, a, T1());
        if (m > 0) upload_colmajor(q, m, S(0));
        const int kept = proj_ortho(n_, T1(), a, S(0), m, S(0).at(m));
        download_colmajor(S(0).at(m), kept, out);
        return kept;
    }
    int harness_hl(const double* s, int d, const double* z, int n_now, int lock, double* x, double* p) {
        upload_colmajor(s, d, S(0));
        const size_t zb = static_cast<size_t>(d) * d * sizeof(double);
        DevMem zcm(zb);
        BKC(cudaMemcpyAsync(zcm.d(), z, zb, cudaMemcpyHostToDevice, stream_));
        BKC(bk_cm_to_rm_d(d, d, zcm.d(), d, Z_.d(), ldH_, st()));
        const int pk = hl_lift(S(0), d, n_now, lock, S(1), -1);
        download_colmajor(S(1), n_now, x);
        download_colmajor(S(1).at(n_now), pk, p);
        return pk;
    }

private:
    StrategyConfig strategy_;
    // ---------------------------------------------------------------- primitives
    void* st() const { return stream_; }
    Blk B(double* p, int ld) const { return {p, ld, cw_}; }
    Blk S(int i) const { return B(S_[i].d(), ldS_); }
    Blk AS() const { return B(AS_.d(), ldS_); }
    Blk T1() const { return B(T1_.d(), ldT_); }
    Blk T2() const { return B(T2_.d(), ldT_); }

    void sync() {
        const auto t0 = std::chrono::steady_clock::now();
        BKC(cudaStreamSynchronize(stream_));
        sync_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        ++syncs_;
        // profiling: the event pairs are resolved once at the end of the solve
        // (resolving at every sync put ~100 us of cudaEventElapsedTime calls on
        // the host critical path per iteration); only the device flags of
        // predicated launches are captured now, before their slots are reused
        for (size_t i = captured_; i < pending_.size(); ++i)
            if (pending_[i].pred) pending_[i].predv = *pending_[i].pred;
        captured_ = pending_.size();
        if (pending_.size() > 60000) prof_resolve();
    }
    size_t captured_ = 0;
    double sync_wait_s_ = 0.0;
    int64_t syncs_ = 0;
    // BLOCKEIG_TIMING: wall time per loop phase (host view, includes waits)
    double phase_s_[8] = {};
    std::chrono::steady_clock::time_point phase_t_ = std::chrono::steady_clock::now();
    void mark(int ph) {
        const auto now = std::chrono::steady_clock::now();
        phase_s_[ph] += std::chrono::duration<double>(now - phase_t_).count();
        phase_t_ = now;
    }

    // ---- optional per-kernel-class CUDA-event timing (ext->profile)
    struct Pending {
        int cls;
        cudaEvent_t a, b;
        double bytes, flops;
        const int* pred;  // predicated launch: host copy of its device flag (valid at the next sync)
        int predv;        // its value, captured at that sync
    };
    // timing events are pooled per host thread across solves (a config-2 solve
    // records ~30k of them)
    // (per host thread AND device: an event belongs to the device it was created on)
    static constexpr int kMaxDev = 64;
    static std::vector<cudaEvent_t>& event_pool(int dev) {
        static thread_local std::vector<cudaEvent_t>* v[kMaxDev] = {};
        auto& p = v[dev % kMaxDev];
        if (!p) p = new std::vector<cudaEvent_t>;
        return *p;
    }
    std::vector<cudaEvent_t>& ev_pool_ = event_pool(cfg_dev_);
    std::vector<Pending> pending_;
    KernelStat kstats_[K_CLASSES];
    cudaEvent_t take_event() {
        if (!ev_pool_.empty()) {
            cudaEvent_t e = ev_pool_.back();
            ev_pool_.pop_back();
            return e;
        }
        cudaEvent_t e;
        BKC(cudaEventCreate(&e));
        return e;
    }
    cudaEvent_t prof_begin() {
        if (!cfg_.profile) return nullptr;
        cudaEvent_t e = take_event();
        BKC(cudaEventRecord(e, stream_));
        return e;
    }
    void prof_end(cudaEvent_t a, int cls, double bytes, double flops, const int* pred = nullptr) {
        if (!a) return;
        cudaEvent_t b = take_event();
        BKC(cudaEventRecord(b, stream_));
        pending_.push_back({cls, a, b, bytes, flops, pred, 1});
    }
    void prof_resolve() {
        for (size_t i = 0; i < pending_.size(); ++i) {
            auto& p = pending_[i];
            float ms = 0.f;
            BKC(cudaEventElapsedTime(&ms, p.a, p.b));
            if (p.pred && p.predv == 0) {  // predicated off: an empty launch, not K2/K3 work
                p.cls = K_OTHER;
                p.bytes = p.flops = 0.0;
            }
            auto& k = kstats_[p.cls];
            k.launches += 1;
            k.ms += ms;
            k.bytes += p.bytes;
            k.flops += p.flops;
            if (i + 1 < pending_.size()) {  // device idle / unprofiled time before the next class
                float gap = 0.f;
                BKC(cudaEventElapsedTime(&gap, p.b, pending_[i + 1].a));
                gap_ms_[pending_[i + 1].cls] += gap;
            }
        }
        for (auto& p : pending_) {
            ev_pool_.push_back(p.a);
            ev_pool_.push_back(p.b);
        }
        pending_.clear();
        captured_ = 0;
    }
    double gap_ms_[K_CLASSES] = {};
    int64_t spmm_win_calls_ = 0;  // K1 launches that ran as K1w

    // K1: algorithmic bytes nnz*12 + (n+1)*4 + 2*n*k*8
    void spmm(Blk x, int k, Blk y) {
        if (k <= 0) return;
        auto t = prof_begin();
        // K1w once the handle's window plan is ready (bit-identical to K1, so the
        // switch can happen mid-solve); X and Y views of the same column parity
        const bool win = cw_ == 1 && csr_->win_state.load(std::memory_order_acquire) == 2 && k >= 8 &&
                         x.ld % 2 == 0 && y.ld % 2 == 0 &&
                         reinterpret_cast<uintptr_t>(x.p) % 16 == reinterpret_cast<uintptr_t>(y.p) % 16;
        if (win) {
            const DeviceCsr::Win& w = csr_->win;
            BKC(bk_spmm_win_d(n_, w.tile, w.ntiles, w.wmax, w.nzmax, w.rp2.as<int32_t>(), w.code.as<int32_t>(),
                              w.val2.d(), w.wptr.as<int32_t>(), w.wrow.as<int32_t>(), x.p, x.ld, k, y.p, y.ld, st()));
            ++spmm_win_calls_;
        } else if (cw_ == 1)
            BKC(bk_spmm_d(n_, csr_->row_ptr.as<int32_t>(), csr_->col.as<int32_t>(), csr_->val.d(), x.p, x.ld, k, y.p,
                          y.ld, st()));
        else
            BKC(bk_spmm_z(n_, csr_->row_ptr.as<int32_t>(), csr_->col.as<int32_t>(), csr_->val.d(), x.p, x.ld, k, y.p,
                          y.ld, st()));
        // complex: nnz*(16+4) + (n+1)*4 + 2*n*k*16 bytes, 8*nnz*k flops
        prof_end(t, K_SPMM, (8.0 * cw_ + 4.0) * csr_->nnz_full + 4.0 * (n_ + 1) + 16.0 * cw_ * n_ * k,
                 2.0 * cw_ * cw_ * csr_->nnz_full * k);
    }
    // K2: flops 2*rows*a*b; bytes 8*rows*(a+b)
    void gram(int rows, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc) {
        auto t = rows >= n_ ? prof_begin() : nullptr;
        if (cw_ == 1)
            BKC(bk_gram_d(rows, x, ldx, a, y, ldy, b, c, ldc, WORK_.p(), st()));
        else
            BKC(bk_gram_z(rows, x, ldx, a, y, ldy, b, c, ldc, WORK_.p(), st()));
        // only the n-row contractions are K2 work; coefficient-space ones (rows = d,
        // HL trick) are latency-bound bookkeeping and counted as "other"
        prof_end(t, rows >= n_ ? K_GRAM : K_OTHER, 8.0 * cw_ * rows * (a + b), 2.0 * cw_ * cw_ * rows * a * b);
    }
    // K3: flops 2*rows*d*k; bytes 8*rows*(d + k (+k when beta != 0))
    void gemm(int rows, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha, double beta,
              double* y, int ldy) {
        auto t = rows >= n_ ? prof_begin() : nullptr;
        if (cw_ == 1)
            BKC(bk_gemm_d(rows, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, st()));
        else
            BKC(bk_gemm_z(rows, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, CEXP_.p(), st()));
        prof_end(t, rows >= n_ ? K_GEMM : K_OTHER, 8.0 * cw_ * rows * (d + k + (beta != 0.0 ? k : 0)),
                 2.0 * cw_ * cw_ * rows * d * k);
    }
    // predicated K2/K3 (run only when *flag != 0 on the device); the profile
    // entry is resolved against the flag's host copy (pin_.info[3]) at the next sync
    void gram_if(int rows, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                 const int* flag, const int* flag_host) {
        auto t = rows >= n_ ? prof_begin() : nullptr;
        if (cw_ == 1) BKC(bk_gram_if_d(rows, x, ldx, a, y, ldy, b, c, ldc, WORK_.p(), flag, st()));
        else BKC(bk_gram_if_z(rows, x, ldx, a, y, ldy, b, c, ldc, WORK_.p(), flag, st()));
        prof_end(t, rows >= n_ ? K_GRAM : K_OTHER, 8.0 * cw_ * rows * (a + b), 2.0 * cw_ * cw_ * rows * a * b,
                 flag_host);
    }
    void gemm_if(int rows, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                 double beta, double* y, int ldy, const int* flag, const int* flag_host) {
        auto t = rows >= n_ ? prof_begin() : nullptr;
        if (cw_ == 1) BKC(bk_gemm_if_d(rows, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, flag, st()));
        else BKC(bk_gemm_if_z(rows, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, CEXP_.p(), flag, st()));
        prof_end(t, rows >= n_ ? K_GEMM : K_OTHER, 8.0 * cw_ * rows * (d + k + (beta != 0.0 ? k : 0)),
                 2.0 * cw_ * cw_ * rows * d * k, flag_host);
    }
    // column movement and elementwise ops work on the real view (cw doubles per element)
    void copy(int rows, Blk src, int k, Blk dst) {
        if (k > 0 && rows > 0) BKO(bk_copy_cols_d(rows, src.p, src.ld * cw_, k * cw_, dst.p, dst.ld * cw_, st()));
    }
    void colnorm2(int rows, Blk x, int k, double* out) {
        if (cw_ == 1) BKO(bk_colnorm2_d(rows, x.p, x.ld, k, out, WORK_.p(), st()));
        else BKO(bk_colnorm2_z(rows, x.p, x.ld, k, out, WORK_.p(), st()));
    }
    void ns_coeff(int a, const double* g, int ldg, double* m, int ldm) {
        if (cw_ == 1) BKO(bk_ns_coeff_d(a, g, ldg, m, ldm, st()));
        else BKO(bk_ns_coeff_z(a, g, ldg, m, ldm, st()));
    }
    void scale_rows(int rows, int k, const double* t, Blk x, Blk y) {
        BKO(bk_scale_rows_d(rows, k * cw_, t, x.p, x.ld * cw_, y.p, y.ld * cw_, st()));
    }
    void zero_rows(Blk x, int k, int r0, int r1) { BKO(bk_zero_rows_d(x.p, x.ld * cw_, k * cw_, r0, r1, st())); }
    void lincomb(int rows, int k, double a, Blk x, double b, Blk y, Blk out) {
        BKO(bk_lincomb_d(rows, k * cw_, a, x.p, x.ld * cw_, b, y.p, y.ld * cw_, out.p, out.ld * cw_, st()));
    }

    // host std::mt19937_64 / normal_distribution block (random_block,
    // kernel.cpp:166-172: a fresh distribution per call, column-major fill),
    // uploaded into dst (row-major)
    void random_block(int cols, Blk dst) {
        if (cols <= 0) return;
        const auto t0 = std::chrono::steady_clock::now();
        // complex: real then imaginary part of each entry (random_block<complex>);
        // the stream is drawn straight into pinned chunks and DMA'd asynchronously
        const size_t count = static_cast<size_t>(n_) * cols * cw_;
        if (stage_.bytes() < count * sizeof(double)) stage_.alloc(count * sizeof(double));
        chunked_h2d(stage_.d(), count, [&](double* buf, size_t, size_t len) { rng_.take(buf, len); });
        if (cw_ == 1) BKC(bk_cm_to_rm_d(n_, cols, stage_.d(), n_, dst.p, dst.ld, st()));
        else BKC(bk_cm_to_rm_z(n_, cols, stage_.d(), n_, dst.p, dst.ld, st()));
        rng_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        rng_cols_ += cols;
    }
    // Host <-> device through two pinned 16 MB chunks per host thread: the DMA of
    // one chunk overlaps the host-side fill / drain of the other (pageable
    // transfers ran at ~3-8 GB/s and synchronised the stream).
    static constexpr size_t kChunk = size_t(2) << 20;  // doubles
    struct PinnedChunks {
        double* buf[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        bool used[2] = {false, false};
        PinnedChunks() {
            for (int i = 0; i < 2; ++i) {
                BKC(cudaMallocHost(reinterpret_cast<void**>(&buf[i]), kChunk * sizeof(double)));
                BKC(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
            }
        }
    };
    // host-side copy between user memory and a pinned chunk on up to 8 threads
    // (one thread moves ~8-10 GB/s; the DMA of the other chunk runs meanwhile)
    static void par_memcpy(void* dst, const void* src, size_t bytes) {
        static const int nthr = std::max(1, std::min(8, static_cast<int>(std::thread::hardware_concurrency()) / 2));
        if (bytes < (size_t(4) << 20) || nthr == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::vector<std::thread> th;
        const size_t part = (bytes / nthr + 63) & ~size_t(63);
        for (int t = 1; t < nthr; ++t) {
            const size_t o = std::min(bytes, part * t), e = std::min(bytes, o + part);
            if (o < e)
                th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, e - o); });
        }
        std::memcpy(dst, src, std::min(bytes, part));
        for (auto& x : th) x.join();
    }
    // per host thread and device (the chunk events belong to one device)
    PinnedChunks& chunks() {
        static thread_local PinnedChunks* c[kMaxDev] = {};
        auto& p = c[cfg_.device % kMaxDev];
        if (!p) p = new PinnedChunks;
        return *p;
    }
    template <class Fill>
    void chunked_h2d(double* dst, size_t count, Fill fill) {
        auto& c = chunks();
        for (size_t off = 0, i = 0; off < count; off += kChunk, ++i) {
            const int b = static_cast<int>(i & 1);
            const size_t len = std::min(kChunk, count - off);
            if (c.used[b]) BKC(cudaEventSynchronize(c.ev[b]));  // its previous DMA is done
            fill(c.buf[b], off, len);
            BKC(cudaMemcpyAsync(dst + off, c.buf[b], len * sizeof(double), cudaMemcpyHostToDevice, stream_));
            BKC(cudaEventRecord(c.ev[b], stream_));
            c.used[b] = true;
        }
    }
    void chunked_d2h(double* dst, const double* src, size_t count) {
        auto& c = chunks();
        const size_t nch = (count + kChunk - 1) / kChunk;
        for (size_t i = 0; i <= nch; ++i) {
            if (i < nch) {  // DMA chunk i (its buffer was drained at step i - 1)
                const int b = static_cast<int>(i & 1);
                const size_t off = i * kChunk, len = std::min(kChunk, count - off);
                BKC(cudaMemcpyAsync(c.buf[b], src + off, len * sizeof(double), cudaMemcpyDeviceToHost, stream_));
                BKC(cudaEventRecord(c.ev[b], stream_));
                c.used[b] = true;
            }
            if (i > 0) {  // drain chunk i - 1 while chunk i is in flight
                const int b = static_cast<int>((i - 1) & 1);
                const size_t off = (i - 1) * kChunk, len = std::min(kChunk, count - off);
                BKC(cudaEventSynchronize(c.ev[b]));
                par_memcpy(dst + off, c.buf[b], len * sizeof(double));
            }
        }
    }
    double rng_s_ = 0.0;
    int64_t rng_cols_ = 0;
    void upload_colmajor(const double* h, int cols, Blk dst) {
        const size_t bytes = static_cast<size_t>(n_) * cols * sizeof(double) * cw_;
        if (stage_.bytes() < bytes) stage_.alloc(bytes);
        // pinned double-buffered chunks filled on several host threads (a pageable
        // cudaMemcpy of config 2's 201 MB X0 ran at ~9 GB/s)
        chunked_h2d(stage_.d(), bytes / sizeof(double),
                    [&](double* buf, size_t off, size_t len) { par_memcpy(buf, h + off, len * sizeof(double)); });
        if (cw_ == 1) BKC(bk_cm_to_rm_d(n_, cols, stage_.d(), n_, dst.p, dst.ld, st()));
        else BKC(bk_cm_to_rm_z(n_, cols, stage_.d(), n_, dst.p, dst.ld, st()));
        sync();  // the host buffer may be released by the caller
    }

    void download_colmajor(Blk src, int cols, double* h) {
        if (cols <= 0) return;
        const size_t count = static_cast<size_t>(n_) * cols;
        DevMem cm(count * sizeof(double));
        BKC(bk_rm_to_cm_d(n_, cols, src.p, src.ld, cm.d(), n_, st()));
        BKC(cudaMemcpyAsync(h, cm.d(), count * sizeof(double), cudaMemcpyDeviceToHost, stream_));
        sync();
    }

    // K4: project w (rows x a, clobbered) against q (rows x m), orthonormalise
    // the rest with the CGS2 drop rule; kept columns land packed in out.
    // (project_orthonormalize, proj/src/kernel.cpp:65-89)
    // slot >= 0: speculative — no host round trip; the caller proceeds as if all
    // a columns were kept and verifies the Cholesky info at the next record
    // readback (spec_ok), redoing the iteration synchronously if not.
    int proj_ortho(int rows, Blk w, int a, Blk q, int m, Blk out, int slot = -1, const double* pre_ref2 = nullptr) {
        if (a <= 0) return 0;
        double* ref2 = SMALL_.d();  // a doubles
        // column norms of w: precomputed by the kernel that wrote w (residual_kernel), else here
        if (pre_ref2) BKC(cudaMemcpyAsync(ref2, pre_ref2, a * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
        else colnorm2(rows, w, a, ref2);
        // [0..2] Cholesky info, [3] DGKS flag; speculative calls use their own slot
        int* info = INFO_.as<int>() + (slot >= 0 ? 40 + 4 * slot : 0);
        int* info_host = pin_.info + (slot >= 0 ? 16 + 4 * slot : 0);
        if (m > 0) {
            // the reference's CGS2 projects twice (kernel.cpp:73-80); the second
            // block pass runs only when the first removed more than half of some
            // column's squared norm ("twice is enough", DGKS eta = 1/sqrt 2) —
            // decided on the device, the pass-2 kernels are predicated on it
            gram(rows, q.p, q.ld, m, w.p, w.ld, a, COEF_.d(), a);
            gemm(rows, q.p, q.ld, m, COEF_.d(), a, a, -1.0, 1.0, w.p, w.ld);
            BKO(bk_dgks_flag_d(m, a, COEF_.d(), a, cw_, ref2, 0.5, info + 3, st()));
            gram_if(rows, q.p, q.ld, m, w.p, w.ld, a, COEF_.d(), a, info + 3, info_host + 3);
            gemm_if(rows, q.p, q.ld, m, COEF_.d(), a, a, -1.0, 1.0, w.p, w.ld, info + 3, info_host + 3);
        } else {
            BKC(cudaMemsetAsync(info + 3, 0, sizeof(int), stream_));
        }
        gram(rows, w.p, w.ld, a, w.p, w.ld, a, GB_.d(), a);
        // conditioning flags of this call: [0] ill (g_jj / p_j > 1e3 for a kept
        // pivot), [1] well — predicates of the two second-pass forms below
        int* cond = INFO_.as<int>() + 64 + 2 * (slot + 1);
        int* cond_host = pin_.info + 48 + 2 * (slot + 1);
        auto tc = prof_begin();
        if (cw_ == 1) BKC(bk_chol_drop_cond_d(a, GB_.d(), a, ref2, kDropTol, M1_.d(), a, info, cond, WORK_.p(), st()));
        else BKC(bk_chol_drop_cond_z(a, GB_.d(), a, ref2, kDropTol, M1_.d(), a, info, cond, WORK_.p(), st()));
        prof_end(tc, K_CHOL, 8.0 * cw_ * a * a, cw_ * cw_ * a * a * a / 3.0);
        BKC(cudaMemcpyAsync(info_host, info, 4 * sizeof(int), cudaMemcpyDeviceToHost, stream_));
        BKC(cudaMemcpyAsync(cond_host, cond, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream_));
        ++proj_calls_;
        int kept = a;
        if (slot >= 0) {
            spec_expect_[slot] = a;
        } else {
            sync();
            pass2_ += pin_.info[3];
            if (debug_ && cw_ == 1) debug_pivots(a, ref2);
            if (pin_.info[2]) throw std::runtime_error("orthonormalization: non-finite values");
            if (pin_.info[1]) return cgs2_fallback(rows, w, a, q, m, out);
            kept = pin_.info[0];
            if (kept == 0) return 0;
        }
        // second pass: the block is orthonormal to ~1e-8 after the pivot-checked
        // first pass (p >= 1e-8 g_jj bounds its condition), so one Newton-Schulz
        // step W1 (3I - G1)/2 restores orthogonality without a second sequential
        // factorisation or host round trip.  For n-row blocks G1 = W1^T W1 is
        // formed from the first Gram (G1 = M1^T G M1, a x a work) and the two
        // steps are fused into one tall update out = W (M1 M2): one n-row Gram
        // and one n-row update fewer per orthonormalisation.  (The tall product's
        // own rounding, O(kappa eps) with kappa <= 1e4 after the pivot check, is
        // below what the Rayleigh-Ritz step resolves.)
        // That fused form corrects only the Cholesky's own rounding: W1's true Gram
        // differs from M1^T G M1 by M1^T dG M1 ~ eps g_jj / p_j, so when a kept
        // pivot lost more than 1e-3 of its projected norm squared (device flag
        // cond[0], from the Cholesky) the tall form below runs instead — W1 = W M1
        // formed, its Gram taken, one Newton-Schulz step — restoring orthogonality
        // to rounding (CholQR2 with the second factorisation replaced by the NS
        // step).  Both forms are launched, each predicated on its flag: no host
        // round trip.
        static const bool ns_tall = std::getenv("BLOCKEIG_NS_TALL") != nullptr;
        if (rows >= n_ && !ns_tall) {
            gemm(a, GB_.d(), a, a, M1_.d(), a, kept, 1.0, 0.0, COEF_.d(), kept);       // T = G M1
            gram(a, M1_.d(), a, kept, COEF_.d(), kept, kept, GB_.d(), kept);           // G1 = M1^T T
            ns_coeff(kept, GB_.d(), kept, M2_.d(), kept);                               // M2 = (3I - G1)/2
            gemm(a, M1_.d(), a, kept, M2_.d(), kept, kept, 1.0, 0.0, COEF_.d(), kept);  // M1 M2
            gemm_if(rows, w.p, w.ld, a, COEF_.d(), kept, kept, 1.0, 0.0, out.p, out.ld, cond + 1, cond_host + 1);
            Blk pt = B(PT_.d(), ldT_);
            gemm_if(rows, w.p, w.ld, a, M1_.d(), a, kept, 1.0, 0.0, pt.p, pt.ld, cond, cond_host);
            gram_if(rows, pt.p, pt.ld, kept, pt.p, pt.ld, kept, GB_.d(), kept, cond, cond_host);
            ns_coeff(kept, GB_.d(), kept, M2_.d(), kept);  // (stale input when skipped: unused)
            gemm_if(rows, pt.p, pt.ld, kept, M2_.d(), kept, kept, 1.0, 0.0, out.p, out.ld, cond, cond_host);
            return kept;
        }
        Blk pt = B(PT_.d(), ldT_);
        gemm(rows, w.p, w.ld, a, M1_.d(), a, kept, 1.0, 0.0, pt.p, pt.ld);
        gram(rows, pt.p, pt.ld, kept, pt.p, pt.ld, kept, GB_.d(), kept);
        ns_coeff(kept, GB_.d(), kept, M2_.d(), kept);
        gemm(rows, pt.p, pt.ld, kept, M2_.d(), kept, kept, 1.0, 0.0, out.p, out.ld);
        return kept;
    }

    // BLOCKEIG_DEBUG=1: recompute the pivot ratios on the host and log them
    void debug_pivots(int a, const double* ref2_dev) {
        std::vector<double> g(static_cast<size_t>(a) * a), ref2(a);
        BKC(cudaMemcpy(g.data(), GB_.d(), g.size() * sizeof(double), cudaMemcpyDeviceToHost));
        BKC(cudaMemcpy(ref2.data(), ref2_dev, a * sizeof(double), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[blockeig] proj_ortho a=%d kept=%d unsure=%d:", a, pin_.info[0], pin_.info[1]);
        std::vector<double> s = g;  // host replica of the right-looking skip-pivot Cholesky
        for (int j = 0; j < a; ++j) {
            const double p = s[static_cast<size_t>(j) * a + j];
            const double gjj = g[static_cast<size_t>(j) * a + j];
            const double ratio = ref2[j] > 0 ? std::sqrt(std::max(p, 0.0) / ref2[j]) : 0.0;
            const double proj = ref2[j] > 0 ? std::sqrt(gjj / ref2[j]) : 0.0;
            const bool keep = ref2[j] > 0 && p >= kDropTol * kDropTol * ref2[j];
            if (ratio < 1e-1 || !keep)
                std::fprintf(stderr, " [col %d piv/ref=%.3e proj/ref=%.3e keep=%d]", j, ratio, proj, keep);
            if (!keep) continue;
            const double r = std::sqrt(p);
            for (int l = j + 1; l < a; ++l) s[static_cast<size_t>(j) * a + l] /= r;
            for (int k = j + 1; k < a; ++k)
                for (int l = k; l < a; ++l)
                    s[static_cast<size_t>(k) * a + l] -= s[static_cast<size_t>(j) * a + k] * s[static_cast<size_t>(j) * a + l];
        }
        std::fprintf(stderr, "\n");
    }

    // exact column CGS2 (kernel.cpp:71-86) for blocks whose Cholesky pivots
    // were not decisive; w already carries the external projection
    // The external projection (two block passes against q) is already applied
    // to w, so only the in-block Gram-Schmidt remains: two passes against the
    // columns accepted so far, then the drop test against the ORIGINAL norm —
    // decided on the device (bk_cgs2_commit_d), one host sync at the end.
    // `out` is zeroed first, so projecting against its first j columns (kept <= j)
    // is exact without knowing the kept count on the host.
    int cgs2_fallback(int rows, Blk w, int a, Blk q, int m, Blk out) {
        (void)q;
        (void)m;
        ++fallbacks_;
        const double* ref2 = SMALL_.d();  // set by proj_ortho
        Blk v = B(VEC_.d(), 1);
        double* c = COEF_.d();
        double* nrm2 = SMALL_.d() + tcap_;
        int* counter = INFO_.as<int>() + 32;
        zero_rows(out, a, 0, rows);
        BKC(cudaMemsetAsync(counter, 0, sizeof(int), stream_));
        for (int j = 0; j < a; ++j) {
            copy(rows, w.at(j), 1, v);
            if (j > 0)
                for (int pass = 0; pass < 2; ++pass) {
                    gram(rows, out.p, out.ld, j, v.p, 1, 1, c, 1);
                    gemm(rows, out.p, out.ld, j, c, 1, 1, -1.0, 1.0, v.p, 1);
                }
            colnorm2(rows, v, 1, nrm2);
            if (cw_ == 1) BKO(bk_cgs2_commit_d(rows, v.p, nrm2, ref2 + j, kDropTol, out.p, out.ld, counter, st()));
            else BKO(bk_cgs2_commit_z(rows, v.p, nrm2, ref2 + j, kDropTol, out.p, out.ld, counter, st()));
        }
        BKC(cudaMemcpyAsync(pin_.info + 13, counter, sizeof(int), cudaMemcpyDeviceToHost, stream_));
        sync();
        return pin_.info[13];
    }

    // count fresh orthonormal random columns orthogonal to q = [vs | acc],
    // written right after q (out == q.at(m)) — fresh_cols, solvers.cpp:64-74
    void fresh_cols(int count, Blk q, int m) {
        int acc = 0;
        for (int attempt = 0; acc < count && attempt < 8; ++attempt) {
            const int want = count - acc;
            random_block(want, T2());
            meter_.proj_ortho(n_, want, m + acc);
            const int kept = proj_ortho(n_, T2(), want, q, m + acc, q.at(m + acc));
            acc += kept;
        }
        if (acc < count) throw std::runtime_error("block rank collapsed beyond recovery");
    }

    // Rayleigh-Ritz on s[:, 0:d]; columns [0, as_from) of AS already hold A s.
    // values -> VALS (ascending), coefficients -> Z (ldH)  (rr.cpp:8-14)
    // n_need: leading Ritz pairs the caller uses (values/vectors beyond it are
    // not computed on the tridiagonal path)
    void rayleigh_ritz(Blk s, int d, int as_from, int n_need = 0) {
        meter_.rr(n_, d);
        spmm(s.at(as_from), d - as_from, AS().at(as_from));
        {  // H = S^T (A S): upper tiles only, mirrored (symmetrised by the eigensolver anyway)
            auto tg = prof_begin();
            if (cw_ == 1) {
                BKC(bk_gram_sym_d(n_, s.p, s.ld, AS_.d(), ldS_, d, H_.d(), ldH_, WORK_.p(), st()));
                // algorithmic flops of a symmetric Gram: n d (d + 1)
                prof_end(tg, K_GRAM, 8.0 * n_ * 2 * d, 1.0 * n_ * d * (d + 1.0));
            } else {
                // complex Hermitian: upper tiles only, 4 n d (d + 1) flops
                BKC(bk_gram_sym_z(n_, s.p, s.ld, AS_.d(), ldS_, d, H_.d(), ldH_, WORK_.p(), st()));
                prof_end(tg, K_GRAM, 16.0 * n_ * 2 * d, 4.0 * n_ * d * (d + 1.0));
            }
        }
        if (d > kMaxRitzDim) throw std::runtime_error("Rayleigh-Ritz dimension exceeds the device eigensolver limit");
        int* info = INFO_.as<int>() + 8;
        auto ts = prof_begin();
        if (cw_ == 1)
            BKC(bk_syev_d(d, H_.d(), ldH_, n_need > 0 ? n_need : d, VALS_.d(), Z_.d(), ldH_, WORK_.p(), info, st()));
        else
            BKC(bk_syev_z(d, H_.d(), ldH_, n_need > 0 ? n_need : d, VALS_.d(), Z_.d(), ldH_, WORK_.p(), info, st()));
        prof_end(ts, K_SYEV, 16.0 * cw_ * d * d, 0.0);
        BKC(cudaMemcpyAsync(pin_.info + 8, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream_));
        syev_pending_ = true;
    }
    void check_syev() {
        if (!syev_pending_) return;
        syev_pending_ = false;
        max_sweeps_ = std::max(max_sweeps_, pin_.info[8]);
        if (pin_.info[9]) throw std::runtime_error("sym_eig_small: eigensolver failed");
    }

    // out[:, 0:k] = s[:, 0:d] Z[:, 0:k]
    void lift(Blk s, int d, const double* z, int ldz, int k, Blk out) {
        gemm(n_, s.p, s.ld, d, z, ldz, k, 1.0, 0.0, out.p, out.ld);
    }
    // HL trick (solvers.cpp:187-196, meter :382) in coefficient space:
    // ZC = [Z(:, :n_now) | orth(Zp)], Zp = Z(:, lock:n_now) with rows < n_now
    // zeroed (a d-row K4 call), then one fused lift out = [X, P] = S ZC.
    // Returns |P|.  slot >= 0: speculative K4 (see proj_ortho).
    int hl_lift(Blk s, int ds, int n_now, int lock, Blk out, int slot) {
        const Blk zc = B(ZC_.d(), ldH_), cz = B(CZ_.d(), ldH_), z = B(Z_.d(), ldH_);
        const int ahl = n_now - lock;
        copy(ds, z, n_now, zc);
        copy(ds, z.at(lock), ahl, cz);
        zero_rows(cz, ahl, 0, n_now);
        mark(0);
        const int pk = proj_ortho(ds, cz, ahl, zc, n_now, zc.at(n_now), slot);
        mark(4);
        meter_.w.ortho_flops += static_cast<int64_t>(ds) * (n_now - lock) * (2 * n_now + (n_now - lock));
        lift(s, ds, zc.p, zc.ld, n_now + pk, out);
        return pk;
    }

    struct Rep {
        double overall;
        int converged;
        bool nonfinite;
        // decision margins (beig_result_margins): per_pair/tol of the last pair
        // inside / first pair outside the converged prefix, and the strategy's
        // warm-up and slope margins (NaN where a test did not run)
        double lo = kNaN, hi = kNaN, warm = kNaN, slope = kNaN;
        void note(const BlockSizer& s) {
            warm = s.warm_margin();
            slope = s.slope_margin();
        }
    };
    // AV into AS[:, 0:k], R = AV - V diag(VALS) into R, record read back
    // (residual_block + assess_convergence, rr.cpp:16-38)
    // tolerate_nonfinite: a speculative iteration is pending and will be redone
    // if its record is non-finite (the caller decides after spec_ok())
    // Speculation support: a redone tail needs the R and AX of its own
    // iteration, which the next residual() overwrote.  save_ritz() keeps the
    // Ritz values the residual used; restore_residual() recomputes R and AX
    // with the same deterministic kernels (bit-identical), no record.
    void save_ritz(int k) {
        BKC(cudaMemcpyAsync(VALS_BAK_.d(), VALS_.d(), sizeof(double) * k, cudaMemcpyDeviceToDevice, stream_));
    }
    void restore_residual(Blk v, int k) {
        spmm(v, k, AS());
        residual_kernel(v, k, VALS_BAK_.d());
    }
    // LOBPCG consumes the residual only as W = T R (solvers.cpp:98-107): the
    // residual kernel writes T R straight into T1 (all n_now columns; the tail
    // takes T1(:, lock:)), R itself is not stored — one read and one write of an
    // n x k block fewer per iteration than R, then scale_rows
    bool fused_w() const { return kind_ == SolverKind::lobpcg; }
    void residual_kernel(Blk v, int k, const double* lam) {
        double* rn2 = SMALL_.d();
        double* vn2 = SMALL_.d() + dcap_ + tcap_;
        const bool f = fused_w();
        double* r = f ? nullptr : R_.d();
        const double* t = f && TD_.bytes() ? TD_.d() : nullptr;
        double* w = f ? T1_.d() : nullptr;
        double* wn2 = f ? w_norms() : nullptr;
        if (cw_ == 1)
            BKC(bk_residual_w_d(n_, v.p, v.ld, AS_.d(), ldS_, lam, k, r, ldT_, t, w, ldT_, 0, rn2, vn2, wn2,
                                WORK_.p(), st()));
        else
            BKC(bk_residual_w_z(n_, v.p, v.ld, AS_.d(), ldS_, lam, k, r, ldT_, t, w, ldT_, 0, rn2, vn2, wn2,
                                WORK_.p(), st()));
    }
    // squared column norms of W = T R (all n_now columns), written by residual_kernel
    double* w_norms() { return SMALL_.d() + 4 * (dcap_ + tcap_); }
    Rep residual(Blk v, int k, int n_ev, bool tolerate_nonfinite = false) {
        meter_.w.spmv_cols += k;
        if (debug_) std::fprintf(stderr, "[blockeig] iteration %zu k=%d\n", out_.history.size() + 1, k);
        spmm(v, k, AS());
        double* rn2 = SMALL_.d();
        double* vn2 = SMALL_.d() + dcap_ + tcap_;
        auto tr = prof_begin();
        residual_kernel(v, k, VALS_.d());
        double* rec = SMALL_.d() + 6 * (dcap_ + tcap_);  // 5 doubles (8 dc allocated)
        if (norm_job_.valid()) norm_a_ = norm_job_.get();
        BKC(bk_convergence_d(k, rn2, vn2, VALS_.d(), norm_a_, n_ev, cfg_.tol, nullptr, rec, st()));
        prof_end(tr, K_RESID, 24.0 * cw_ * n_ * k, 6.0 * cw_ * n_ * k);
        BKC(cudaMemcpyAsync(pin_.rec, rec, 5 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
        sync();
        const bool bad = pin_.rec[2] != 0.0;
        if (!(bad && tolerate_nonfinite)) check_syev();
        if (bad && !tolerate_nonfinite) throw std::runtime_error("non-finite residual or Ritz value");
        Rep rep{pin_.rec[0], static_cast<int>(pin_.rec[1]), bad};
        rep.lo = pin_.rec[3] >= 0.0 ? pin_.rec[3] / cfg_.tol : kNaN;
        rep.hi = pin_.rec[4] >= 0.0 ? pin_.rec[4] / cfg_.tol : kNaN;
        return rep;
    }

    // y = op(x): shifted operator c x - M x (extension) or shift-and-invert
    // (A - zeta I)^{-1} x through the dense factor (reference SpdFactor dense path)
    void apply_op(Blk x, int k, Blk ax_known, bool have_ax, Blk y) {
        if (k <= 0) return;
        if (cfg_.op_shifted) {
            if (!have_ax) {
                spmm(x, k, T2());
                ax_known = T2();
            }
            lincomb(n_, k, cfg_.op_c, x, -1.0, ax_known, y);
            return;
        }
        if (spchol_) {  // n > 2000: sparse factor, device triangular solves
            auto t = prof_begin();
            spchol_->solve(x.p, x.ld, k, y.p, y.ld, st());
            prof_end(t, K_OTHER, 0.0, 0.0);
            return;
        }
        // (A - zeta I)^{-1} = M M^T with M = R^{-1} from the dense Cholesky
        gram(n_, INV_.d(), n_, n_, x.p, x.ld, k, PT_.d(), ldT_);
        gemm(n_, INV_.d(), n_, n_, PT_.d(), ldT_, k, 1.0, 0.0, y.p, y.ld);
    }
    void factor_shift_invert();

    template <class R>
    void push(int j, const R& rep, int n_now, Event ev, int lock) {
        Record r{j, rep.overall, n_now, ev, lock, meter_.w};
        r.work.rr_dim = meter_.iter_rr_dim;
        out_.history.push_back(r);
        out_.margins.insert(out_.margins.end(), {rep.lo, rep.hi, rep.warm, rep.slope});
    }
    void truncate_history(size_t records) {
        out_.history.resize(records);
        out_.margins.resize(4 * records);
    }
    void finish(Status status, Blk v, int n_ev) {
        sync();
        check_syev();
        out_.status = status;
        out_.values.resize(n_ev);
        BKC(cudaMemcpyAsync(out_.values.data(), VALS_.d(), n_ev * sizeof(double), cudaMemcpyDeviceToHost, stream_));
        // beig_solve_ext.vectors_device: the vectors stay on the device
        double* cm = cfg_.vectors_device ? cfg_.vectors_device : PT_.d();
        if (cw_ == 1) BKC(bk_rm_to_cm_d(n_, n_ev, v.p, v.ld, cm, n_, st()));
        else BKC(bk_rm_to_cm_z(n_, n_ev, v.p, v.ld, cm, n_, st()));
        out_.complex_vectors = cw_ == 2;
        if (!cfg_.vectors_device) {
            out_.vectors.resize(static_cast<size_t>(n_) * n_ev * cw_);
            chunked_d2h(out_.vectors.data(), PT_.d(), out_.vectors.size());
        }
        sync();
        if (cfg_.largest)
            for (auto& x : out_.values) x = -x;
        out_.iterations = static_cast<int>(out_.history.size());
        out_.work = meter_.w;
        out_.work.rr_dim = meter_.iter_rr_dim;
        out_.rr_flops = meter_.rr_flops;
        out_.cgs2_fallbacks = fallbacks_;
        out_.spmm_windowed = spmm_win_calls_;
        if (std::getenv("BLOCKEIG_TIMING"))
            std::fprintf(stderr, "[blockeig] second Gram-Schmidt pass taken in %lld of %lld orthonormalisations; "
                         "speculative iterations %lld, redone %lld\n",
                         static_cast<long long>(pass2_), static_cast<long long>(proj_calls_),
                         static_cast<long long>(spec_runs_), static_cast<long long>(spec_redos_));
        out_.max_jacobi_sweeps = max_sweeps_;
        prof_resolve();
        if (std::getenv("BLOCKEIG_TIMING"))
            std::fprintf(stderr,
                         "[blockeig] syncs=%lld host_wait_in_sync=%.3fs host_in_calls=%.3fs phases: other=%.3f "
                         "resid=%.3f W=%.3f rr=%.3f hl=%.3f lift=%.3f tail=%.3f expand=%.3f\n",
                         static_cast<long long>(syncs_), sync_wait_s_, g_host_call_s, phase_s_[0], phase_s_[1],
                         phase_s_[2], phase_s_[3], phase_s_[4], phase_s_[5], phase_s_[6], phase_s_[7]);
        if (std::getenv("BLOCKEIG_TIMING"))
            std::fprintf(stderr, "[blockeig] device gaps before class (ms): spmm=%.1f gram=%.1f gemm=%.1f syev=%.1f "
                         "chol=%.1f resid=%.1f other=%.1f; host rng %.3fs for %lld cols\n",
                         gap_ms_[0], gap_ms_[1], gap_ms_[2], gap_ms_[3], gap_ms_[4], gap_ms_[5], gap_ms_[6],
                         rng_s_, static_cast<long long>(rng_cols_));
        for (int c = 0; c < K_CLASSES; ++c) out_.kstats[c] = kstats_[c];
    }

    int initial_block(const double* x0, int x0_cols, Blk dst);
    void solve_si();
    void solve_sd();
    void solve_lobpcg();
    void solve_tracemin();

    const SparseSym& a_;
    SolverConfig cfg_;
    SolverKind kind_;
    int n_;
    int cw_;  // doubles per scalar element: 1 real, 2 complex128
    NormalPairStream rng_;  // the reference's per-solve mt19937_64 normal stream, produced ahead
    const DeviceCsr* csr_ = nullptr;
    cudaStream_t stream_ = nullptr;
    int tcap_ = 0, dcap_ = 0, ldS_ = 0, ldT_ = 0, ldH_ = 0;
    DevMem S_[2], AS_, R_, XD_, T1_, T2_, PT_, VEC_, H_, Z_, ZC_, CZ_, VALS_, COEF_, GB_, M1_, M2_, SMALL_,
        INFO_, WORK_, TD_, INV_, stage_, CEXP_, VALS_BAK_;
    std::unique_ptr<SpChol> spchol_;
    DevMem cg_cnt_;  // TraceMIN: live CG columns per step
    DevMem CG_[6];
    // pinned staging is per host thread and outlives the solve (cudaFreeHost
    // synchronises the device and costs ms per solve)
    static Pinned& pinned() {
        static thread_local Pinned* p = new Pinned;
        return *p;
    }
    Pinned& pin_ = pinned();
    double norm_a_ = 0.0;
    std::future<double> norm_job_;
    Meter meter_;
    SolveOutput out_;
    int fallbacks_ = 0, max_sweeps_ = 0;
    int64_t pass2_ = 0, proj_calls_ = 0;  // DGKS second passes taken / orthonormalisations
    int spec_expect_[4] = {-1, -1, -1, -1};  // speculative K4 slots: assumed kept count (-1: unused)
    int64_t spec_runs_ = 0, spec_redos_ = 0;
    int spec_cooldown_ = 0;
    // after a sync: did every speculative K4 call keep all its columns, decisively?
    bool spec_ok() {
        bool ok = true;
        for (int s = 0; s < 4; ++s) {
            if (spec_expect_[s] < 0) continue;
            const int* inf = pin_.info + 16 + 4 * s;
            pass2_ += inf[3];
            if (inf[2]) throw std::runtime_error("orthonormalization: non-finite values");
            if (inf[1] || inf[0] != spec_expect_[s]) ok = false;
            spec_expect_[s] = -1;
        }
        return ok;
    }
    bool syev_pending_ = false;
    const bool debug_ = std::getenv("BLOCKEIG_DEBUG") != nullptr;
    int cur_ = 0;  // which S buffer holds the current block
    int xd_cols_ = 0;
    const double* x0_ = nullptr;
    int x0_cols_ = 0;
};

// Dense factor of A - zeta I for the reference's shift-and-invert SI (the
// SpdFactor dense path, kernel.cpp:102-137, n <= 2000): K4's Cholesky kernel
// without dropping gives M = R^{-1}, so (A - zeta I)^{-1} = M M^T.
void Engine::factor_shift_invert() {
    if (cw_ != 1)
        throw std::invalid_argument("shift-and-invert SI: complex matrices need the shifted operator mode");
    if (n_ > 2000) {  // reference sparse path (SimplicialLLT, AMD): host symbolic, device numeric
        spchol_ = std::make_unique<SpChol>(a_, cfg_.largest ? -1.0 : 1.0, cfg_.shift, stream_);
        return;
    }
    const size_t nn = static_cast<size_t>(n_) * n_;
    std::vector<double> dense(nn, 0.0);
    const double sgn = cfg_.largest ? -1.0 : 1.0;
    for (int r = 0; r < n_; ++r)
        for (int64_t p = a_.row_ptr()[r]; p < a_.row_ptr()[r + 1]; ++p) {
            const int c = a_.col()[p];
            dense[static_cast<size_t>(r) * n_ + c] = sgn * a_.val()[p];
            dense[static_cast<size_t>(c) * n_ + r] = sgn * a_.val()[p];
        }
    for (int i = 0; i < n_; ++i) dense[static_cast<size_t>(i) * n_ + i] -= cfg_.shift;
    DevMem g(nn * sizeof(double)), work(bk_chol_work_bytes(n_));
    INV_.alloc(nn * sizeof(double));
    BKC(cudaMemcpyAsync(g.d(), dense.data(), nn * sizeof(double), cudaMemcpyHostToDevice, stream_));
    int* info = INFO_.as<int>() + 16;
    BKC(bk_chol_drop_d(n_, g.d(), n_, nullptr, 0.0, INV_.d(), n_, info, work.p(), st()));
    BKC(cudaMemcpyAsync(pin_.info + 4, info, 3 * sizeof(int), cudaMemcpyDeviceToHost, stream_));
    sync();
    if (pin_.info[4] != n_ || pin_.info[6]) throw std::runtime_error("SpdFactor: matrix is not positive definite");
}

// solvers.cpp:82-96
int Engine::initial_block(const double* x0, int x0_cols, Blk dst) {
    const int n_ex = cfg_.n_ex;
    if (x0 != nullptr) {
        if (x0_cols != n_ex) throw std::invalid_argument("initial block must be n x n_ex");
        if (cfg_.x0_on_device) {
            // device-resident x0 (beig_solve_ext.x0_on_device): transposed in place
            // into the row-major block, no host staging
            if (cw_ == 1) BKC(bk_cm_to_rm_d(n_, n_ex, x0, n_, T1().p, T1().ld, st()));
            else BKC(bk_cm_to_rm_z(n_, n_ex, x0, n_, T1().p, T1().ld, st()));
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            upload_colmajor(x0, n_ex, T1());
            if (std::getenv("BLOCKEIG_TIMING"))
                std::fprintf(stderr, "[blockeig] x0 upload %.4fs (%.2f GB)\n",
                             std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                             1e-9 * n_ * n_ex * cw_ * sizeof(double));
        }
    } else {
        random_block(n_ex, T1());
    }
    meter_.ortho(n_, n_ex);
    const int kept = proj_ortho(n_, T1(), n_ex, B(nullptr, 0), 0, dst);
    if (x0 != nullptr && kept < n_ex) throw std::invalid_argument("initial block is rank deficient");
    if (kept < n_ex) fresh_cols(n_ex - kept, dst, kept);
    return n_ex;
}

// solvers.cpp:204-259 (+ operator mode).  Speculative like LOBPCG (one host
// readback per iteration): the head (residual, stagnation guard, decision,
// Y = op(V) into T1, expansion) runs synchronously; the tail (orthonormalise
// Y into S, Rayleigh-Ritz, lift, shrink) is enqueued assuming the
// orthonormalisation keeps every column and is redone from T1 (untouched by
// the tail) if the next record shows otherwise.
void Engine::solve_si() {
    const int n_ex = cfg_.n_ex, n_es = cfg_.n_es, n_ev = cfg_.n_ev;
    if (!cfg_.op_shifted) factor_shift_invert();
    initial_block(x0_, x0_cols_, S(cur_));
    rayleigh_ritz(S(cur_), n_ex, 0);
    lift(S(cur_), n_ex, Z_.d(), ldH_, n_ex, S(1 - cur_));
    cur_ ^= 1;
    int n_now = n_ex;
    BlockSizer sizer(strategy_);
    Stagnation guard;
    const Blk xd = B(XD_.d(), ldT_);
    static const bool spec_off = std::getenv("BLOCKEIG_NO_SPEC") != nullptr;
    auto tail = [&](int j, const Rep& rep, Decision d, int ycols, Event ev, bool spec) {
        meter_.ortho(n_, ycols);
        const int kept = proj_ortho(n_, T1(), ycols, B(nullptr, 0), 0, S(cur_), spec ? 0 : -1);
        if (kept < n_now) fresh_cols(n_now - kept, S(cur_), kept);
        rayleigh_ritz(S(cur_), n_now, 0);
        lift(S(cur_), n_now, Z_.d(), ldH_, n_now, S(1 - cur_));
        cur_ ^= 1;
        if (d == Decision::shrink) {
            copy(n_, S(cur_).at(n_es), n_now - n_es, xd);
            xd_cols_ = n_now - n_es;
            n_now = n_es;
            ev = Event::shrink;
        }
        push(j, rep, n_now, ev, 0);
    };
    struct Snap {
        int j, cur, n_now, xd_cols, ycols;
        Event ev;
        Decision d;
        Rep rep;
        Meter meter;
        size_t hist;
    };
    Snap snap{};
    bool spec_pending = false;
    auto settle = [&](const Rep& rep) -> bool {  // true if the previous tail was redone
        if (!spec_pending) return false;
        spec_pending = false;
        if (spec_ok() && !rep.nonfinite) return false;
        ++spec_redos_;
        spec_cooldown_ = 8;  // failing speculations: stay synchronous for a while
        cur_ = snap.cur;
        n_now = snap.n_now;
        xd_cols_ = snap.xd_cols;
        meter_ = snap.meter;
        truncate_history(snap.hist);
        tail(snap.j, snap.rep, snap.d, snap.ycols, snap.ev, false);
        return true;
    };
    for (int j = 1; j <= cfg_.max_iters; ++j) {
        meter_.begin_iteration();
        Rep rep = residual(S(cur_), n_now, n_ev, spec_pending);
        if (settle(rep)) {
            meter_.begin_iteration();
            rep = residual(S(cur_), n_now, n_ev, false);
        }
        const Blk v = S(cur_);
        if (rep.converged >= n_ev) {
            push(j, rep, n_now, Event::none, 0);
            return finish(Status::converged, v, n_ev);
        }
        if (guard.update(j, rep.overall)) {
            push(j, rep, n_now, Event::none, 0);
            return finish(Status::stagnated, v, n_ev);
        }
        const Decision d = sizer.step(rep.overall, n_now, n_es, n_ex);
        rep.note(sizer);
        meter_.w.solve_cols += n_now;
        apply_op(v, n_now, AS(), true, T1());
        if (cfg_.expand == ExpandMode::powered && xd_cols_ > 0) {
            meter_.w.solve_cols += xd_cols_;
            apply_op(xd, xd_cols_, AS(), false, xd);
        }
        Event ev = Event::none;
        int ycols = n_now;
        if (d == Decision::expand) {
            const int e = cfg_.expand == ExpandMode::random ? n_ex - n_now : xd_cols_;
            if (e > 0) {
                if (cfg_.expand == ExpandMode::random) random_block(e, T1().at(n_now));
                else copy(n_, xd, e, T1().at(n_now));
                ycols += e;
                xd_cols_ = 0;
                n_now = n_ex;
                ev = Event::expand;
            }
        }
        const bool spec = !spec_off && d != Decision::expand && spec_cooldown_ == 0;
        if (spec_cooldown_ > 0) --spec_cooldown_;
        if (spec) {
            snap = Snap{j, cur_, n_now, xd_cols_, ycols, ev, d, rep, meter_, out_.history.size()};
            ++spec_runs_;
        }
        tail(j, rep, d, ycols, ev, spec);
        spec_pending = spec;
    }
    sync();
    settle(Rep{0.0, 0, false});
    finish(Status::max_iters, S(cur_), n_ev);
}

// solvers.cpp:261-314.  Speculative tail as for LOBPCG: X = S(cur)[:, 0:n_now],
// AX and R are not overwritten by the tail, so a failed speculation is redone
// from them.
void Engine::solve_sd() {
    const int n_ex = cfg_.n_ex, n_es = cfg_.n_es, n_ev = cfg_.n_ev;
    initial_block(x0_, x0_cols_, S(cur_));
    rayleigh_ritz(S(cur_), n_ex, 0);
    lift(S(cur_), n_ex, Z_.d(), ldH_, n_ex, S(1 - cur_));
    cur_ ^= 1;
    int n_now = n_ex;
    BlockSizer sizer(strategy_);
    const Blk xd = B(XD_.d(), ldT_);
    const double* td = TD_.bytes() ? TD_.d() : nullptr;
    static const bool spec_off = std::getenv("BLOCKEIG_NO_SPEC") != nullptr;
    // false when the solve ended inside
    auto tail = [&](int j, const Rep& rep, Decision d, bool spec) -> bool {
        const Blk v = S(cur_);
        Event ev = Event::none;
        const int n_old = n_now;
        int xb = n_now;
        if (d == Decision::expand) {
            const int e = cfg_.expand == ExpandMode::random ? n_ex - n_now : xd_cols_;
            if (e > 0) {
                if (cfg_.expand == ExpandMode::random) random_block(e, T1());
                else copy(n_, xd, e, T1());
                meter_.proj_ortho(n_, e, xb);
                xb += proj_ortho(n_, T1(), e, v, xb, v.at(xb));
                if (xb < n_ex) {
                    fresh_cols(n_ex - xb, v, xb);
                    xb = n_ex;
                }
                xd_cols_ = 0;
                n_now = n_ex;
                ev = Event::expand;
            }
        }
        scale_rows(n_, n_old, td, B(R_.d(), ldT_), T1());
        meter_.proj_ortho(n_, n_old, xb);
        const int kw = proj_ortho(n_, T1(), n_old, v, xb, v.at(xb), spec ? 0 : -1);
        if (kw == 0) {
            push(j, rep, n_now, ev, 0);
            finish(Status::stagnated, v, n_ev);
            return false;
        }
        const int ds = xb + kw;
        rayleigh_ritz(v, ds, n_old, n_now);
        lift(v, ds, Z_.d(), ldH_, n_now, S(1 - cur_));
        cur_ ^= 1;
        if (d == Decision::shrink) {
            copy(n_, S(cur_).at(n_es), n_now - n_es, xd);
            xd_cols_ = n_now - n_es;
            n_now = n_es;
            ev = Event::shrink;
        }
        push(j, rep, n_now, ev, 0);
        return true;
    };
    struct Snap {
        int j, cur, n_now, xd_cols;
        Decision d;
        Rep rep;
        Meter meter;
        size_t hist;
    };
    Snap snap{};
    bool spec_pending = false;
    auto settle = [&](const Rep& rep) -> int {  // 0 ok, 1 redone, -1 solve ended
        if (!spec_pending) return 0;
        spec_pending = false;
        if (spec_ok() && !rep.nonfinite) return 0;
        ++spec_redos_;
        spec_cooldown_ = 8;  // failing speculations: stay synchronous for a while
        cur_ = snap.cur;
        n_now = snap.n_now;
        xd_cols_ = snap.xd_cols;
        meter_ = snap.meter;
        truncate_history(snap.hist);
        restore_residual(S(cur_), n_now);  // R, AX of the redone iteration
        return tail(snap.j, snap.rep, snap.d, false) ? 1 : -1;
    };
    for (int j = 1; j <= cfg_.max_iters; ++j) {
        meter_.begin_iteration();
        Rep rep = residual(S(cur_), n_now, n_ev, spec_pending);
        const int st = settle(rep);
        if (st < 0) return;
        if (st > 0) {
            meter_.begin_iteration();
            rep = residual(S(cur_), n_now, n_ev, false);
        }
        if (rep.converged >= n_ev) {
            push(j, rep, n_now, Event::none, 0);
            return finish(Status::converged, S(cur_), n_ev);
        }
        const Decision d = sizer.step(rep.overall, n_now, n_es, n_ex);
        rep.note(sizer);
        const bool spec = !spec_off && d != Decision::expand && spec_cooldown_ == 0;
        if (spec_cooldown_ > 0) --spec_cooldown_;
        if (spec) {
            snap = Snap{j, cur_, n_now, xd_cols_, d, rep, meter_, out_.history.size()};
            save_ritz(n_now);
            ++spec_runs_;
        }
        if (!tail(j, rep, d, spec)) return;
        spec_pending = spec;
    }
    sync();
    if (settle(Rep{0.0, 0, false}) < 0) return;
    finish(Status::max_iters, S(cur_), n_ev);
}

// solvers.cpp:316-401.  Layout of the current buffer: [X (n_now) | P (np)],
// with W appended after P inside the iteration.
//
// One host readback per iteration: the two orthonormalisations of an
// iteration (W against [X, P] and the HL trick's coefficient block) run
// speculatively — the iteration is enqueued as if both kept all their columns
// (the common case) and their Cholesky infos travel back with the next
// residual record.  If a speculation failed (a column dropped, or an
// undecided pivot), the iteration is restored from its snapshot (host scalars,
// meter, history; the device state it started from — [X, P], AX, R — is not
// overwritten by the speculative tail) and redone with synchronous decisions.
// Expansion iterations are always synchronous.  BLOCKEIG_NO_SPEC=1 disables it.
void Engine::solve_lobpcg() {
    const int n_ex = cfg_.n_ex, n_es = cfg_.n_es, n_ev = cfg_.n_ev;
    initial_block(x0_, x0_cols_, S(cur_));
    rayleigh_ritz(S(cur_), n_ex, 0);
    lift(S(cur_), n_ex, Z_.d(), ldH_, n_ex, S(1 - cur_));
    cur_ ^= 1;
    int n_now = n_ex, np = 0, prev_lock = 0;
    BlockSizer sizer(strategy_);
    const Blk xd = B(XD_.d(), ldT_);
    static const bool spec_off = std::getenv("BLOCKEIG_NO_SPEC") != nullptr;

    // everything after the decision; false when the solve ended inside
    auto tail = [&](int j, const Rep& rep, int lock, Decision d, bool spec) -> bool {
        Blk s = S(cur_);
        const int active = n_now - lock;
        // W = T R(:, lock:) (written by the residual kernel) orthonormalised against [X, P]
        int m = n_now + np;
        meter_.proj_ortho(n_, active, m);
        mark(0);
        const int kw = proj_ortho(n_, T1().at(lock), active, s, m, s.at(m), spec ? 0 : -1, w_norms() + lock);
        mark(2);
        if (kw == 0) {
            push(j, rep, n_now, Event::none, lock);
            finish(Status::stagnated, s, n_ev);
            return false;
        }
        Event ev = Event::none;
        const int n_old = n_now;
        int ds = m + kw;
        if (d == Decision::expand) {
            const int want = 2 * (n_ex - n_es);
            const int e = cfg_.expand == ExpandMode::random ? want : xd_cols_;
            if (e > 0) {
                if (cfg_.expand == ExpandMode::random) random_block(e, T1());
                else copy(n_, xd, e, T1());
                meter_.proj_ortho(n_, e, ds);
                const int oe = proj_ortho(n_, T1(), e, s, ds, T2());
                const int hx = std::min((oe + 1) / 2, n_ex - n_now);
                // other buffer: [X | oe(:, :hx) | P | oe(:, hx:) | W]
                Blk o = S(1 - cur_);
                int c = 0;
                copy(n_, s, n_now, o);
                c += n_now;
                copy(n_, T2(), hx, o.at(c));
                c += hx;
                const int xb = c;
                copy(n_, s.at(n_now), np, o.at(c));
                c += np;
                copy(n_, T2().at(hx), oe - hx, o.at(c));
                c += oe - hx;
                const int pn = np + oe - hx;
                copy(n_, s.at(m), kw, o.at(c));
                c += kw;
                if (xb < n_ex) {
                    // fresh columns orthogonal to [xb, p, W]; then insert them after xb
                    const int f = n_ex - xb;
                    fresh_cols(f, o, c);
                    copy(n_, o, xb, s);
                    copy(n_, o.at(c), f, s.at(xb));
                    copy(n_, o.at(xb), pn + kw, s.at(n_ex));
                } else {
                    cur_ ^= 1;
                    s = S(cur_);
                }
                xd_cols_ = 0;
                n_now = n_ex;
                np = pn;
                ev = Event::expand;
                m = n_now + np;
                ds = m + kw;
            }
        }
        mark(7);
        // Rayleigh-Ritz on S = [X, P, W]; A X is still in AS(:, 0:n_old)
        mark(0);
        rayleigh_ritz(s, ds, n_old, n_now);
        mark(3);
        // HL trick (solvers.cpp:187-196): [X, P] = S [Z1, orth(Zp)] (n_now is post-expansion here)
        const int pk = hl_lift(s, ds, n_now, lock, S(1 - cur_), spec ? 1 : -1);
        mark(5);
        cur_ ^= 1;
        np = pk;
        if (d == Decision::shrink) {
            const Blk nx = S(cur_);
            const int dx = n_now - n_es;
            const int dp = np > n_es ? np - n_es : 0;
            copy(n_, nx.at(n_es), dx, xd);
            copy(n_, nx.at(n_now + n_es), dp, xd.at(dx));
            xd_cols_ = dx + dp;
            np = std::min(np, n_es);
            copy(n_, nx.at(n_now), np, nx.at(n_es));
            n_now = n_es;
            ev = Event::shrink;
        }
        if (ev == Event::none && lock > prev_lock) ev = Event::lock;
        push(j, rep, n_now, ev, lock);
        mark(6);
        prev_lock = lock;
        return true;
    };

    struct Snap {
        int j, cur, n_now, np, prev_lock, xd_cols, lock;
        Decision d;
        Rep rep;
        Meter meter;
        size_t hist;
    };
    Snap snap{};
    bool spec_pending = false;
    // verify the previous iteration's speculation (after a sync); redo it if needed
    auto settle = [&](const Rep& rep) -> int {  // 0 ok, 1 redone, -1 solve ended
        if (!spec_pending) return 0;
        spec_pending = false;
        const bool ok = spec_ok();
        if (ok && !rep.nonfinite) return 0;
        ++spec_redos_;
        spec_cooldown_ = 8;  // failing speculations: stay synchronous for a while
        cur_ = snap.cur;
        n_now = snap.n_now;
        np = snap.np;
        prev_lock = snap.prev_lock;
        xd_cols_ = snap.xd_cols;
        meter_ = snap.meter;
        truncate_history(snap.hist);
        restore_residual(S(cur_), n_now);  // R, AX of the redone iteration
        return tail(snap.j, snap.rep, snap.lock, snap.d, false) ? 1 : -1;
    };
    for (int j = 1; j <= cfg_.max_iters; ++j) {
        meter_.begin_iteration();
        mark(0);
        Rep rep = residual(S(cur_), n_now, n_ev, spec_pending);
        mark(1);
        const int st = settle(rep);
        if (st < 0) return;
        if (st > 0) {
            meter_.begin_iteration();
            rep = residual(S(cur_), n_now, n_ev, false);
        }
        Blk s = S(cur_);
        const int lock = std::min(rep.converged, n_now - 1);
        if (rep.converged >= n_ev) {
            push(j, rep, n_now, Event::none, lock);
            return finish(Status::converged, s, n_ev);
        }
        const Decision d = sizer.step(rep.overall, n_now, n_es, n_ex);
        rep.note(sizer);
        // soft locking: P loses its leading (lock - prev_lock) columns
        if (lock > prev_lock && np > 0) {
            const int drop = std::min(lock - prev_lock, np);
            copy(n_, s.at(n_now + drop), np - drop, s.at(n_now));
            np -= drop;
        }
        const bool spec = !spec_off && d != Decision::expand && spec_cooldown_ == 0;
        if (spec_cooldown_ > 0) --spec_cooldown_;
        if (spec) {
            snap = Snap{j, cur_, n_now, np, prev_lock, xd_cols_, lock, d, rep, meter_, out_.history.size()};
            save_ritz(n_now);
            ++spec_runs_;
        }
        if (!tail(j, rep, lock, d, spec)) return;
        spec_pending = spec;
    }
    // the last iteration may still be speculative: settle it before finishing
    sync();
    if (settle(Rep{0.0, 0, false}) < 0) return;
    finish(Status::max_iters, S(cur_), n_ev);
}

// solvers.cpp:403-463 with cg_solve (kernel.cpp:139-164) batched over columns
void Engine::solve_tracemin() {
    const int n_ex = cfg_.n_ex, n_es = cfg_.n_es, n_ev = cfg_.n_ev;
    initial_block(x0_, x0_cols_, S(cur_));
    rayleigh_ritz(S(cur_), n_ex, 0);
    lift(S(cur_), n_ex, Z_.d(), ldH_, n_ex, S(1 - cur_));
    cur_ ^= 1;
    const size_t blk = static_cast<size_t>(std::max(n_, 1)) * ldT_ * sizeof(double) * cw_;
    for (int i = 0; i < 4; ++i) CG_[i].alloc(blk);
    CG_[4].alloc(8 * static_cast<size_t>(tcap_) * sizeof(double));
    CG_[5].alloc(static_cast<size_t>(tcap_) * sizeof(int) + 64);
    const Blk cx = B(CG_[0].d(), ldT_), cr = B(CG_[1].d(), ldT_), cp = B(CG_[2].d(), ldT_), cap = B(CG_[3].d(), ldT_);
    double* rs = CG_[4].d();
    double* bnorm = rs + tcap_;
    double* pap = rs + 2 * tcap_;
    double* rs_new = rs + 3 * tcap_;
    int* act = CG_[5].as<int>();
    int n_now = n_ex;
    BlockSizer sizer(strategy_);
    const Blk xd = B(XD_.d(), ldT_);
    for (int j = 1; j <= cfg_.max_iters; ++j) {
        meter_.begin_iteration();
        const Blk v = S(cur_);
        Rep rep = residual(v, n_now, n_ev);
        if (rep.converged >= n_ev) {
            push(j, rep, n_now, Event::none, 0);
            return finish(Status::converged, v, n_ev);
        }
        const Decision d = sizer.step(rep.overall, n_now, n_es, n_ex);
        rep.note(sizer);
        const int k = n_now;
        // project(u) = u - V (V^T u), in place
        auto project = [&](Blk u) {
            gram(n_, v.p, v.ld, k, u.p, u.ld, k, COEF_.d(), k);
            gemm(n_, v.p, v.ld, k, COEF_.d(), k, k, -1.0, 1.0, u.p, u.ld);
        };
        // rhs = P_V R; x = 0; p = r = rhs
        copy(n_, B(R_.d(), ldT_), k, cr);
        project(cr);
        BKO(bk_axpby_d(n_, k * cw_, 0.0, cr.p, cr.ld * cw_, 0.0, cx.p, cx.ld * cw_, st()));
        copy(n_, cr, k, cp);
        colnorm2(n_, cr, k, rs);
        BKC(bk_cg_init_d(k, rs, bnorm, act, st()));
        // all cg_iters steps are enqueued without a host round trip: a column
        // whose CG stopped (kernel.cpp:151,153) is frozen by its device flag, so
        // the steps after the last live column change nothing; the live counts
        // per step (the work meter's spmv_cols) come back in one readback
        const int steps = cfg_.cg_iters;
        if (cg_cnt_.bytes() < steps * sizeof(int)) cg_cnt_.alloc(steps * sizeof(int));
        int* cnt = cg_cnt_.as<int>();
        for (int it = 0; it < steps; ++it) {
            BKC(bk_cg_check_d(k, rs, bnorm, act, cnt + it, st()));
            // ap = P_V A P_V p
            copy(n_, cp, k, T2());
            project(T2());
            spmm(T2(), k, cap);
            project(cap);
            if (cw_ == 1) {
                BKC(bk_coldot_d(n_, cp.p, cp.ld, cap.p, cap.ld, k, pap, WORK_.p(), st()));
                BKC(bk_cg_step1_d(n_, k, rs, pap, act, cx.p, cx.ld, cr.p, cr.ld, cp.p, cp.ld, cap.p, cap.ld, st()));
            } else {
                BKC(bk_coldot_z(n_, cp.p, cp.ld, cap.p, cap.ld, k, pap, WORK_.p(), st()));
                BKC(bk_cg_step1_z(n_, k, rs, pap, act, cx.p, cx.ld, cr.p, cr.ld, cp.p, cp.ld, cap.p, cap.ld, st()));
            }
            colnorm2(n_, cr, k, rs_new);
            if (cw_ == 1) BKC(bk_cg_step2_d(n_, k, rs, rs_new, act, cr.p, cr.ld, cp.p, cp.ld, st()));
            else BKC(bk_cg_step2_z(n_, k, rs, rs_new, act, cr.p, cr.ld, cp.p, cp.ld, st()));
        }
        {
            std::vector<int> live(steps);
            BKC(cudaMemcpyAsync(live.data(), cnt, steps * sizeof(int), cudaMemcpyDeviceToHost, stream_));
            sync();
            for (int it = 0; it < steps && live[it] > 0; ++it) meter_.w.spmv_cols += live[it];
        }
        // y = V - delta
        lincomb(n_, k, 1.0, v, -1.0, cx, T1());
        Event ev = Event::none;
        int ycols = n_now;
        if (d == Decision::expand) {
            const int e = cfg_.expand == ExpandMode::random ? n_ex - n_now : xd_cols_;
            if (e > 0) {
                if (cfg_.expand == ExpandMode::random) random_block(e, T1().at(n_now));
                else copy(n_, xd, e, T1().at(n_now));
                ycols += e;
                xd_cols_ = 0;
                n_now = n_ex;
                ev = Event::expand;
            }
        }
        meter_.ortho(n_, ycols);
        const int kept = proj_ortho(n_, T1(), ycols, B(nullptr, 0), 0, S(cur_));
        if (kept < n_now) fresh_cols(n_now - kept, S(cur_), kept);
        rayleigh_ritz(S(cur_), n_now, 0);
        lift(S(cur_), n_now, Z_.d(), ldH_, n_now, S(1 - cur_));
        cur_ ^= 1;
        if (d == Decision::shrink) {
            copy(n_, S(cur_).at(n_es), n_now - n_es, xd);
            xd_cols_ = n_now - n_es;
            n_now = n_es;
            ev = Event::shrink;
        }
        push(j, rep, n_now, ev, 0);
    }
    finish(Status::max_iters, S(cur_), n_ev);
}

SolveOutput Engine::run(const double* x0, int x0_cols) {
    x0_ = x0;
    x0_cols_ = x0_cols;
    switch (kind_) {
        case SolverKind::si: solve_si(); break;
        case SolverKind::sd: solve_sd(); break;
        case SolverKind::lobpcg: solve_lobpcg(); break;
        case SolverKind::tracemin: solve_tracemin(); break;
    }
    return std::move(out_);
}

}  // namespace

// solvers.cpp:147-169 (+ extension checks)
SolverConfig resolve_config(SolverConfig cfg, SolverKind kind, const StrategyConfig& s, int n) {
    if (n < 1) throw std::invalid_argument("matrix is empty");
    if (cfg.n_ev < 1) throw std::invalid_argument("n_ev must be positive");
    if (cfg.n_ev > n) throw std::invalid_argument("n_ev exceeds the matrix dimension");
    if (cfg.n_ex == 0) {
        const double mult = kind == SolverKind::lobpcg ? 1.5 : 2.0;
        cfg.n_ex = std::min(n, static_cast<int>(std::ceil(mult * cfg.n_ev)));
    }
    const bool nes_given = cfg.n_es != 0;
    if (!nes_given) cfg.n_es = std::max(cfg.n_ev, std::min(cfg.n_ev + 5, cfg.n_ex - 1));
    if (cfg.n_ex < cfg.n_ev || cfg.n_ex > n) throw std::invalid_argument("need n_ev <= n_ex <= n");
    const bool se = s.kind != StrategyKind::none;
    if ((se || nes_given) && !(cfg.n_ev <= cfg.n_es && cfg.n_es < cfg.n_ex))
        throw std::invalid_argument("need n_ev <= n_es < n_ex");
    if (!(cfg.tol > 0)) throw std::invalid_argument("tol must be positive");
    if (cfg.max_iters < 1) throw std::invalid_argument("max_iters must be positive");
    if (cfg.cg_iters < 1) throw std::invalid_argument("cg_iters must be positive");
    if (cfg.expand == ExpandMode::powered && kind != SolverKind::si)
        throw std::invalid_argument("powered expansion vectors require the SI solver");
    if (cfg.op_shifted && kind != SolverKind::si)
        throw std::invalid_argument("the shifted operator mode applies to the SI solver only");
    validate_strategy(s);
    // extension check (no reference counterpart: Eigen has no size limit): the
    // Rayleigh-Ritz dimension is at most n_ex (SI, TraceMIN), 2 n_ex (SD) or
    // 3 n_ex (LOBPCG, expansion iterations included), capped by n; the device
    // eigensolver K5 handles d <= kMaxRitzDim, so larger problems are refused
    // here, before any device work, instead of failing mid-solve
    {
        const int64_t f = kind == SolverKind::lobpcg ? 3 : kind == SolverKind::sd ? 2 : 1;
        const int64_t dmax = std::min<int64_t>(n, f * cfg.n_ex);
        if (dmax > kMaxRitzDim)
            throw std::invalid_argument("Rayleigh-Ritz dimension " + std::to_string(dmax) +
                                        " exceeds the device eigensolver limit " + std::to_string(kMaxRitzDim) +
                                        " (LOBPCG: 3 n_ex, SD: 2 n_ex, SI/TraceMIN: n_ex)");
    }
    return cfg;
}

// Harness engines: identity matrix of order n (only the block machinery is
// used), widths sized for the call.
namespace {
SparseSym harness_identity(int n) {
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1);
    std::vector<int> col(n);
    for (int i = 0; i <= n; ++i) rp[i] = i;
    for (int i = 0; i < n; ++i) col[i] = i;
    return SparseSym(n, std::move(rp), std::move(col), std::vector<double>(n, 1.0));
}
SolverConfig harness_cfg(int width, int device) {
    SolverConfig c;
    c.n_ev = 1;
    c.n_ex = std::max(width, 2);
    c.n_es = c.n_ex - 1;
    c.device = device;
    return c;
}
}  // namespace

int harness_project_orthonormalize(const double* w, int n, int a, const double* q, int m, double* out, int device) {
    if (n < 1 || a < 0 || m < 0 || a + m > n) throw std::invalid_argument("harness: bad block sizes");
    const SparseSym id = harness_identity(n);
    Engine e(id, harness_cfg(std::max(a, m), device), SolverKind::lobpcg);
    return e.harness_proj_ortho(w, a, q, m, out);
}

int harness_hl_trick(const double* s, int n, int d, const double* z, int n_now, int lock, double* x, double* p,
                     int device) {
    // reference hl_trick argument checks (solvers.cpp:187-190)
    if (n_now < 1 || n_now > d) throw std::invalid_argument("hl_trick: bad n_now");
    lock = std::clamp(lock, 0, n_now);
    if (d > n) throw std::invalid_argument("harness: d exceeds n");
    const SparseSym id = harness_identity(n);
    Engine e(id, harness_cfg(d, device), SolverKind::lobpcg);
    return e.harness_hl(s, d, z, n_now, lock, x, p);
}

SolveOutput solve(SolverKind kind, const SparseSym& a, const SolverConfig& cfg_in, const StrategyConfig& s,
                  const double* x0, int x0_cols) {
    const auto t0 = std::chrono::steady_clock::now();
    const SolverConfig cfg = resolve_config(cfg_in, kind, s, a.rows());
    SolveOutput out;
    double t_setup = 0.0, t_run = 0.0;
    {
        Engine e(a, cfg, kind);
        e.set_strategy(s);
        t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out = e.run(x0, x0_cols);
        t_run = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() - t_setup;
    }
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (std::getenv("BLOCKEIG_TIMING"))
        std::fprintf(stderr, "[blockeig] solve: setup %.4fs run %.4fs teardown %.4fs\n", t_setup, t_run,
                     out.seconds - t_setup - t_run);
    return out;
}

}  // namespace b2
