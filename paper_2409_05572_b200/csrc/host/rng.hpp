// Background generator of the reference's normal variates.
//
// The reference draws every random block (X0 when none is given, refill
// columns, random expansion vectors) with a FRESH std::normal_distribution over
// one std::mt19937_64 per solve (proj/src/kernel.cpp:166-172,
// solvers.cpp:209,265,320,407).  libstdc++'s normal_distribution is the polar
// method: each rejection-sampled pair (x, y) yields y*m first and caches x*m
// for the next call; a fresh distribution per block discards a cached value
// left at the end of a block.  So a block of N values consumes exactly
// ceil(N/2) pairs of one pair stream, whatever the block sizes are.
//
// This class produces that pair stream on a worker thread, ahead of demand,
// with the same arithmetic (std::generate_canonical<double, 53>, std::log,
// std::sqrt), so take() returns bit-identical values to the reference while
// the host generation overlaps the device work (it was 15% of a config-2
// solve when done inline at the point of use).
#pragma once

#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <limits>
#include <cstring>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

namespace b2 {

class NormalPairStream {
public:
    explicit NormalPairStream(uint64_t seed, size_t capacity_pairs = size_t{1} << 22)
        : rng_(seed), cap_(capacity_pairs), ring_(2 * capacity_pairs) {
        worker_ = std::thread([this] { run(); });
    }
    ~NormalPairStream() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        worker_.join();
    }
    NormalPairStream(const NormalPairStream&) = delete;
    NormalPairStream& operator=(const NormalPairStream&) = delete;

    // one random_block of `count` values (column-major fill order)
    void take(double* out, size_t count) {
        const size_t pairs = (count + 1) / 2;
        size_t done = 0;  // pairs consumed by this call
        while (done < pairs) {
            size_t avail;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return produced_ > head_; });
                avail = produced_ - head_;
            }
            const size_t use = std::min(avail, pairs - done);
            // the ring holds (y * mult, x * mult) pairs in output order: copy the
            // (at most two) contiguous ring segments; an odd block drops the last x
            for (size_t p = 0; p < use;) {
                const size_t slot = (head_ + p) % cap_;
                const size_t seg = std::min(use - p, cap_ - slot);
                const size_t i = 2 * (done + p);
                const size_t n = std::min(2 * seg, count - i);
                std::memcpy(out + i, ring_.data() + 2 * slot, n * sizeof(double));
                p += seg;
            }
            {
                std::lock_guard<std::mutex> lk(mu_);
                head_ += use;
            }
            cv_.notify_all();
            done += use;
        }
    }

private:
    void run() {
        constexpr size_t kChunk = 4096;
        for (;;) {
            size_t start, room;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || produced_ - head_ < cap_; });
                if (stop_) return;
                start = produced_;
                room = std::min(kChunk, cap_ - (produced_ - head_));
            }
            for (size_t p = 0; p < room; ++p) {
                double x, y, r2;
                do {
                    x = 2.0 * std::generate_canonical<double, std::numeric_limits<double>::digits>(rng_) - 1.0;
                    y = 2.0 * std::generate_canonical<double, std::numeric_limits<double>::digits>(rng_) - 1.0;
                    r2 = x * x + y * y;
                } while (r2 > 1.0 || r2 == 0.0);
                const double mult = std::sqrt(-2 * std::log(r2) / r2);
                const size_t slot = (start + p) % cap_;
                // normal_distribution(0, 1) applies ret * stddev + mean
                ring_[2 * slot] = y * mult * 1.0 + 0.0;
                ring_[2 * slot + 1] = x * mult * 1.0 + 0.0;
            }
            {
                std::lock_guard<std::mutex> lk(mu_);
                produced_ += room;
            }
            cv_.notify_all();
        }
    }

    std::mt19937_64 rng_;
    size_t cap_;
    std::vector<double> ring_;
    size_t produced_ = 0, head_ = 0;
    bool stop_ = false;
    std::mutex mu_;
    std::condition_variable cv_;
    std::thread worker_;
};

}  // namespace b2
