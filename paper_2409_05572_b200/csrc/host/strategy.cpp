// Block-size strategy (shrink-and-expand decisions): host code, O(1) per
// iteration, fed by the single convergence record read back from the device.
// Same decisions as proj/src/strategy.cpp:42-98 (fix / slope / slopek with the
// warm-up gate and c_max bookkeeping) — the code follows the reference's
// implementation, not the paper's printed j_l = j_e.
#include <algorithm>
#include <cmath>
#include <limits>

#include "host.hpp"

namespace b2 {

void validate_strategy(const StrategyConfig& c) {
    if (c.kind == StrategyKind::none) return;
    if (c.j_s < 1 || c.j_s >= c.j_e) throw std::invalid_argument("strategy: need 1 <= j_s < j_e");
    if (c.j_p < 1) throw std::invalid_argument("strategy: j_p must be positive");
    if (!(c.mu > 0)) throw std::invalid_argument("strategy: mu must be positive");
    if (c.j_warm < 0) throw std::invalid_argument("strategy: j_warm must be nonnegative");
    if (!(c.r_warm > 0)) throw std::invalid_argument("strategy: r_warm must be positive");
}

Decision BlockSizer::step(double r_now, int n_now, int n_es, int n_ex) {
    m_warm_ = m_slope_ = std::numeric_limits<double>::quiet_NaN();
    ++j_;
    lg_.push_back(std::log10(std::max(r_now, 1e-300)));
    if (c_.kind == StrategyKind::none) return Decision::hold;
    const bool wide = n_now >= n_ex;
    const bool narrow = !wide && n_now <= n_es;

    // warm-up: the first shrink needs the expanded state, j >= j_warm and r <= r_warm
    if (!warmed_) {
        if (wide && j_ >= c_.j_warm) m_warm_ = r_now / c_.r_warm;
        if (wide && j_ >= c_.j_warm && r_now <= c_.r_warm) {
            warmed_ = true;
            have_ref_ = false;
            c_max_ = 0.0;
            return Decision::shrink;
        }
        return Decision::hold;
    }

    if (c_.kind == StrategyKind::fix) {
        if (narrow && j_ % c_.j_e == 0) {
            last_expand_ = j_;
            return Decision::expand;
        }
        if (wide && (j_ - c_.j_s) % c_.j_e == 0) {
            have_ref_ = false;
            c_max_ = 0.0;
            return Decision::shrink;
        }
        return Decision::hold;
    }

    if (narrow) {
        const size_t need = c_.kind == StrategyKind::slope ? 2 : static_cast<size_t>(c_.j_p) + 1;
        if (lg_.size() < need) return Decision::hold;
        const size_t back = c_.kind == StrategyKind::slope ? 1 : static_cast<size_t>(c_.j_p);
        double c = lg_[lg_.size() - 1 - back] - lg_.back();
        if (c_.kind == StrategyKind::slopek) c /= c_.j_p;
        if (!have_ref_) {  // first slope after a shrink seeds the reference
            c_max_ = c;
            have_ref_ = true;
            return Decision::hold;
        }
        m_slope_ = c > 0.0 ? (c_max_ - c_.mu * c) / (c_.mu * c) : c_max_;
        const bool stalled = c > 0.0 ? c_max_ > c_.mu * c : c_max_ > 0.0;
        if (stalled) {
            last_expand_ = j_;
            return Decision::expand;
        }
        c_max_ = std::max(c_max_, c);
        return Decision::hold;
    }
    if (wide && last_expand_ >= 0 && j_ - last_expand_ == c_.j_s) {
        have_ref_ = false;
        c_max_ = 0.0;
        return Decision::shrink;
    }
    return Decision::hold;
}

}  // namespace b2

extern "C" int bk_host_decide_sequence(int kind, int j_e, int j_s, double mu, int j_p, int j_warm,
                                       double r_warm, const double* r, int count, int n_es, int n_ex,
                                       int start_n_now, int start_shrunk, int apply_changes,
                                       int* decisions) {
    try {
        b2::StrategyConfig c;
        c.kind = static_cast<b2::StrategyKind>(kind);
        c.j_e = j_e;
        c.j_s = j_s;
        c.mu = mu;
        c.j_p = j_p;
        c.j_warm = j_warm;
        c.r_warm = r_warm;
        b2::BlockSizer s(c);
        if (start_shrunk) s.mark_warmed();
        int n_now = start_n_now;
        for (int i = 0; i < count; ++i) {
            const auto d = s.step(r[i], n_now, n_es, n_ex);
            decisions[i] = static_cast<int>(d);
            if (apply_changes) {
                if (d == b2::Decision::expand) n_now = n_ex;
                if (d == b2::Decision::shrink) n_now = n_es;
            }
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

#include <cstring>

#include "rng.hpp"

// host-only hook: consecutive random blocks (sizes[i] values each) from one
// per-solve normal stream, as the solver draws them — CPU test of bit parity
// with std::normal_distribution over std::mt19937_64 (the reference's
// random_block, proj/src/kernel.cpp:166-172)
extern "C" int bk_host_normal_blocks(uint64_t seed, const int* sizes, int nblocks, double* out) {
    try {
        b2::NormalPairStream s(seed, 1024);
        size_t off = 0;
        for (int b = 0; b < nblocks; ++b) {
            s.take(out + off, static_cast<size_t>(sizes[b]));
            off += static_cast<size_t>(sizes[b]);
        }
        return 0;
    } catch (...) {
        return 1;
    }
}
