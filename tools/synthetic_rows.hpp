// synthetic_rows.hpp -- the reference's synthetic row stream on the host (shared by the
// `sfdg generate|bench` CLI and the reference-suite compat layer, tests/refsuite).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <utility>
#include <vector>

namespace sfdg_tools {

// The synthetic row stream of SyntheticSpec / SyntheticStream (bench.hpp:9-36,
// bench.cpp:13-66): every row has exactly z distinct columns with +-1 values; the first
// min(ceil(1.5 z), d) columns form the "head", drawn with probability p_head per slot. The
// draws are sfd::Rng's fixed formulas over std::mt19937_64 (rng.hpp:12-31): uniform() =
// (w >> 11) 2^-53, uniform_below(n) by rejection above the largest multiple of n
// (rng.cpp:9-17). Per slot: one uniform() picks the group (a full group redirects to the
// other), uniform_below redraws until an unused column of that group comes up, one uniform()
// picks the sign; the row is emitted sorted by column. Same seed -> the same rows as the
// reference, bit for bit.
class SyntheticRows {
  public:
    SyntheticRows(size_t n, size_t d, size_t z, double p_head, uint64_t seed)
        : n_(n), d_(d), z_(z), p_head_(p_head), eng_(seed) {
        if (d == 0 || z == 0 || z > d) throw std::invalid_argument("SyntheticSpec: requires 1 <= z <= d");
        if (!(p_head >= 0.0 && p_head <= 1.0)) throw std::invalid_argument("SyntheticSpec: p_head out of range");
        head_ = std::min((size_t)std::ceil(1.5 * (double)z), d);
        tail_ = d - head_;
        stamp_.assign(d, 0);
    }
    bool more() const { return made_ < n_; }
    // Appends the next row's sorted (col, value) pairs to `out`.
    void next(std::vector<std::pair<uint32_t, double>>& out) {
        ++made_;
        out.clear();
        size_t in_head = 0, in_tail = 0;
        while (out.size() < z_) {
            bool head = uniform() < p_head_;
            if (tail_ == 0 || in_tail == tail_) head = true;
            if (in_head == head_) head = false;
            uint64_t c;
            do c = head ? below(head_) : head_ + below(tail_);
            while (stamp_[c] == made_);
            stamp_[c] = made_;
            ++(head ? in_head : in_tail);
            out.emplace_back((uint32_t)c, uniform() < 0.5 ? 1.0 : -1.0);
        }
        std::sort(out.begin(), out.end(),
                  [](const std::pair<uint32_t, double>& a, const std::pair<uint32_t, double>& b) {
                      return a.first < b.first;
                  });
    }

  private:
    double uniform() { return (double)(eng_() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t m) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % m;
        uint64_t w;
        do w = eng_();
        while (w >= limit);
        return w % m;
    }
    size_t n_, d_, z_, head_ = 0, tail_ = 0, made_ = 0;
    double p_head_;
    std::mt19937_64 eng_;
    std::vector<size_t> stamp_;  // stamp_[c] == row number: column c used in this row
};

}  // namespace sfdg_tools
