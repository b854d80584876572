// compat/sfd/rng.hpp -- sfd::Rng for the reference suite run against the device build.
//
// Same draws as the reference (rng.hpp:12-31, rng.cpp:9-34: std::mt19937_64, uniform() =
// (w >> 11) 2^-53, rejection uniform_below, Box-Muller with the sin half cached), plus the
// position bookkeeping the device ABI needs: device_state() / set_device_state() exchange
// sfdg_rng_state {seed, words drawn, spare} with the sfdg_* entry points that consume draws.
#pragma once

#include <cstdint>
#include <random>

#include "sfdg.h"

namespace sfd {

class Rng {
  public:
    explicit Rng(std::uint64_t seed) : seed_(seed), engine_(seed) {}

    std::uint64_t next_u64() {
        ++words_;
        return engine_();
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    std::uint64_t uniform_below(std::uint64_t n);
    double normal();

    sfdg_rng_state device_state() const { return {seed_, words_, has_spare_ ? 1 : 0, spare_}; }
    // Adopt the state a device call advanced this stream to (same seed, words >= ours).
    void set_device_state(const sfdg_rng_state& s);

  private:
    std::uint64_t seed_;
    std::uint64_t words_ = 0;
    std::mt19937_64 engine_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

}  // namespace sfd
