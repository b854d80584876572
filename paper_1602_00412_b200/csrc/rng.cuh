// rng.cuh -- device reproduction of sfd::Rng's normal stream (see rng.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

namespace sfdg {

// Position in the draw stream of sfd::Rng (rng.hpp:12-31): raw engine words consumed
// and whether a Box-Muller spare is cached (its value lives on the device).
struct RngPos {
    uint64_t words = 0;
    bool has_spare = false;
};

// Advance a position by n normals (rng.cpp:19-34: a carried spare is used first, then
// pairs of raw words, the sin half of an odd tail becomes the new spare).
RngPos rng_advance(RngPos p, uint64_t n);

// The mt19937_64 word stream generated on the device into a ring, consumed by any number
// of streams at explicit positions (the flush pipeline draws for several flushes at once).
// A normal is a pure function of its pair of ring words, so a carried spare is recomputed
// from words (w-2, w-1) unless the caller supplied it explicitly (set_spare).
class RngStream {
  public:
    RngStream() = default;
    RngStream(const RngStream&) = delete;
    RngStream& operator=(const RngStream&) = delete;
    ~RngStream() { release(); }

    void init(uint64_t seed, uint64_t min_ring_words, int device);
    void restart(uint64_t seed);  // back to Rng(seed), keeping the allocations
    void release();

    // Draw n normals at `pos` into d_out (rows of `cols`, leading dimension ld), advancing pos.
    void normals(RngPos& pos, uint64_t n, uint64_t cols, uint64_t ld, double* d_out, int* d_err,
                 cudaStream_t stream);
    // Generate ahead (side stream) up to raw word w_end.
    void prefetch(uint64_t w_end);
    double spare_value(const RngPos& pos, cudaStream_t stream);
    void set_spare(const RngPos& pos, double v, cudaStream_t stream);
    uint64_t ring_words() const { return ring_cap; }

  private:
    void reseed();
    void generate_to(uint64_t words_end);
    void ensure(uint64_t w_begin, uint64_t w_end, cudaStream_t consumer);
    void mark_consumed(uint64_t w_begin, cudaStream_t consumer);

    int device = 0;
    uint64_t seed = 0;
    uint64_t gen_words = 0;  // tempered output words produced so far
    uint64_t ring_cap = 0;   // power of two
    uint64_t* d_ring = nullptr;
    uint64_t* d_window = nullptr;
    double* d_spare = nullptr;        // explicit spare (standalone entry points)
    double* d_tmp = nullptr;          // spare read-back
    uint64_t explicit_at = ~0ull;     // word position the explicit spare belongs to
    cudaStream_t s_gen = nullptr;
    cudaEvent_t ev_gen = nullptr;
    struct Consumer {
        uint64_t begin;
        cudaEvent_t ev;
    };
    std::vector<Consumer> live;       // readers not yet known to be done
    std::vector<cudaEvent_t> pool;    // recycled events
    std::recursive_mutex mu;          // lanes enqueue from their own host threads
};

}  // namespace sfdg
