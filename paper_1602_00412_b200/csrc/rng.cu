// rng.cu -- the reference's Gaussian draw stream, generated on the device.
//
// Reference: sfd::Rng (core/include/sfd/rng.hpp:12-31, core/src/rng.cpp:19-34) draws
// normals from std::mt19937_64 with a fixed Box-Muller formula (cos first, sin cached
// as the spare). gaussian_matrix (la_core.cpp:167-172) and unit_sphere_vector
// (la_core.cpp:174-189) consume that stream in row-major order. The host generator
// costs 42 ns per normal, 16-56x the GPU flush at c2-c5, so the exact
// integer stream is reproduced here:
//
//  * mt_generate_kernel: one CTA of 156 threads advances the mt19937_64 linear
//    recurrence x[k+312] = x[k+156] ^ twist(x[k], x[k+1]) 156 words per barrier step
//    (all 156 words of a step depend only on the previous 312), tempers them and
//    streams them into an HBM ring buffer. It runs on a side stream, ahead of use.
//  * box_muller_kernel: one thread per Box-Muller pair turns ring words into the
//    normals of a d x ell panel (or a d-vector), honouring the carried spare.
//
// The integer stream is bit-exact; log/sincos are CUDA's FP64 versions (<= 1-2 ulp
// from glibc's), which the parity gate absorbs (1e-15 vs 1e-8 budget).
#include "common.cuh"
#include "rng.cuh"

namespace sfdg {

namespace {

constexpr int MT_N = 312;
constexpr int MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t MT_LM = 0x7FFFFFFFULL;

__device__ __forceinline__ uint64_t temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

// window: the 312 most recent untempered words x[G..G+311]; produces output words
// G .. G + 156*steps - 1 (output word j = temper(x[312 + j])) into ring[j & mask].
__global__ void __launch_bounds__(MT_M) mt_generate_kernel(uint64_t* __restrict__ window, uint64_t* __restrict__ ring,
                                                           uint64_t ring_mask, uint64_t first_word, int steps) {
    pdl_entry();
    __shared__ uint64_t r[2 * MT_N];  // slot = local index mod 624
    const int t = threadIdx.x;
    r[t] = window[t];
    r[t + MT_M] = window[t + MT_M];
    __syncthreads();
    for (int s = 0; s < steps; ++s) {
        const int l = MT_N + MT_M * s + t;  // local index of the word this thread makes
        const uint64_t xk = r[(l - MT_N) % (2 * MT_N)];
        const uint64_t xk1 = r[(l - MT_N + 1) % (2 * MT_N)];
        const uint64_t xm = r[(l - MT_M) % (2 * MT_N)];
        const uint64_t y = (xk & MT_UM) | (xk1 & MT_LM);
        const uint64_t x = xm ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
        r[l % (2 * MT_N)] = x;
        ring[(first_word + (uint64_t)(l - MT_N)) & ring_mask] = temper(x);
        __syncthreads();
    }
    const int base = MT_M * steps;  // new window = local [base, base + 312)
    window[t] = r[(base + t) % (2 * MT_N)];
    window[t + MT_M] = r[(base + t + MT_M) % (2 * MT_N)];
}

__device__ __forceinline__ void box_muller_pair(uint64_t e1, uint64_t e2, double& c, double& sn, int* err) {
    const double u1 = (double)(e1 >> 11) * 0x1.0p-53;  // rng.hpp:19
    const double u2 = (double)(e2 >> 11) * 0x1.0p-53;
    if (u1 <= 0.0) atomicOr(err, ERR_RNG_U1_ZERO);  // rng.cpp:27-29 redraw: p = 2^-53
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;  // (2.0 * pi) * u2
    double s, cs;
    sincos(theta, &s, &cs);
    c = rad * cs;
    sn = rad * s;
}

// Normals j = 0 .. n-1 of the stream at raw word w0 with an optional carried spare (j == 0
// when has_spare): from *spare_in when given, else the sin half of ring words (w0-2, w0-1).
// Output element j goes to out[(j / cols) * ld + j % cols].
__global__ void box_muller_kernel(const uint64_t* __restrict__ ring, uint64_t ring_mask, uint64_t w0,
                                  int has_spare, const double* __restrict__ spare_in, uint64_t n, uint64_t cols,
                                  uint64_t ld, double* __restrict__ out, int* __restrict__ err) {
    pdl_entry();
    const uint64_t s = has_spare ? 1 : 0;
    const uint64_t rest = n > s ? n - s : 0;
    const uint64_t pairs = (rest + 1) / 2;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (tid == 0 && s && n > 0) {
        if (spare_in) {
            out[0] = *spare_in;
        } else {
            double c, sn;
            box_muller_pair(ring[(w0 - 2) & ring_mask], ring[(w0 - 1) & ring_mask], c, sn, err);
            out[0] = sn;
        }
    }
    for (uint64_t p = tid; p < pairs; p += stride) {
        double c, sn;
        box_muller_pair(ring[(w0 + 2 * p) & ring_mask], ring[(w0 + 2 * p + 1) & ring_mask], c, sn, err);
        const uint64_t j0 = s + 2 * p;
        out[(j0 / cols) * ld + j0 % cols] = c;
        const uint64_t j1 = j0 + 1;
        if (j1 < n) out[(j1 / cols) * ld + j1 % cols] = sn;
    }
}

__global__ void spare_kernel(const uint64_t* __restrict__ ring, uint64_t ring_mask, uint64_t w, double* __restrict__ out,
                             int* __restrict__ err) {
    pdl_entry();
    double c, sn;
    box_muller_pair(ring[(w - 2) & ring_mask], ring[(w - 1) & ring_mask], c, sn, err);
    *out = sn;
}

__global__ void zero_pad_kernel(double* __restrict__ out, uint64_t rows, uint64_t cols, uint64_t ld) {
    pdl_entry();
    const uint64_t padw = ld - cols;
    const uint64_t total = rows * padw;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        out[(i / padw) * ld + cols + i % padw] = 0.0;
}

}  // namespace

RngPos rng_advance(RngPos p, uint64_t n) {
    if (n == 0) return p;
    const uint64_t s = p.has_spare ? 1 : 0;
    const uint64_t rest = n > s ? n - s : 0;
    p.words += 2 * ((rest + 1) / 2);
    p.has_spare = rest > 0 && (rest % 2) == 1;
    return p;
}

void RngStream::init(uint64_t seed_, uint64_t min_ring_words, int device_) {
    release();
    device = device_;
    seed = seed_;
    uint64_t cap = 1 << 16;
    while (cap < min_ring_words) cap <<= 1;
    ring_cap = cap;
    CK(cudaMalloc(&d_ring, ring_cap * sizeof(uint64_t)));
    CK(cudaMalloc(&d_window, MT_N * sizeof(uint64_t)));
    CK(cudaMalloc(&d_spare, 2 * sizeof(double)));
    CK(cudaMemset(d_spare, 0, 2 * sizeof(double)));
    d_tmp = d_spare + 1;
    CK(cudaStreamCreateWithFlags(&s_gen, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_gen, cudaEventDisableTiming));
    reseed();
}

void RngStream::reseed() {
    // std::mt19937_64(seed) initial state ([rand.eng.mers], f = 6364136223846793005).
    uint64_t mt[MT_N];
    mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    // every queued reader of the old stream must be done before the ring is rewritten
    for (auto& c : live) {
        CK(cudaEventSynchronize(c.ev));
        pool.push_back(c.ev);
    }
    live.clear();
    CK(cudaStreamSynchronize(s_gen));
    CK(cudaMemcpy(d_window, mt, sizeof mt, cudaMemcpyHostToDevice));
    gen_words = 0;
}

void RngStream::restart(uint64_t seed_) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    seed = seed_;
    explicit_at = ~0ull;
    reseed();
}

void RngStream::release() {
    for (auto& c : live) cudaEventDestroy(c.ev);
    for (auto e : pool) cudaEventDestroy(e);
    live.clear();
    pool.clear();
    if (d_ring) cudaFree(d_ring);
    if (d_window) cudaFree(d_window);
    if (d_spare) cudaFree(d_spare);
    if (s_gen) cudaStreamDestroy(s_gen);
    if (ev_gen) cudaEventDestroy(ev_gen);
    d_ring = nullptr;
    d_window = nullptr;
    d_spare = nullptr;
    d_tmp = nullptr;
    s_gen = nullptr;
    ev_gen = nullptr;
}

void RngStream::generate_to(uint64_t words_end) {
    if (words_end <= gen_words) return;
    const uint64_t need = words_end - gen_words;
    const int steps = (int)((need + MT_M - 1) / MT_M);
    const uint64_t new_end = gen_words + (uint64_t)steps * MT_M;
    // Never overwrite words a queued reader may still need: writing word p replaces p - ring_cap.
    if (new_end > ring_cap) {
        const uint64_t limit = new_end - ring_cap;
        size_t keep = 0;
        for (auto& c : live) {
            if (c.begin < limit) {
                CK(cudaStreamWaitEvent(s_gen, c.ev, 0));
                pool.push_back(c.ev);
            } else {
                live[keep++] = c;
            }
        }
        live.resize(keep);
    }
    ProfScope prof("rng_gen", s_gen);
    LAUNCH(mt_generate_kernel, 1, MT_M, 0, s_gen, d_window, d_ring, ring_cap - 1, gen_words, steps);
    gen_words = new_end;
    CK(cudaEventRecord(ev_gen, s_gen));
}

void RngStream::ensure(uint64_t w_begin, uint64_t w_end, cudaStream_t consumer) {
    if (w_end - w_begin > ring_cap) throw invalid_argument("rng: request exceeds the device ring");
    if (w_begin + ring_cap < gen_words) reseed();  // fell out of the ring (standalone calls): regenerate
    generate_to(w_end);
    CK(cudaStreamWaitEvent(consumer, ev_gen, 0));
}

void RngStream::prefetch(uint64_t w_end) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    uint64_t cap_end = w_end;
    if (cap_end > gen_words + ring_cap / 2) cap_end = gen_words + ring_cap / 2;
    generate_to(cap_end);
}

void RngStream::mark_consumed(uint64_t w_begin, cudaStream_t consumer) {
    cudaEvent_t ev;
    if (!pool.empty()) {
        ev = pool.back();
        pool.pop_back();
    } else {
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ev, consumer));
    live.push_back({w_begin, ev});
}

// Draws n normals (rng.cpp:19-34 semantics) into out (rows of `cols` values, leading
// dimension ld, zero padding beyond cols), advancing pos.
void RngStream::normals(RngPos& pos, uint64_t n, uint64_t cols, uint64_t ld, double* d_out, int* d_err,
                        cudaStream_t stream) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    if (n == 0) return;
    const RngPos next = rng_advance(pos, n);
    const bool from_ring = pos.has_spare && explicit_at != pos.words;
    const uint64_t w_begin = from_ring ? pos.words - 2 : pos.words;
    ensure(w_begin, std::max(next.words, pos.words), stream);
    ProfScope prof("box_muller", stream);
    const uint64_t s = pos.has_spare ? 1 : 0;
    const uint64_t pairs = ((n > s ? n - s : 0) + 1) / 2;
    const unsigned blocks = (unsigned)std::min<uint64_t>(4 * kSMs, (pairs + 255) / 256 + 1);
    LAUNCH(box_muller_kernel, blocks, 256, 0, stream, d_ring, ring_cap - 1, pos.words, (int)pos.has_spare,
           from_ring ? (const double*)nullptr : (const double*)d_spare, n, cols, ld, d_out, d_err);
    if (ld > cols) {
        const uint64_t rows = (n + cols - 1) / cols;
        LAUNCH(zero_pad_kernel, (unsigned)std::min<uint64_t>(4 * kSMs, (rows * (ld - cols) + 255) / 256), 256, 0,
               stream, d_out, rows, cols, ld);
    }
    mark_consumed(w_begin, stream);
    pos = next;
}

double RngStream::spare_value(const RngPos& pos, cudaStream_t stream) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    if (!pos.has_spare) return 0.0;
    double v = 0.0;
    if (explicit_at == pos.words) {
        CK(cudaMemcpyAsync(&v, d_spare, sizeof v, cudaMemcpyDeviceToHost, stream));
    } else {
        ensure(pos.words - 2, pos.words, stream);
        int* err = nullptr;
        CK(cudaMallocAsync(&err, sizeof(int), stream));
        LAUNCH(spare_kernel, 1, 1, 0, stream, d_ring, ring_cap - 1, pos.words, d_tmp, err);
        mark_consumed(pos.words - 2, stream);
        CK(cudaMemcpyAsync(&v, d_tmp, sizeof v, cudaMemcpyDeviceToHost, stream));
        CK(cudaFreeAsync(err, stream));
    }
    CK(cudaStreamSynchronize(stream));
    return v;
}

void RngStream::set_spare(const RngPos& pos, double v, cudaStream_t stream) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    CK(cudaMemcpyAsync(d_spare, &v, sizeof v, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
    explicit_at = pos.words;
}

}  // namespace sfdg
