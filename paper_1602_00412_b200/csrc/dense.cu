// dense.cu -- FP64 tall-skinny dense kernels on the DMMA tensor-core path.
//
// tcgen05 has no f64 kind on sm_100a, so FP64 contractions use the
// legacy mma.sync m8n8k4 f64 (SASS DMMA.884); on B200 it runs at the FP64 peak
// (36.9 TFLOP/s measured, profiles/r01_fp64_peak.txt -- same as DFMA) while cutting
// register/LSU traffic per flop 8x versus scalar DFMA.
//
//  * gram_tn: C = X^T X for a tall X (n x k, k <= 512). The reference forms these
//    Grams in orthonormalize (la_core.cpp:144-156, as MGS dot products), svd_top
//    (la_core.cpp:90-100) and dense_shrink's tall path (shrink.cpp:43-52). Split-K
//    over n into fixed chunks + fixed-order reduction: deterministic, no atomics.
//  * gemm_nn: C = X S for tall X and small S (k x c): the CholQR apply Y R^-1,
//    the right-vector recovery V = A^T U / sigma (la_core.cpp:113-126) fused with the
//    shrink row scale (shrink.cpp:15-26).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int TB = 64;   // output tile
constexpr int KT = 32;   // k-chunk staged in smem
constexpr int LDT = TB + 4;  // 68: conflict-free fragment reads (68 mod 16 == 4)
constexpr int LDK = KT + 4;  // 36

// cp.async (LDGSTS) with zero fill: `bytes` = 0 writes zeros, so tile edges need no branches.
template <int VEC>
__device__ __forceinline__ void cp_async(double* smem, const double* gmem, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if (VEC == 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 16 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Partial Gram of rows [r0, r1) for the upper tile (ti, tj): partial[chunk] (k x k).
// Two-stage cp.async pipeline: the next 32-row chunk streams in while DMMA consumes this one.
template <int VEC>
__global__ void __launch_bounds__(128) gram_tn_kernel(const double* __restrict__ X, int n, int k, int ldx,
                                                      int rows_per_chunk, int T, double* __restrict__ partial) {
    pdl_entry();
    extern __shared__ double smg[];  // [stage][A|B][KT][LDT]
    int ti = 0, rem = blockIdx.x;  // linear upper-triangle tile index -> (ti, tj)
    while (rem >= T - ti) {
        rem -= T - ti;
        ++ti;
    }
    const int tj = ti + rem;
    const int i0 = ti * TB, j0 = tj * TB;
    const int chunk = blockIdx.y;
    const int r0 = chunk * rows_per_chunk;
    const int r1 = min(n, r0 + rows_per_chunk);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = w & 1, wn = w >> 1;
    auto tile = [&](int stage, int ab) { return smg + (size_t)((stage * 2 + ab) * KT) * LDT; };
    auto load = [&](int stage, int kb) {
        double* As = tile(stage, 0);
        double* Bs = tile(stage, 1);
        for (int e = threadIdx.x; e < KT * (TB / VEC); e += 128) {
            const int r = e / (TB / VEC), c = (e % (TB / VEC)) * VEC;
            const int row = kb + r;
            const bool rok = row < r1;
            const bool oa = rok && i0 + c < k, ob = rok && j0 + c < k;
            cp_async<VEC>(As + r * LDT + c, oa ? X + (size_t)row * ldx + i0 + c : X, oa);
            cp_async<VEC>(Bs + r * LDT + c, ob ? X + (size_t)row * ldx + j0 + c : X, ob);
        }
        cp_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    int stage = 0;
    if (r0 < r1) load(0, r0);
    for (int kb = r0; kb < r1; kb += KT) {
        if (kb + KT < r1) {
            load(stage ^ 1, kb + KT);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* As = tile(stage, 0);
        const double* Bs = tile(stage, 1);
#pragma unroll
        for (int ks = 0; ks < KT; ks += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As[(ks + t) * LDT + wm * 32 + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(ks + t) * LDT + wn * 32 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
        stage ^= 1;
    }
    double* P = partial + (size_t)chunk * k * k;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            const int row = i0 + wm * 32 + mi * 8 + g;
            const int col = j0 + wn * 32 + ni * 8 + 2 * t;
            if (row < k) {
                if (col < k) P[(size_t)row * k + col] = acc[mi][ni][0];
                if (col + 1 < k) P[(size_t)row * k + col + 1] = acc[mi][ni][1];
            }
        }
}

// ---- TMA-staged Gram (opt-in, SFDG_GRAM=tma: measured slower than cp.async, see gram_tn) ------
// The same tiles, chunks and DMMA order as gram_tn_kernel (bit-identical partials), but each
// stage's 2 x KT row segments (<= 512 B each, contiguous in X) arrive by 1-D TMA bulk copies
// (cp.async.bulk, SASS UBLKCP) issued by one warp and counted in bytes on the stage's
// mbarrier, three stages deep: the other warps issue only LDS + DMMA, no per-element LDGSTS.
// Columns past k in an edge tile are zeroed once; rows past the chunk end in the last stage
// are zeroed by the consumers before they read.
constexpr int kGStages = 3;

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__global__ void __launch_bounds__(128) gram_tma_kernel(const double* __restrict__ X, int n, int k, int ldx,
                                                      int rows_per_chunk, int T, double* __restrict__ partial) {
    extern __shared__ __align__(128) double smg[];  // [stage][A|B][KT][LDT]
    __shared__ __align__(8) uint64_t full[kGStages];
    int ti = 0, rem = blockIdx.x;
    while (rem >= T - ti) {
        rem -= T - ti;
        ++ti;
    }
    const int tj = ti + rem;
    const int i0 = ti * TB, j0 = tj * TB;
    const int chunk = blockIdx.y;
    const int r0 = chunk * rows_per_chunk;
    const int r1 = min(n, r0 + rows_per_chunk);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = w & 1, wn = w >> 1;
    auto tile = [&](int stage, int ab) { return smg + (size_t)((stage * 2 + ab) * KT) * LDT; };
    const int ca = min(TB, k - i0), cb = min(TB, k - j0);  // valid columns of the A / B tiles
    // zero the columns no copy will write (edge tiles), then the barriers; all before PDL wait
    if (ca < TB || cb < TB)
        for (int e = threadIdx.x; e < kGStages * 2 * KT * TB; e += 128) {
            const int c = e % TB, r = (e / TB) % KT, ab = (e / (TB * KT)) % 2, stg = e / (2 * TB * KT);
            if (c >= (ab ? cb : ca)) tile(stg, ab)[r * LDT + c] = 0.0;
        }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kGStages; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zeros before any async write
    __syncthreads();
    pdl_entry();
    const int nst = (r1 - r0 + KT - 1) / KT;
    auto issue = [&](int s) {  // warp 0: stage s's row segments
        if (w != 0 || s >= nst) return;
        const int kb = r0 + s * KT, nr = min(KT, r1 - kb);
        const int stg = s % kGStages;
        if (lane == 0) mbar_expect_tx(&full[stg], (unsigned)(nr * (ca + cb) * 8));
        __syncwarp();
        if (lane < nr) {
            const double* row = X + (size_t)(kb + lane) * ldx;
            bulk_g2s(tile(stg, 0) + lane * LDT, row + i0, (unsigned)ca * 8u, &full[stg]);
            bulk_g2s(tile(stg, 1) + lane * LDT, row + j0, (unsigned)cb * 8u, &full[stg]);
        }
    };
    for (int s = 0; s < kGStages - 1; ++s) issue(s);
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int s = 0; s < nst; ++s) {
        issue(s + kGStages - 1);  // its buffer was released by the barrier that ended step s - 1
        const int stg = s % kGStages;
        mbar_wait(&full[stg], (unsigned)((s / kGStages) & 1));
        const int nr = min(KT, r1 - (r0 + s * KT));
        double* As = tile(stg, 0);
        double* Bs = tile(stg, 1);
        if (nr < KT) {  // last stage of the chunk: rows past its end count as zero
            for (int e = threadIdx.x; e < (KT - nr) * TB; e += 128) {
                const int r = nr + e / TB, c = e % TB;
                As[r * LDT + c] = 0.0;
                Bs[r * LDT + c] = 0.0;
            }
            __syncthreads();
        }
#pragma unroll
        for (int ks = 0; ks < KT; ks += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As[(ks + t) * LDT + wm * 32 + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(ks + t) * LDT + wn * 32 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();  // stage stg free for the copy issued at the top of step s + 1
    }
    double* P = partial + (size_t)chunk * k * k;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            const int row = i0 + wm * 32 + mi * 8 + g;
            const int col = j0 + wn * 32 + ni * 8 + 2 * t;
            if (row < k) {
                if (col < k) P[(size_t)row * k + col] = acc[mi][ni][0];
                if (col + 1 < k) P[(size_t)row * k + col + 1] = acc[mi][ni][1];
            }
        }
}

// Sum of the split-K partials (fixed order: warp w takes chunks w, w+8, ..., then the 8
// warp sums in warp order). A block owns 32 consecutive entries of the k x k output; only
// computed (upper) tiles are read -- coalesced -- and mirrored on write.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) gram_reduce_kernel(const double* __restrict__ partial, int nchunks,
                                                                     int k, double* __restrict__ out, int ldo) {
    pdl_entry();
    __shared__ double sh[kRedWarps][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int total = k * k;
    const int e = blockIdx.x * 32 + lane;
    const int i = e / k, j = e % k;
    const bool on = e < total && i / TB <= j / TB;
    double s = 0.0;
    if (on)
        for (int c = w; c < nchunks; c += kRedWarps) s += __ldcg(partial + (size_t)c * total + e);
    sh[w][lane] = s;
    __syncthreads();
    if (w == 0 && on) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kRedWarps; ++q) t += sh[q][lane];
        out[(size_t)i * ldo + j] = t;
        if (i / TB < j / TB) out[(size_t)j * ldo + i] = t;
    }
}

template <int VEC>
__global__ void __launch_bounds__(128) gemm_nn_kernel(const double* __restrict__ X, int n, int k, int ldx,
                                                      const double* __restrict__ S, int c, int lds,
                                                      double* __restrict__ C, int ldc,
                                                      const double* __restrict__ pred) {
    pdl_entry();
    if (pred && *pred == 0.0) return;
    extern __shared__ double smg[];  // [stage][Xs TB x LDK | Ss KT x LDT]
    constexpr int XS = TB * LDK, SS = KT * LDT;
    const int r0 = blockIdx.x * TB, c0 = blockIdx.y * TB;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = w & 1, wn = w >> 1;
    auto load = [&](int stage, int kk) {
        double* Xs = smg + stage * (XS + SS);
        double* Ss = Xs + XS;
        for (int e = threadIdx.x; e < TB * (KT / VEC); e += 128) {
            const int r = e / (KT / VEC), q = (e % (KT / VEC)) * VEC;
            const bool ok = r0 + r < n && kk + q < k;
            cp_async<VEC>(Xs + r * LDK + q, ok ? X + (size_t)(r0 + r) * ldx + kk + q : X, ok);
        }
        for (int e = threadIdx.x; e < KT * (TB / VEC); e += 128) {
            const int q = e / (TB / VEC), cc = (e % (TB / VEC)) * VEC;
            const bool ok = kk + q < k && c0 + cc < c;
            cp_async<VEC>(Ss + q * LDT + cc, ok ? S + (size_t)(kk + q) * lds + c0 + cc : S, ok);
        }
        cp_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    int stage = 0;
    load(0, 0);
    for (int kk = 0; kk < k; kk += KT) {
        if (kk + KT < k) {
            load(stage ^ 1, kk + KT);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* Xs = smg + stage * (XS + SS);
        const double* Ss = Xs + XS;
#pragma unroll
        for (int ks = 0; ks < KT; ks += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = Xs[(wm * 32 + mi * 8 + g) * LDK + ks + t];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Ss[(ks + t) * LDT + wn * 32 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
        stage ^= 1;
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            const int row = r0 + wm * 32 + mi * 8 + g;
            const int col = c0 + wn * 32 + ni * 8 + 2 * t;
            if (row < n) {
                if (col < c) C[(size_t)row * ldc + col] = acc[mi][ni][0];
                if (col + 1 < c) C[(size_t)row * ldc + col + 1] = acc[mi][ni][1];
            }
        }
}

constexpr int kRedBlocks = 2 * kSMs;

// Deterministic sum of squares: fixed grid, fixed per-thread stride order, fixed trees.
__global__ void sumsq_partial_kernel(const double* __restrict__ X, int64_t rows, int cols, int ld,
                                     double* __restrict__ partial, int* __restrict__ err, int err_bit) {
    pdl_entry();
    __shared__ double sh[32];
    double s = 0.0;
    bool bad = false;
    const int64_t total = rows * (int64_t)cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const double v = X[(e / cols) * ld + e % cols];
        if (!isfinite(v)) bad = true;
        s = fma(v, v, s);
    }
    if (bad && err) atomicOr(err, err_bit);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int n, double* __restrict__ out) {
    pdl_entry();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += partial[i];
        *out = s;
    }
}

__global__ void transpose_kernel(const double* __restrict__ in, int rows, int cols, int ldi, double* __restrict__ out,
                                 int ldo) {
    pdl_entry();
    __shared__ double tile[32][33];
    // 32 x 32 tiles in a flat block-stride loop: any rows x cols (a d-row panel has d / 32 tile
    // rows, past the 65535 limit of a grid's y dimension at d > 2.1e6)
    const int64_t tc = (cols + 31) / 32, ntile = tc * (((int64_t)rows + 31) / 32);
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
        const int bx = (int)(t % tc) * 32, by = (int)(t / tc) * 32;
        for (int j = threadIdx.y; j < 32; j += blockDim.y) {
            const int r = by + j, c = bx + threadIdx.x;
            if (r < rows && c < cols) tile[j][threadIdx.x] = in[(size_t)r * ldi + c];
        }
        __syncthreads();
        for (int j = threadIdx.y; j < 32; j += blockDim.y) {
            const int r = bx + j, c = by + threadIdx.x;  // out row = in col
            if (r < cols && c < rows) out[(size_t)r * ldo + c] = tile[threadIdx.x][j];
        }
        __syncthreads();
    }
}

__global__ void copy2d_kernel(const double* __restrict__ in, int rows, int cols, int ldi, double* __restrict__ out,
                              int ldo) {
    pdl_entry();
    const int64_t total = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[(e / cols) * ldo + e % cols] = in[(e / cols) * ldi + e % cols];
}

__global__ void fill2d_kernel(double* __restrict__ out, int rows, int cols, int ldo, double v) {
    pdl_entry();
    const int64_t total = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[(e / cols) * ldo + e % cols] = v;
}

}  // namespace

static bool vec16(const double* p, int ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); }

void gram_tn(const double* X, int n, int k, int ldx, double* out, int ldo, Scratch& scr, cudaStream_t st) {
    if (k <= 0) return;
    if (n <= 0) {
        fill2d(out, k, k, ldo, 0.0, st);
        return;
    }
    ProfScope prof("gram", st);
    // algorithmic: the k(k+1)/2 distinct dot products of length n, X read once
    prof.work((double)n * k * (k + 1), 8.0 * ((double)n * k + (double)k * k));
    const int T = (k + TB - 1) / TB;
    const int ntiles = T * (T + 1) / 2;
    // split-K chunks: two waves of tile-chunks, and up to six for tall X (>= 8192 rows per chunk
    // at two waves) -- kbench, 1 B200: 1e6 x 256 4.13 ms at two waves, 3.03 ms at six; 5e4 x 128
    // 46.9 us at two, 50-56 us at more (profiles/r02c_gram_ab.txt). SFDG_GRAM_WAVES overrides.
    static const int waves_env = std::getenv("SFDG_GRAM_WAVES") ? std::max(1, std::atoi(std::getenv("SFDG_GRAM_WAVES"))) : 0;
    const int64_t lo = (2 * (int64_t)kSMs + ntiles - 1) / ntiles, hi = (6 * (int64_t)kSMs + ntiles - 1) / ntiles;
    int target_chunks = waves_env ? std::max(1, (waves_env * kSMs + ntiles - 1) / ntiles)
                                  : (int)std::max<int64_t>(1, std::max(lo, std::min(hi, (int64_t)n / 8192)));
    int rows_per_chunk = (int)round_up(std::max<int64_t>(KT * 4, ((int64_t)n + target_chunks - 1) / target_chunks), KT);
    const int nchunks = (n + rows_per_chunk - 1) / rows_per_chunk;
    double* partial = scr.take<double>((int64_t)nchunks * k * k);
    const size_t smem = 2 * 2 * KT * LDT * sizeof(double);
    if (first_on_device((const void*)(gram_tn_kernel<2>))) {
        allow_max_dynamic_smem(gram_tn_kernel<2>);
        allow_max_dynamic_smem(gram_tn_kernel<1>);
    }
    // SFDG_GRAM=tma: stages by TMA bulk copies (bit-identical; measured slower: three 35 KB
    // stages leave two CTAs per SM and 64 512-byte copies per stage, 7.2 against 4.1 ms at
    // 1e6 x 256, profiles/r02c_gram_ab.txt), so per-thread cp.async stays the default
    const char* gsel = std::getenv("SFDG_GRAM");
    const bool tma = gsel && std::string(gsel) == "tma";
    if (tma && vec16(X, ldx) && k % 2 == 0) {
        if (first_on_device((const void*)gram_tma_kernel)) allow_max_dynamic_smem(gram_tma_kernel);
        const size_t tsmem = (size_t)kGStages * 2 * KT * LDT * sizeof(double);
        LAUNCH(gram_tma_kernel, dim3(ntiles, nchunks), 128, tsmem, st, X, n, k, ldx, rows_per_chunk, T, partial);
    } else if (vec16(X, ldx) && k % 2 == 0)
        LAUNCH(gram_tn_kernel<2>, dim3(ntiles, nchunks), 128, smem, st, X, n, k, ldx, rows_per_chunk, T, partial);
    else
        LAUNCH(gram_tn_kernel<1>, dim3(ntiles, nchunks), 128, smem, st, X, n, k, ldx, rows_per_chunk, T, partial);
    LAUNCH(gram_reduce_kernel, ceil_div((size_t)k * k, 32), 32 * kRedWarps, 0, st, partial, nchunks, k, out, ldo);
}

void gemm_nn(const double* X, int n, int k, int ldx, const double* S, int c, int lds, double* C, int ldc,
             cudaStream_t st, const double* pred) {
    if (n <= 0 || c <= 0) return;
    if (k <= 0) {
        fill2d(C, n, c, ldc, 0.0, st);
        return;
    }
    ProfScope prof("gemm", st);
    prof.work(2.0 * n * (double)k * c, 8.0 * ((double)n * k + (double)k * c + (double)n * c));
    const size_t smem = 2 * (TB * LDK + KT * LDT) * sizeof(double);
    if (first_on_device((const void*)(gemm_nn_kernel<2>))) {
        allow_max_dynamic_smem(gemm_nn_kernel<2>);
        allow_max_dynamic_smem(gemm_nn_kernel<1>);
    }
    if (vec16(X, ldx) && vec16(S, lds) && k % 2 == 0 && c % 2 == 0)
        LAUNCH(gemm_nn_kernel<2>, dim3(ceil_div(n, TB), ceil_div(c, TB)), 128, smem, st, X, n, k, ldx, S, c, lds, C,
               ldc, pred);
    else
        LAUNCH(gemm_nn_kernel<1>, dim3(ceil_div(n, TB), ceil_div(c, TB)), 128, smem, st, X, n, k, ldx, S, c, lds, C,
               ldc, pred);
}

void sumsq(const double* X, int64_t rows, int cols, int ld, double* d_out, int* d_err, int err_bit, Scratch& scr,
           cudaStream_t st) {
    ProfScope prof("reduce", st);
    double* partial = scr.take<double>(kRedBlocks);
    LAUNCH(sumsq_partial_kernel, kRedBlocks, 256, 0, st, X, rows, cols, ld, partial, d_err, err_bit);
    LAUNCH(sum_partials_kernel, 1, 32, 0, st, partial, kRedBlocks, d_out);
}

namespace {
__global__ void scale_vector_kernel(double* __restrict__ x, int64_t n, double s) {
    pdl_entry();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= s;
}
}  // namespace

void scale_vector(double* x, int64_t n, double s, cudaStream_t st) {
    if (n <= 0) return;
    LAUNCH(scale_vector_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)n, 256))), 256, 0, st, x, n, s);
}

void transpose(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return;
    const size_t ntile = (size_t)ceil_div((size_t)cols, 32) * (size_t)ceil_div((size_t)rows, 32);
    LAUNCH(transpose_kernel, (unsigned)std::min<size_t>(ntile, 16 * kSMs * 8), dim3(32, 8), 0, st, in, rows, cols, ldi,
           out, ldo);
}

void copy2d(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return;
    LAUNCH(copy2d_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)rows * cols, 256))), 256, 0, st, in, rows,
           cols, ldi, out, ldo);
}

void fill2d(double* out, int rows, int cols, int ldo, double v, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return;
    LAUNCH(fill2d_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)rows * cols, 256))), 256, 0, st, out, rows,
           cols, ldo, v);
}

}  // namespace sfdg
