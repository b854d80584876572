// verify.cu -- the spectral-norm verifier as one persistent cooperative kernel.
//
// Reference: verify_spectral (core/src/shrink.cpp:75-102) runs `steps` power-method
// steps on diff_op(x) = (2/Delta)(A'^T A' x - B'^T B' x) (shrink.cpp:121-126) from a
// random unit vector (la_core.cpp:174-189), tracking log|y| and exiting early on
// annihilation (accept) or on growth past 1 (reject). Every step depends on the last,
// and each has a global norm, so a host loop would pay a launch + round trip per step.
// Here all steps run inside one cooperative grid: per step
//   phase 1: u = A' x (CSR, warp/row) and per-block partials of t = B' x
//   phase 2: t reduced (block b owns entries j = b mod nblocks)
//   phase 3: y = scale (A'^T u - B'^T t) (CSC gather + dense row), per-block |y|^2
//   phase 4: every block sums the |y|^2 partials in the same fixed order, so all
//            blocks take the same accept/reject/continue decision without a sync.
// x_{k+1} = y_k / |y_k| is never materialised: phase 1 reads y_k and scales it on the fly
// by 1/|y_k| (the reference divides; the two differ by at most one ulp per entry).
#include <cooperative_groups.h>

#include "common.cuh"
#include "verify.cuh"

namespace sfdg {

namespace {

constexpr int kVThreads = 512;
constexpr int kXStage = 4096;  // rows of B'^T staged in shared memory per chunk

struct GridBar {
    unsigned* count;
    unsigned* gen;
};

__device__ __forceinline__ void grid_sync(const GridBar& b, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = b.gen;
        const unsigned g = *vgen;
        __threadfence();
        if (atomicAdd(b.count, 1u) == nblocks - 1) {
            atomicExch(b.count, 0u);
            __threadfence();
            atomicAdd(b.gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
        sh[32] = s;
    }
    __syncthreads();
    s = sh[32];
    __syncthreads();
    return s;
}

// Sum of the nb per-block partials in a fixed order (lane-strided then a fixed shuffle
// tree): every block computes the identical value.
__device__ __forceinline__ double grid_total(const double* part, unsigned nb, double* sh) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < nb; b += 32) s += __ldcg(part + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) sh[32] = s;
    }
    __syncthreads();
    const double t = sh[32];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(kVThreads) verify_kernel(VerifyArgs a) {
    __shared__ double sh[33];
    __shared__ double tloc[512];
    __shared__ double xl[kXStage];
    const unsigned nb = gridDim.x;
    const GridBar bar{a.bar, a.bar + 1};
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gwarp = (int64_t)blockIdx.x * (kVThreads / 32) + wib;
    const int64_t nwarps = (int64_t)nb * (kVThreads / 32);
    const int L = a.ell;

    // phase 0: |x0|^2 for the unit-sphere normalisation (la_core.cpp:177-186)
    {
        double s = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)kVThreads + threadIdx.x; i < a.d; i += (int64_t)nb * kVThreads)
            s = fma(a.x0[i], a.x0[i], s);
        s = block_sum(s, sh);
        if (threadIdx.x == 0) a.part[blockIdx.x] = s;
    }
    grid_sync(bar, nb);
    const double nsq0 = grid_total(a.part, nb, sh);
    if (!(nsq0 > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            atomicOr(a.err, ERR_RNG_U1_ZERO);  // all-zero draw: would need a redraw
            a.out[0] = 0.0;
        }
        return;
    }
    const double inv0 = 1.0 / sqrt(nsq0);
    const double* xsrc = a.x0;
    double xscale = inv0;
    double log_mag = 0.0;
    int verdict = -1;  // -1 running, 0 reject, 1 accept
    int step = 0;
    for (; step < a.steps; ++step) {
        double* y = a.ybuf + (size_t)(step & 1) * a.d;
        // ---- phase 1: u = A' x ; t partials = B' x (B't is d x ell, row stride ldb)
        for (int64_t r = gwarp; r < a.m; r += nwarps) {
            double s = 0.0;
            for (int k = a.row_ptr[r] + lane; k < a.row_ptr[r + 1]; k += 32) {
                const int c = (int)a.col[k];
                s = fma(a.val[k], __ldcg(xsrc + c) * xscale, s);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) a.u[r] = s;
        }
        {
            // this block's rows of B'^T: stage x once in shared memory, then one column j
            // per thread (coalesced across j) accumulates over the rows in order
            const int64_t per = (a.d + nb - 1) / nb;
            const int64_t t0 = (int64_t)blockIdx.x * per;
            const int64_t t1 = min((int64_t)a.d, t0 + per);
            const int j = threadIdx.x;  // ell <= 256 < kVThreads: one column per thread
            double s = 0.0;
            for (int64_t c0 = t0; c0 < t1; c0 += kXStage) {
                const int64_t c1 = min(t1, c0 + kXStage);
                for (int64_t t = c0 + threadIdx.x; t < c1; t += kVThreads) xl[t - c0] = __ldcg(xsrc + t) * xscale;
                __syncthreads();
                if (j < L)
                    for (int64_t t = c0; t < c1; ++t) s = fma(a.bt[t * a.ldb + j], xl[t - c0], s);
                __syncthreads();
            }
            if (j < L) a.tpart[(size_t)blockIdx.x * L + j] = s;
        }
        grid_sync(bar, nb);
        // ---- phase 2: t[j] = sum_b tpart[b][j] in block order
        for (int j = (int)blockIdx.x * (kVThreads / 32) + wib; j < L; j += (int)nb * (kVThreads / 32)) {
            double s = 0.0;
            for (unsigned b = lane; b < nb; b += 32) s += __ldcg(a.tpart + (size_t)b * L + j);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) a.t[j] = s;
        }
        grid_sync(bar, nb);
        for (int j = threadIdx.x; j < L; j += kVThreads) tloc[j] = __ldcg(a.t + j);
        __syncthreads();
        // ---- phase 3: y = scale * (A'^T u - B'^T t), per-warp |y|^2 in fixed order
        double nsq = 0.0;
        bool bad = false;
        for (int64_t c = gwarp; c < a.d; c += nwarps) {
            double s = 0.0;
            for (int k = a.col_ptr[c] + lane; k < a.col_ptr[c + 1]; k += 32) s = fma(a.cval[k], __ldcg(a.u + a.row_idx[k]), s);
            double bsum = 0.0;
            for (int j = lane; j < L; j += 32) bsum = fma(a.bt[c * a.ldb + j], tloc[j], bsum);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                s += __shfl_xor_sync(0xffffffffu, s, o);
                bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
            }
            const double yc = a.scale * (s - bsum);  // shrink.cpp:124
            if (!isfinite(yc)) bad = true;
            if (lane == 0) y[c] = yc;
            nsq = fma(yc, yc, nsq);
        }
        if (bad) atomicOr(a.err, ERR_NONFINITE_VERIFY);
        if (lane != 0) nsq = 0.0;
        nsq = block_sum(nsq, sh);
        if (threadIdx.x == 0) a.part[blockIdx.x] = nsq;
        grid_sync(bar, nb);
        // ---- phase 4: identical decision in every block (shrink.cpp:88-99)
        const double tot = grid_total(a.part, nb, sh);
        if (*((volatile int*)a.err) & ERR_NONFINITE_VERIFY) {
            verdict = 0;
            break;
        }
        if (tot == 0.0) {
            verdict = 1;
            break;
        }
        const double nrm = sqrt(tot);
        log_mag += log(nrm);
        if (log_mag > 0.0 && nrm >= 1.0) {
            verdict = 0;
            ++step;
            break;
        }
        xsrc = y;
        xscale = 1.0 / nrm;
    }
    if (verdict < 0) verdict = log_mag <= 0.0 ? 1 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out[0] = (double)verdict;
        a.out[1] = log_mag;
        a.out[2] = (double)step;
    }
}

}  // namespace

int verify_grid_blocks(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, verify_kernel, kVThreads, 0));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // one block per SM, leaving two SMs for a concurrently running shrink (eigh) CTA so the
    // cooperative grid never waits for it to drain
    const int nb = std::max(1, std::min(per_sm, 1) * sms - 2);
    if (device >= 0 && device < 64) cached[device] = nb;
    return nb;
}

void verify_launch(const VerifyArgs& args, int nblocks, cudaStream_t st) {
    ProfScope prof("verify", st);
    CK(cudaMemsetAsync(args.bar, 0, 2 * sizeof(unsigned), st));
    void* params[] = {(void*)&args};
    CK(cudaLaunchCooperativeKernel((const void*)verify_kernel, dim3(nblocks), dim3(kVThreads), params, 0, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace sfdg
