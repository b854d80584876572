// probe_bar.cu -- latency of software grid barriers (the verifier's step barrier) on B200.
// 32 blocks x 512 threads (the c2 verifier grid), 2000 barriers per launch, best of 5.
//   gen      : the verifier's generation barrier (atomicAdd count, last arriver bumps gen,
//              others spin on ld.acquire with __nanosleep(32))
//   gen_spin : same without the nanosleep
//   flags    : each block writes its own arrival flag (epoch), block 0's warp 0 polls all flags
//              then releases one epoch word everyone polls
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void bar_kernel(unsigned* count, unsigned* gen, unsigned* flags, int iters, double* sink) {
    double acc = threadIdx.x;
    const unsigned nb = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        acc = acc * 1.0000001 + 1.0;
        __syncthreads();
        if (MODE < 2) {
            if (threadIdx.x == 0) {
                const unsigned g = ld_acquire(gen);
                __threadfence();
                if (atomicAdd(count, 1u) == nb - 1) {
                    atomicExch(count, 0u);
                    __threadfence();
                    atomicAdd(gen, 1u);
                } else {
                    if (MODE == 0)
                        while (ld_acquire(gen) == g) __nanosleep(32);
                    else
                        while (ld_acquire(gen) == g) {
                        }
                }
            }
        } else {
            const unsigned epoch = it + 1;
            if (threadIdx.x == 0) st_release(flags + 32 * blockIdx.x, epoch);
            if (blockIdx.x == 0 && threadIdx.x < 32) {
                for (unsigned b = threadIdx.x; b < nb; b += 32)
                    while (ld_acquire(flags + 32 * b) < epoch) {
                    }
                __syncwarp();
                if (threadIdx.x == 0) st_release(gen, epoch);
            }
            if (threadIdx.x == 0)
                while (ld_acquire(gen) < epoch) {
                }
        }
        __syncthreads();
    }
    if (acc == -1.0) sink[0] = acc;
}

int main() {
    unsigned *count, *gen, *flags;
    double* sink;
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaMalloc(&flags, 4 * 32 * 256);
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    const char* names[] = {"gen (nanosleep 32)", "gen (spin)", "flags"};
    for (int nb : {16, 32, 64, 148}) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(count, 0, 4);
                cudaMemset(gen, 0, 4);
                cudaMemset(flags, 0, 4 * 32 * 256);
                void* args[] = {&count, &gen, &flags, (void*)&iters, &sink};
                const void* fn = mode == 0 ? (const void*)bar_kernel<0> : mode == 1 ? (const void*)bar_kernel<1>
                                                                                   : (const void*)bar_kernel<2>;
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(512), args, 0, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            std::printf("blocks %3d %-20s %.3f us per barrier\n", nb, names[mode], best * 1e3 / iters);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
