// probe_lat.cu -- dependent-chain latencies of the FP64 operations the latency-bound
// eigensolver kernels are built from (one warp, clock64 around 1024 dependent ops).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

template <int OP>
__global__ void lat(double* out, long long* cyc, double seed) {
    __shared__ double sh[64];
    sh[threadIdx.x] = seed + threadIdx.x;
    __syncwarp();
    double x = seed + threadIdx.x * 1e-3;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) {
        if (OP == 0) x = fma(x, 0.999999, 1e-7);
        if (OP == 1) x = x / (x + 1.5);
        if (OP == 2) x = fast_rcp(x + 1.5);
        if (OP == 3) x = sqrt(x + 1.0);
        if (OP == 4) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-9;
        if (OP == 5) x = sh[((int)x) & 31] + 1.0;
        if (OP == 6) x = x * 0.999 + 1e-7;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&cyc, 8);
    const char* names[] = {"dfma", "ddiv (IEEE)", "fast_rcp", "dsqrt", "shfl+dfma", "lds (dep)", "dmul+dadd"};
    for (int op = 0; op < 7; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: lat<0><<<1, 32>>>(out, cyc, 1.0); break;
                case 1: lat<1><<<1, 32>>>(out, cyc, 1.0); break;
                case 2: lat<2><<<1, 32>>>(out, cyc, 1.0); break;
                case 3: lat<3><<<1, 32>>>(out, cyc, 1.0); break;
                case 4: lat<4><<<1, 32>>>(out, cyc, 1.0); break;
                case 5: lat<5><<<1, 32>>>(out, cyc, 1.0); break;
                case 6: lat<6><<<1, 32>>>(out, cyc, 1.0); break;
            }
        }
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-14s %6.1f cycles/op\n", names[op], c / 1024.0);
    }
    printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
