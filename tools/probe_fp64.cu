// FP64 peak probe for B200 (sm_100a): DFMA (CUDA cores) vs DMMA (mma.sync m8n8k4 f64).
// Prints achieved TFLOP/s for each; used to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sms=%d l2=%d MB smem/block optin=%zu KB clock=%d kHz\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin >> 10, p.clockRate);
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / threads);
    int iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA  threads=%4d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", threads, blocks, flops / ms / 1e9, ms);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = p.multiProcessorCount * (1024 / threads);
    int iters = 4096;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA  threads=%4d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", threads, blocks, flops / ms / 1e9, ms);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
