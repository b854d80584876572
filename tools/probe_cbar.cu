// probe_cbar.cu -- latency of barrier.cluster (arrive.release + wait.acquire) vs __syncthreads
// for 512-thread CTAs in clusters of 1, 2, 4, 8; 10000 barriers per launch.
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ void cbar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE>
__global__ void k(int iters, double* sink) {
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        acc = acc * 1.0000001 + 1.0;
        if (MODE == 0) __syncthreads();
        else cbar();
    }
    if (acc == -1.0) sink[0] = acc;
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 10000;
    for (int C : {1, 2, 4, 8}) {
        for (int mode = 0; mode < 2; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(C);
                cfg.blockDim = dim3(512);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = C;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaEventRecord(a);
                if (mode == 0) cudaLaunchKernelEx(&cfg, k<0>, iters, sink);
                else cudaLaunchKernelEx(&cfg, k<1>, iters, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            std::printf("cluster %d %-16s %.1f ns per barrier\n", C, mode ? "barrier.cluster" : "__syncthreads",
                        best * 1e6 / iters);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
