// probe_l2.cu -- measured L2 bandwidth for the c2 SpMM access pattern (roofline denominator
// for L2-resident gathers; MEASURED_PEAKS.json only carries the HBM copy bandwidth).
//
//   gather : 1e5 random row gathers of `row` doubles (832 B at c2's lp = 104) from an 8 MB
//            table (Y or W of one c2 flush), one warp per 10 gathers like spmm_rows_kernel,
//            best of 50 launches timed with CUDA events, table warm in L2
//   stream : the same bytes read as contiguous rows (sequential 8 MB sweeps)
// Prints GB/s for both (bytes = gathers x row bytes).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            std::exit(1);                                                      \
        }                                                                      \
    } while (0)

__global__ void __launch_bounds__(256, 5) gather(const int* __restrict__ idx, int per_warp, int ngroups,
                                                 const double* __restrict__ tab, int ld, int ncols,
                                                 double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= ngroups) return;
    double2 acc0 = make_double2(0, 0), acc1 = make_double2(0, 0);
    // all row indices first, then every gather of the warp in flight at once (per_warp = 10)
    const int my = lane < per_warp ? idx[warp * per_warp + lane] : 0;
    double2 x0[10], x1[10];
#pragma unroll
    for (int e = 0; e < 10; ++e) {
        const int r = __shfl_sync(0xffffffffu, my, e);
        const int c0 = 2 * lane, c1 = 64 + 2 * lane;
        x0[e] = __ldg(reinterpret_cast<const double2*>(tab + (size_t)r * ld + c0));
        x1[e] = c1 < ncols ? __ldg(reinterpret_cast<const double2*>(tab + (size_t)r * ld + c1)) : make_double2(0, 0);
    }
#pragma unroll
    for (int e = 0; e < 10; ++e) {
        acc0.x += x0[e].x;
        acc0.y += x0[e].y;
        acc1.x += x1[e].x;
        acc1.y += x1[e].y;
    }
    out[(size_t)warp * 64 + lane] = acc0.x + acc0.y + acc1.x + acc1.y;
}

int main(int argc, char** argv) {
    // argv[1]: gathers per launch in units of 1e5 (default 1 = one c2 SpMM's worth); larger
    // values measure the sustained rate without the launch ramp-up and tail of a ~10 us kernel
    const int scale = argc > 1 ? std::atoi(argv[1]) : 1;
    const int rows = 10000, ld = 104, ncols = 104, per_warp = 10, ngroups = 10000 * scale;
    const size_t gathers = (size_t)per_warp * ngroups;
    std::vector<int> h_idx(gathers);
    srand(1);
    for (auto& v : h_idx) v = rand() % rows;
    std::printf("gathers per launch: %zu\n", gathers);
    int* d_idx;
    double *tab, *out, *seq_idx_tab;
    CK(cudaMalloc(&d_idx, gathers * sizeof(int)));
    CK(cudaMalloc(&tab, (size_t)rows * ld * sizeof(double)));
    CK(cudaMalloc(&out, (size_t)ngroups * 64 * sizeof(double)));
    CK(cudaMemset(tab, 0, (size_t)rows * ld * sizeof(double)));
    CK(cudaMemcpy(d_idx, h_idx.data(), gathers * sizeof(int), cudaMemcpyHostToDevice));
    // sequential pattern: warp w reads rows w*10 .. w*10+9 (mod rows)
    std::vector<int> h_seq(gathers);
    for (size_t i = 0; i < gathers; ++i) h_seq[i] = (int)(i % rows);
    int* d_seq;
    CK(cudaMalloc(&d_seq, gathers * sizeof(int)));
    CK(cudaMemcpy(d_seq, h_seq.data(), gathers * sizeof(int), cudaMemcpyHostToDevice));
    (void)seq_idx_tab;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const unsigned grid = (ngroups * 32 + 255) / 256;
    const double bytes = (double)gathers * ncols * sizeof(double);
    for (int pass = 0; pass < 2; ++pass) {
        const int* ix = pass == 0 ? d_idx : d_seq;
        float best = 1e30f;
        for (int it = 0; it < 60; ++it) {
            CK(cudaEventRecord(a));
            gather<<<grid, 256>>>(ix, per_warp, ngroups, tab, ld, ncols, out);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (it >= 10 && ms < best) best = ms;
        }
        std::printf("%s: %.2f us, %.1f GB/s (%.0f MB)\n", pass == 0 ? "random gather" : "sequential rows",
                    best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 1e6);
    }
    return 0;
}
