// spmm_bench.cu -- the flush SpMMs (Y = A'W over the CSR, W = A'^T Y over the CSC) on a real
// flush buffer written by tools/dump_flush.py, timed with CUDA events on the launching stream.
//   spmm_bench <flush.bin> [reps]
// Reports per launch: microseconds, SURVEY 8(d) algorithmic bytes / time (the roofline's
// `achieved`), and the L2 -> SM gather rate (one ell-wide panel row per stored entry).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1602_00412_b200/csrc/sparse.cuh"

using namespace sfdg;

template <class F>
static double time_us(cudaStream_t st, int reps, F&& f) {
    for (int i = 0; i < 2; ++i) f();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e3 * ms / reps;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: spmm_bench <flush.bin> [reps]\n");
        return 1;
    }
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 1;
    int64_t hdr[4];
    if (fread(hdr, 8, 4, f) != 4) return 1;
    const int m = (int)hdr[0], d = (int)hdr[1], ell = (int)hdr[3];
    const int64_t nnz = hdr[2];
    const int lp = (ell + 7) / 8 * 8;
    std::vector<int64_t> rp64(m + 1);
    std::vector<uint32_t> cols(nnz);
    std::vector<double> vals(nnz);
    if (fread(rp64.data(), 8, m + 1, f) != (size_t)m + 1 || fread(cols.data(), 4, nnz, f) != (size_t)nnz ||
        fread(vals.data(), 8, nnz, f) != (size_t)nnz)
        return 1;
    fclose(f);
    std::vector<int> rp(m + 1);
    for (int i = 0; i <= m; ++i) rp[i] = (int)rp64[i];
    cudaStream_t st;
    cudaStreamCreate(&st);
    Scratch scr, s2;
    DevCsr a;
    a.set_shape(m, d, nnz);
    cudaMemcpy(a.row_ptr, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(a.col, cols.data(), nnz * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(a.val, vals.data(), nnz * 8, cudaMemcpyHostToDevice);
    SegPlan pr, pc;
    build_transpose(a, scr, st);
    pr.build(a.row_ptr, m, a.nnz, scr, st);
    pc.build(a.col_ptr, d, a.nnz, scr, st);
    cudaStreamSynchronize(st);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> h((size_t)std::max(m, d) * lp, 0.0);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (i % lp) < (size_t)ell ? nd(g) : 0.0;
    double *Y, *W;
    cudaMalloc(&Y, (size_t)m * lp * 8);
    cudaMalloc(&W, (size_t)d * lp * 8);
    cudaMemcpy(Y, h.data(), (size_t)m * lp * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(W, h.data(), (size_t)d * lp * 8, cudaMemcpyHostToDevice);
    const double alg = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * ell * d + 8.0 * ell * m;
    const double gath = 8.0 * lp * nnz;
    printf("flush m=%d d=%d ell=%d lp=%d nnz=%lld (%.1f per row); alg bytes %.1f MB, gathered %.1f MB\n", m, d, ell,
           lp, (long long)nnz, (double)nnz / m, alg / 1e6, gath / 1e6);
    const double hbm = 6548.8;
    const double t_csr = time_us(st, reps, [&] {
        s2.reset();
        spmm(a.row_ptr, (const int*)a.col, a.val, m, pr, a.nnz, W, lp, lp, Y, lp, s2, st);
    });
    const double t_csc = time_us(st, reps, [&] {
        s2.reset();
        spmm(a.col_ptr, a.row_idx, a.cval, d, pc, a.nnz, Y, lp, lp, W, lp, s2, st);
    });
    // hot-column staging for the CSR direction (the engine's per-flush choice, Engine::choose_hot)
    const int cap = std::min(hot_rows_capacity(lp), d);
    std::vector<int> cp(d + 1), ids(d);
    cudaMemcpy(cp.data(), a.col_ptr, (d + 1) * 4, cudaMemcpyDeviceToHost);
    for (int c = 0; c < d; ++c) ids[c] = c;
    auto cnt = [&](int c) { return cp[c + 1] - cp[c]; };
    auto better = [&](int x, int y) { return cnt(x) != cnt(y) ? cnt(x) > cnt(y) : x < y; };
    std::nth_element(ids.begin(), ids.begin() + (cap - 1), ids.end(), better);
    std::sort(ids.begin(), ids.begin() + cap, better);
    long long in_hot = 0;
    for (int i = 0; i < cap; ++i) in_hot += cnt(ids[i]);
    int *hcols, *slot, *idx2;
    cudaMalloc(&hcols, cap * 4);
    cudaMalloc(&slot, (size_t)d * 4);
    cudaMalloc(&idx2, nnz * 4);
    cudaMemcpy(hcols, ids.data(), cap * 4, cudaMemcpyHostToDevice);
    hot_relabel(hcols, cap, a.col, nnz, d, slot, idx2, st);
    HotSet hs{hcols, idx2, cap};
    double* Y2;
    cudaMalloc(&Y2, (size_t)m * lp * 8);
    const double t_hot = time_us(st, reps, [&] {
        s2.reset();
        spmm(a.row_ptr, (const int*)a.col, a.val, m, pr, a.nnz, W, lp, lp, Y2, lp, s2, st, -1, -1, &hs);
    });
    s2.reset();
    spmm(a.row_ptr, (const int*)a.col, a.val, m, pr, a.nnz, W, lp, lp, Y, lp, s2, st);
    cudaStreamSynchronize(st);
    std::vector<double> h1((size_t)m * lp), h2((size_t)m * lp);
    cudaMemcpy(h1.data(), Y, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), Y2, h2.size() * 8, cudaMemcpyDeviceToHost);
    size_t diff = 0;
    for (size_t i = 0; i < h1.size(); ++i) diff += h1[i] != h2[i];
    printf("hot columns: %d staged rows hold %.1f%% of the entries; hot result differs in %zu of %zu values\n", cap,
           100.0 * in_hot / nnz, diff, h1.size());
    for (auto [name, t] : {std::pair<const char*, double>{"csr (Y = A'W)", t_csr}, {"csr + hot smem", t_hot},
                           {"csc (W = A'^T Y)", t_csc}})
        printf("%-18s %9.2f us  alg %7.1f GB/s (frac %.3f of %.0f)  gather %7.1f GB/s\n", name, t, alg / t / 1e3,
               alg / t / 1e3 / hbm, hbm, gath / t / 1e3);
    printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
