// kbench.cu -- per-kernel microbenchmarks of libsfdg's device building blocks at the
// c2 flush shape (m = d = 1e4, ell = 100 -> lp = 104, ~10 nnz/row), timed with CUDA
// events on the launching stream. Build: make -C tools kbench (links libsfdg.so).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1602_00412_b200/csrc/dense.cuh"
#include "../paper_1602_00412_b200/csrc/sparse.cuh"

using namespace sfdg;

template <class F>
static double time_us(cudaStream_t st, int reps, F&& f) {
    for (int i = 0; i < 3; ++i) f();
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
    const int m = argc > 1 ? atoi(argv[1]) : 10000;
    const int d = m;
    const int ell = argc > 2 ? atoi(argv[2]) : 100;
    const int lp = (ell + 7) / 8 * 8;
    const int nnz_row = argc > 3 ? atoi(argv[3]) : 10;
    const int reps = argc > 4 ? atoi(argv[4]) : 50;
    cudaStream_t st;
    cudaStreamCreate(&st);
    Scratch scr;
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    // panels
    std::vector<double> hY((size_t)m * lp);
    for (auto& v : hY) v = nd(g);
    for (int i = 0; i < m; ++i)
        for (int j = ell; j < lp; ++j) hY[(size_t)i * lp + j] = 0.0;
    double *Y, *Y2, *W, *G, *R, *st4, *K;
    int* err;
    cudaMalloc(&Y, 2 * hY.size() * 8);  // eigh test Grams read 2 lp columns
    cudaMemset(Y, 0, 2 * hY.size() * 8);
    cudaMalloc(&Y2, hY.size() * 8);
    cudaMalloc(&W, (size_t)d * lp * 8);
    cudaMalloc(&G, (size_t)4 * lp * lp * 8);
    cudaMalloc(&R, (size_t)lp * lp * 8);
    cudaMalloc(&K, (size_t)4 * lp * lp * 8);
    cudaMalloc(&st4, 64);
    cudaMalloc(&err, 16);
    cudaMemset(err, 0, 16);
    cudaMemcpy(Y, hY.data(), hY.size() * 8, cudaMemcpyHostToDevice);
    // sparse A' (m x d)
    std::vector<int> rp(m + 1, 0);
    std::vector<uint32_t> cols;
    std::vector<double> vals;
    std::uniform_int_distribution<int> ud(0, d - 1);
    for (int i = 0; i < m; ++i) {
        std::vector<int> r;
        for (int k = 0; k < nnz_row; ++k) r.push_back(ud(g));
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        for (int c : r) {
            cols.push_back((uint32_t)c);
            vals.push_back(nd(g));
        }
        rp[i + 1] = (int)cols.size();
    }
    DevCsr a;
    a.set_shape(m, d, (int64_t)cols.size());
    cudaMemcpy(a.row_ptr, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(a.col, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(a.val, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice);
    SegPlan pr, pc;
    build_transpose(a, scr, st);
    pr.build(a.row_ptr, m, a.nnz, scr, st);
    pc.build(a.col_ptr, d, a.nnz, scr, st);
    cudaStreamSynchronize(st);
    Scratch s2;
    printf("shape m=d=%d ell=%d lp=%d nnz=%zu\n", m, ell, lp, cols.size());
    printf("spmm_csr    %8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               spmm(a.row_ptr, (const int*)a.col, a.val, m, pr, a.nnz, W, lp, lp, Y2, lp, s2, st);
           }));
    printf("spmm_csc    %8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               spmm(a.col_ptr, a.row_idx, a.cval, d, pc, a.nnz, Y, lp, lp, W, lp, s2, st);
           }));
    printf("gram m x lp %8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               gram_tn(Y, m, lp, lp, G, lp, s2, st);
           }));
    printf("gram d x 2lp%8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               gram_tn(Y, m / 2, 2 * lp, 2 * lp, K, 2 * lp, s2, st);
           }));
    // make G SPD & well conditioned: G = Y^T Y / m + I
    gram_tn(Y, m, lp, lp, G, lp, s2, st);
    printf("chol        %8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               chol_factor(G, lp, lp, R, R + lp * lp / 2, nullptr, 0, st4, err, 1, s2, st, false);
           }));
    printf("chol_polar  %8.2f us\n", time_us(st, reps, [&] {
               s2.reset();
               chol_factor(G, lp, lp, R, R + lp * lp / 2, K, lp, st4, err, 1, s2, st, true);
           }));
    printf("gemm m x lp %8.2f us\n", time_us(st, reps, [&] { gemm_nn(Y, m, lp, lp, R, lp, lp, Y2, lp, st); }));
    {  // CholeskyQR apply: X = Y R^-1 (trinv + triangular DMMA GEMM, the engine's default)
        double *Rf, *D8, *Tinv;
        cudaMalloc(&Rf, (size_t)lp * lp * 8);
        cudaMalloc(&D8, (size_t)lp * 8 * 8);
        cudaMalloc(&Tinv, (size_t)lp * lp * 8);
        gram_tn(Y, m, lp, lp, G, lp, s2, st);
        chol_factor(G, lp, lp, Rf, D8, nullptr, 0, st4, err, 1, s2, st, false);
        printf("trsm m x lp %8.2f us\n", time_us(st, reps, [&] {
                   trsm_apply(Y, m, lp, lp, Rf, D8, Y2, lp, nullptr, st, Tinv);
               }));
        cudaFree(Rf);
        cudaFree(D8);
        cudaFree(Tinv);
    }
    for (int n : {ell, 2 * ell}) {
        double* vals_d;
        double* vecs;
        cudaMalloc(&vals_d, n * 8);
        cudaMalloc(&vecs, (size_t)n * n * 8);
        gram_tn(Y, m, n, n <= lp ? lp : 2 * lp, K, n, s2, st);  // a dense SPD test matrix
        const int r = std::max(1, reps / 10);
        printf("eigh n=%-4d %8.2f us\n", n, time_us(st, r, [&] {
                   s2.reset();
                   eigh(K, n, n, 1e-12 * 1e4 * n, nullptr, vals_d, vecs, n, err, s2, st);
               }));
        printf("eigh n=%-4d top %d %8.2f us\n", n, ell, time_us(st, r, [&] {
                   s2.reset();
                   eigh(K, n, n, 1e-12 * 1e4 * n, nullptr, vals_d, vecs, n, err, s2, st, ell);
               }));
    }
    int herr = 0;
    cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
    printf("err flags %d, cuda %s\n", herr, cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
