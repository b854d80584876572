// tri_probe.cu -- where a Householder step of the single-CTA row tridiagonalisation goes:
// eigh_tri.cu compiled with SFDG_TRI_PROBE stamps clock64() per step (0 step start, 1 owner
// warp done with S1, 2 after barrier 1, 3/4 warps 0 and NW-1 done with S2, 5 after barrier 2).
// Build: make -C tools tri_probe. Run: tools/tri_probe [n]
#define SFDG_TRI_PROBE 1
#include "../paper_1602_00412_b200/csrc/eigh_tri.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char** argv) {
    using namespace sfdg;
    const int n = argc > 1 ? atoi(argv[1]) : 100;
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> a((size_t)(n + 5) * n), K((size_t)n * n, 0.0);
    for (auto& v : a) v = nd(g);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int r = 0; r < n + 5; ++r) s += a[(size_t)r * n + i] * a[(size_t)r * n + j];
            K[(size_t)i * n + j] = s;
        }
    double *dK, *vals, *vecs;
    int* fb;
    cudaMalloc(&dK, K.size() * 8);
    cudaMalloc(&vals, n * 8);
    cudaMalloc(&vecs, (size_t)n * n * 8);
    cudaMalloc(&fb, 4);
    cudaMemcpy(dK, K.data(), K.size() * 8, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreate(&st);
    Scratch scr;
    for (int it = 0; it < 3; ++it) {
        scr.reset();
        eigh_tri(dK, n, n, 1e-12, nullptr, n / 2, vals, vecs, n, fb, scr, st);
    }
    cudaStreamSynchronize(st);
    std::vector<long long> p(8 * 1100);
    cudaMemcpyFromSymbol(p.data(), g_tri_probe, p.size() * 8);
    printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
    double tot[5] = {0};
    int cnt = 0;
    for (int k = 0; k + 1 < n; ++k) {
        const long long* q = &p[8 * k];
        const double s1 = q[1] - q[0], b1 = q[2] - q[1], s2a = q[3] - q[2], s2b = q[4] - q[2], b2 = q[5] - std::max(q[3], q[4]);
        if (k < 4 || k % 20 == 0)
            printf("k=%3d S1 %6.0f  bar1 %5.0f  S2(w0) %6.0f  S2(wlast) %6.0f  bar2 %5.0f  step %6lld cycles\n", k, s1, b1,
                   s2a, s2b, b2, k + 2 < n ? p[8 * (k + 1)] - q[0] : 0);
        tot[0] += s1; tot[1] += b1; tot[2] += s2a; tot[3] += s2b; tot[4] += b2;
        ++cnt;
    }
    printf("mean cycles: S1 %.0f bar1 %.0f S2(w0) %.0f S2(wlast) %.0f bar2 %.0f; total %lld cycles for %d steps\n",
           tot[0] / cnt, tot[1] / cnt, tot[2] / cnt, tot[3] / cnt, tot[4] / cnt, p[8 * (n - 2) + 5] - p[0], cnt);
    return 0;
}
