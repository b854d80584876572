// spmv_lab.cu -- design experiments for the verifier's SpMV u = A' x (one FP64 column) on a real
// flush buffer (tools/dump_flush.py), warm, CUDA events. Variants:
//   grp8    8 lanes per row, rows longest first, 4 entries per lane in flight (vg_rows today)
//   grpG    G lanes per row (G = 4, 16, 32)
//   *_ldg   the x gather through L1 (ld.global.nc): safe in a kernel sequence, x is read-only
//           for the launch and L1 is invalidated at launch boundaries
//   spmv <flush.bin> [reps]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CKL(x)                                                                         \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

template <bool LDG>
__device__ __forceinline__ double gx(const double* x, int c) {
    if constexpr (LDG) return __ldg(x + c);
    else return __ldcg(x + c);
}

template <int G, bool LDG, int U>
__global__ void __launch_bounds__(256) grp_kernel(const int* __restrict__ ptr, const int* __restrict__ col,
                                                  const double* __restrict__ val, const int* __restrict__ order,
                                                  int n, const double* __restrict__ x, double* __restrict__ u) {
    const int lane = threadIdx.x & 31, sub = lane & (G - 1);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t gi = gw; gi < n; gi += ng) {
        const int r = order[gi];
        const int kb = ptr[r], ke = ptr[r + 1];
        double sp[U];
#pragma unroll
        for (int q = 0; q < U; ++q) sp[q] = 0.0;
        for (int k = kb + sub; k < ke; k += G * U) {
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (k + G * q < ke) sp[q] = fma(val[k + G * q], gx<LDG>(x, col[k + G * q]), sp[q]);
        }
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < U; ++q) t += sp[q];
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (sub == 0) u[r] = t;
    }
}

// the rows stored in the processing (LPT) order: start offsets in the permuted storage, so the
// chain is start -> entries -> x; the output index is an independent load
template <int G, int U>
__global__ void __launch_bounds__(256) perm_kernel(const int* __restrict__ pptr, const int* __restrict__ col,
                                                   const double* __restrict__ val, const int* __restrict__ order,
                                                   int n, const double* __restrict__ x, double* __restrict__ u) {
    const int lane = threadIdx.x & 31, sub = lane & (G - 1);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t gi = gw; gi < n; gi += ng) {
        const int kb = pptr[gi], ke = pptr[gi + 1];
        const int r = order[gi];
        double sp[U];
#pragma unroll
        for (int q = 0; q < U; ++q) sp[q] = 0.0;
        for (int k = kb + sub; k < ke; k += G * U) {
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (k + G * q < ke) sp[q] = fma(val[k + G * q], __ldg(x + col[k + G * q]), sp[q]);
        }
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < U; ++q) t += sp[q];
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (sub == 0) u[r] = t;
    }
}

template <class T>
static T* dev(const std::vector<T>& h) {
    T* d = nullptr;
    CKL(cudaMalloc(&d, std::max<size_t>(1, h.size()) * sizeof(T)));
    if (!h.empty()) CKL(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

template <class F>
static double time_us(int reps, F&& f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1);
    CKL(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e3 * ms / reps;
}

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    const int reps = argc > 2 ? atoi(argv[2]) : 50;
    FILE* f = fopen(argv[1], "rb");
    int64_t hdr[4];
    if (!f || fread(hdr, 8, 4, f) != 4) return 1;
    const int m = (int)hdr[0], d = (int)hdr[1];
    const int64_t nnz = hdr[2];
    std::vector<int64_t> rp64(m + 1);
    std::vector<uint32_t> cols(nnz);
    std::vector<double> vals(nnz);
    if (fread(rp64.data(), 8, m + 1, f) != (size_t)m + 1 || fread(cols.data(), 4, nnz, f) != (size_t)nnz ||
        fread(vals.data(), 8, nnz, f) != (size_t)nnz)
        return 1;
    fclose(f);
    // both directions: CSR (u = A'x) and CSC (w = A'^T u)
    struct Op {
        const char* name;
        int n, nin;
        std::vector<int> ptr, idx;
        std::vector<double> v;
    };
    Op csr{"csr", m, d, std::vector<int>(m + 1), std::vector<int>(nnz), vals};
    for (int i = 0; i <= m; ++i) csr.ptr[i] = (int)rp64[i];
    for (int64_t k = 0; k < nnz; ++k) csr.idx[k] = (int)cols[k];
    Op csc{"csc", d, m, std::vector<int>(d + 1, 0), std::vector<int>(nnz), std::vector<double>(nnz)};
    for (int64_t k = 0; k < nnz; ++k) csc.ptr[cols[k] + 1]++;
    for (int c = 0; c < d; ++c) csc.ptr[c + 1] += csc.ptr[c];
    {
        std::vector<int> pos(csc.ptr.begin(), csc.ptr.end() - 1);
        for (int r = 0; r < m; ++r)
            for (int k = csr.ptr[r]; k < csr.ptr[r + 1]; ++k) {
                const int p = pos[cols[k]]++;
                csc.idx[p] = r;
                csc.v[p] = vals[k];
            }
    }
    printf("flush m=%d d=%d nnz=%lld\n", m, d, (long long)nnz);
    int sms = 0;
    CKL(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (Op* O : {&csr, &csc}) {
        std::vector<int> ord(O->n), nat(O->n);
        std::iota(ord.begin(), ord.end(), 0);
        std::iota(nat.begin(), nat.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
            return O->ptr[a + 1] - O->ptr[a] > O->ptr[b + 1] - O->ptr[b];
        });
        std::mt19937_64 g(3);
        std::normal_distribution<double> nd;
        std::vector<double> hx(O->nin);
        for (auto& v : hx) v = nd(g);
        std::vector<double> ref(O->n, 0.0);
        for (int r = 0; r < O->n; ++r) {
            long double s = 0;
            for (int k = O->ptr[r]; k < O->ptr[r + 1]; ++k) s += (long double)O->v[k] * hx[O->idx[k]];
            ref[r] = (double)s;
        }
        int *dp = dev(O->ptr), *di = dev(O->idx), *dord = dev(ord), *dnat = dev(nat);
        double *dv = dev(O->v), *dx = dev(hx), *du;
        CKL(cudaMalloc(&du, O->n * 8));
        std::vector<double> got(O->n);
        auto check = [&]() {
            CKL(cudaMemcpy(got.data(), du, O->n * 8, cudaMemcpyDeviceToHost));
            double mx = 0;
            for (int r = 0; r < O->n; ++r) mx = std::max(mx, std::fabs(got[r] - ref[r]) / (std::fabs(ref[r]) + 1e-3));
            return mx;
        };
        struct V {
            const char* name;
            void (*fn)(const int*, const int*, const double*, const int*, int, const double*, double*);
            int G;
            bool lpt;
        };
        std::vector<V> vs = {
            {"grp8 U4 ldcg LPT", grp_kernel<8, false, 4>, 8, true},   {"grp8 U4 ldg LPT", grp_kernel<8, true, 4>, 8, true},
            {"grp8 U4 ldg natural", grp_kernel<8, true, 4>, 8, false}, {"grp8 U8 ldg LPT", grp_kernel<8, true, 8>, 8, true},
            {"grp4 U8 ldg LPT", grp_kernel<4, true, 8>, 4, true},     {"grp16 U4 ldg LPT", grp_kernel<16, true, 4>, 16, true},
            {"grp32 U4 ldg LPT", grp_kernel<32, true, 4>, 32, true},  {"grp32 U2 ldcg LPT", grp_kernel<32, false, 2>, 32, true},
            {"grp4 U4 ldg LPT", grp_kernel<4, true, 4>, 4, true},     {"grp2 U8 ldg LPT", grp_kernel<2, true, 8>, 2, true},
        };
        {  // permuted storage in LPT order
            std::vector<int> pptr(O->n + 1, 0), pidx;
            std::vector<double> pv;
            for (int gi = 0; gi < O->n; ++gi) {
                const int r = ord[gi];
                for (int k = O->ptr[r]; k < O->ptr[r + 1]; ++k) {
                    pidx.push_back(O->idx[k]);
                    pv.push_back(O->v[k]);
                }
                pptr[gi + 1] = (int)pidx.size();
            }
            int *dpp = dev(pptr), *dpi = dev(pidx);
            double* dpv = dev(pv);
            for (int bps : {4, 6, 8}) {
                const int grid = bps * sms;
                CKL(cudaMemset(du, 0, O->n * 8));
                double t = time_us(reps, [&] { perm_kernel<16, 4><<<grid, 256>>>(dpp, dpi, dpv, dord, O->n, dx, du); });
                printf("[%s] %-22s %d blk/SM  %7.1f us  maxrel %.1e\n", O->name, "perm16 U4 ldg LPT", bps, t, check());
                CKL(cudaMemset(du, 0, O->n * 8));
                t = time_us(reps, [&] { perm_kernel<8, 4><<<grid, 256>>>(dpp, dpi, dpv, dord, O->n, dx, du); });
                printf("[%s] %-22s %d blk/SM  %7.1f us  maxrel %.1e\n", O->name, "perm8 U4 ldg LPT", bps, t, check());
            }
            cudaFree(dpp);
            cudaFree(dpi);
            cudaFree(dpv);
        }
        for (const V& v : vs) {
            for (int bps : {4, 6, 8}) {
                const int grid = bps * sms;
                const int* o = v.lpt ? dord : dnat;
                CKL(cudaMemset(du, 0, O->n * 8));
                const double t = time_us(reps, [&] { v.fn<<<grid, 256>>>(dp, di, dv, o, O->n, dx, du); });
                printf("[%s] %-22s %d blk/SM  %7.1f us  maxrel %.1e\n", O->name, v.name, bps, t, check());
            }
        }
        cudaFree(dp);
        cudaFree(di);
        cudaFree(dord);
        cudaFree(dnat);
        cudaFree(dv);
        cudaFree(dx);
        cudaFree(du);
    }
    printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
