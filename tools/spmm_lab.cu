// spmm_lab.cu -- design experiments for the flush SpMM on a real flush buffer (tools/dump_flush.py).
//   spmm_lab <flush.bin> [reps]
// Variants of the ell-wide gather SpMM, both directions (CSR: Y = A'W, CSC: W = A'^T Y), timed with
// CUDA events, each checked against the library's spmm() (same per-row FMA order => equal bits for
// rows without pieces; long rows are summed in pieces, so those may differ by roundoff):
//   sched   static grid-stride (the library) | persistent grid + atomic work queue over rows in
//           longest-first order (no tail wave)
//   NB      nonzeros whose panel rows are in flight per warp (4 | 8)
//   POL     0 = ld.global.nc for every gather; 1 = hot columns (the top of the flush's column
//           frequency ranking, flagged in bit 31 of the index) cached normally, the rest
//           L1::no_allocate, so cold rows stop evicting the hot set from L1
//   S       SM-sliced panels: SM s only handles columns [s % S] of every row, so each SM's L1
//           holds S times as many (narrower) hot rows
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "../paper_1602_00412_b200/csrc/sparse.cuh"

using namespace sfdg;

#define CKL(x)                                                                              \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));      \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

constexpr int kPc = 128;  // piece length for long rows

__device__ __forceinline__ double2 ld_nc(const double* p) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_noalloc(const double* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_last(const double* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::evict_last.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

template <int NB, int POL, int JS>
__device__ __forceinline__ void gather(int kb, int ke, const int* __restrict__ idx, const double* __restrict__ val,
                                       const double* __restrict__ in, int ld, int c0, int ncols, int lane,
                                       double2 (&acc)[JS]) {
    for (int k0 = kb; k0 < ke; k0 += 32) {
        const int kk = k0 + lane;
        const int my_idx = kk < ke ? idx[kk] : 0;
        const double my_val = kk < ke ? val[kk] : 0.0;
        const int cnt = min(32, ke - k0);
        int e = 0;
        for (; e + NB <= cnt; e += NB) {
            int ci[NB];
            double cv[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                ci[u] = __shfl_sync(0xffffffffu, my_idx, e + u);
                cv[u] = __shfl_sync(0xffffffffu, my_val, e + u);
            }
            double2 x[NB][JS];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const double* rp = in + (size_t)(ci[u] & 0x7fffffff) * ld + c0;
#pragma unroll
                for (int j = 0; j < JS; ++j) {
                    const int c = 2 * lane + 64 * j;
                    if (c0 + c < ncols) {
                        if constexpr (POL == 0) x[u][j] = ld_nc(rp + c);
                        else x[u][j] = ci[u] < 0 ? ld_last(rp + c) : ld_noalloc(rp + c);
                    } else {
                        x[u][j] = make_double2(0.0, 0.0);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < NB; ++u)
#pragma unroll
                for (int j = 0; j < JS; ++j) {
                    acc[j].x = fma(cv[u], x[u][j].x, acc[j].x);
                    acc[j].y = fma(cv[u], x[u][j].y, acc[j].y);
                }
        }
        for (; e < cnt; ++e) {
            const int ci = __shfl_sync(0xffffffffu, my_idx, e);
            const double cv = __shfl_sync(0xffffffffu, my_val, e);
            const double* rp = in + (size_t)(ci & 0x7fffffff) * ld + c0;
#pragma unroll
            for (int j = 0; j < JS; ++j) {
                const int c = 2 * lane + 64 * j;
                if (c0 + c < ncols) {
                    const double2 x = POL == 0 ? ld_nc(rp + c) : (ci < 0 ? ld_last(rp + c) : ld_noalloc(rp + c));
                    acc[j].x = fma(cv, x.x, acc[j].x);
                    acc[j].y = fma(cv, x.y, acc[j].y);
                }
            }
        }
    }
}

// Work item w: w < np is piece w (beg/end, partial slot w), else row order[w - np] (short rows,
// longest first). Each SM serves slice (smid % S) of the columns from its own queue.
template <int NB, int POL, int JS, int MINB>
__global__ void __launch_bounds__(256, MINB) lab_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                  const double* __restrict__ val, const int* __restrict__ order,
                                                  int nshort, const int* __restrict__ pbeg,
                                                  const int* __restrict__ pend, int np, const double* __restrict__ in,
                                                  int ld, int ncols, double* __restrict__ out, int ldo,
                                                  double* __restrict__ partial, int* __restrict__ counter, int S,
                                                  int chunk, int dynamic) {
    const int lane = threadIdx.x & 31;
    int slice = 0;
    if (S > 1) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        slice = (int)(smid % (unsigned)S);
    }
    const int c0 = slice * JS * 64;
    const int total = np + nshort;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    int next = gw * chunk;
    while (true) {
        int base;
        if (dynamic) {
            if (lane == 0) base = atomicAdd(counter + slice, chunk);
            base = __shfl_sync(0xffffffffu, base, 0);
        } else {
            base = next;
            next += nw * chunk;
        }
        if (base >= total) break;
        const int lim = min(total, base + chunk);
        for (int w = base; w < lim; ++w) {
            double2 acc[JS];
#pragma unroll
            for (int j = 0; j < JS; ++j) acc[j] = make_double2(0.0, 0.0);
            double* dst;
            int kb, ke;
            if (w < np) {
                kb = pbeg[w];
                ke = pend[w];
                dst = partial + (size_t)w * ld;
            } else {
                const int r = order[w - np];
                kb = ptr[r];
                ke = ptr[r + 1];
                dst = out + (size_t)r * ldo;
            }
            gather<NB, POL, JS>(kb, ke, idx, val, in, ld, c0, ncols, lane, acc);
#pragma unroll
            for (int j = 0; j < JS; ++j) {
                const int c = c0 + 2 * lane + 64 * j;
                if (c < ncols) *reinterpret_cast<double2*>(dst + c) = acc[j];
            }
        }
    }
}

// long row l: sum its pieces [first[l], first[l+1]) in order
__global__ void fixup_kernel(const int* __restrict__ lrow, const int* __restrict__ lfirst, int nl,
                             const double* __restrict__ partial, int ld, int ncols, double* __restrict__ out, int ldo) {
    const int l = blockIdx.x;
    if (l >= nl) return;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
        double t = 0.0;
        int p = lfirst[l];
        const int pe = lfirst[l + 1];
        for (; p + 8 <= pe; p += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(partial + (size_t)(p + u) * ld + c);
#pragma unroll
            for (int u = 0; u < 8; ++u) t += v[u];
        }
        for (; p < pe; ++p) t += __ldcg(partial + (size_t)p * ld + c);
        out[(size_t)lrow[l] * ldo + c] = t;
    }
}

struct Plan {  // host-built work list for one direction
    std::vector<int> order, pbeg, pend, lrow, lfirst;
};

static Plan make_plan(const std::vector<int>& ptr, int n) {
    Plan p;
    std::vector<int> shorts;
    for (int r = 0; r < n; ++r) {
        const int len = ptr[r + 1] - ptr[r];
        if (len > 2 * kPc) {
            p.lrow.push_back(r);
            p.lfirst.push_back((int)p.pbeg.size());
            for (int k = ptr[r]; k < ptr[r + 1]; k += kPc) {
                p.pbeg.push_back(k);
                p.pend.push_back(std::min(ptr[r + 1], k + kPc));
            }
        } else {
            shorts.push_back(r);
        }
    }
    p.lfirst.push_back((int)p.pbeg.size());
    std::stable_sort(shorts.begin(), shorts.end(),
                     [&](int a, int b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
    p.order = shorts;
    return p;
}

template <class T>
static T* dev(const std::vector<T>& h) {
    T* d = nullptr;
    CKL(cudaMalloc(&d, std::max<size_t>(1, h.size()) * sizeof(T)));
    if (!h.empty()) CKL(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

template <class F>
static double time_us(cudaStream_t st, int reps, F&& f) {
    for (int i = 0; i < 2; ++i) f();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1, st);
    CKL(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e3 * ms / reps;
}

struct Dir {
    const char* name;
    int n;                  // output rows
    int nin;                // input panel rows
    std::vector<int> ptr;   // n+1
    std::vector<int> idx;   // plain
    std::vector<int> idxh;  // hot-flagged
    std::vector<double> val;
};

using KFn = void (*)(const int*, const int*, const double*, const int*, int, const int*, const int*, int,
                     const double*, int, int, double*, int, double*, int*, int, int, int);

template <int NB, int POL, int JS, int MINB = 1>
static KFn kfn() {
    return lab_kernel<NB, POL, JS, MINB>;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: spmm_lab <flush.bin> [reps]\n");
        return 1;
    }
    const int reps = argc > 2 ? atoi(argv[2]) : 10;
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
    // CSR and its stable transpose on the host
    Dir csr{"csr", m, d, std::vector<int>(m + 1), std::vector<int>(nnz), {}, vals};
    for (int i = 0; i <= m; ++i) csr.ptr[i] = (int)rp64[i];
    for (int64_t k = 0; k < nnz; ++k) csr.idx[k] = (int)cols[k];
    Dir csc{"csc", d, m, std::vector<int>(d + 1, 0), std::vector<int>(nnz), {}, std::vector<double>(nnz)};
    for (int64_t k = 0; k < nnz; ++k) csc.ptr[cols[k] + 1]++;
    for (int c = 0; c < d; ++c) csc.ptr[c + 1] += csc.ptr[c];
    {
        std::vector<int> pos(csc.ptr.begin(), csc.ptr.end() - 1);
        for (int r = 0; r < m; ++r)
            for (int k = csr.ptr[r]; k < csr.ptr[r + 1]; ++k) {
                const int p = pos[cols[k]]++;
                csc.idx[p] = r;
                csc.val[p] = vals[k];
            }
    }
    // hot flags: the most frequent input rows of each direction, as many as one SM's L1 holds
    auto flag_hot = [&](Dir& D, int nhot) {
        std::vector<int> cnt(D.nin, 0);
        for (int v : D.idx) cnt[v]++;
        std::vector<int> ids(D.nin);
        std::iota(ids.begin(), ids.end(), 0);
        nhot = std::min(nhot, D.nin);
        std::nth_element(ids.begin(), ids.begin() + (nhot - 1), ids.end(),
                         [&](int a, int b) { return cnt[a] > cnt[b]; });
        std::vector<char> hot(D.nin, 0);
        long long in_hot = 0;
        for (int i = 0; i < nhot; ++i) {
            hot[ids[i]] = 1;
            in_hot += cnt[ids[i]];
        }
        D.idxh.resize(D.idx.size());
        for (size_t k = 0; k < D.idx.size(); ++k) D.idxh[k] = hot[D.idx[k]] ? (int)(D.idx[k] | 0x80000000u) : D.idx[k];
        return (double)in_hot / (double)D.idx.size();
    };

    printf("flush m=%d d=%d ell=%d nnz=%lld; alg bytes %.1f MB, gathered %.1f MB\n", m, d, ell, (long long)nnz,
           (12.0 * nnz + 8.0 * (m + 1) + 8.0 * ell * (m + d)) / 1e6, 8.0 * lp * nnz / 1e6);
    cudaStream_t st;
    CKL(cudaStreamCreate(&st));
    int sms = 0;
    CKL(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> h((size_t)std::max(m, d) * lp, 0.0);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (i % lp) < (size_t)ell ? nd(g) : 0.0;
    double* panel = dev(h);
    double *out_ref, *out, *partial;
    CKL(cudaMalloc(&out_ref, (size_t)std::max(m, d) * lp * 8));
    CKL(cudaMalloc(&out, (size_t)std::max(m, d) * lp * 8));
    CKL(cudaMalloc(&partial, (size_t)(2 * nnz / kPc + 16) * lp * 8));
    int* counter;
    CKL(cudaMalloc(&counter, 64 * sizeof(int)));
    const double hbm = 6548.8;
    const double alg = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * ell * (m + d);

    for (Dir* D : {&csr, &csc}) {
        const int J = (lp + 63) / 64;
        const double hf = flag_hot(*D, (200 * 1024) / (lp * 8));
        Plan P = make_plan(D->ptr, D->n);
        int *d_ptr = dev(D->ptr), *d_idx = dev(D->idx), *d_idxh = dev(D->idxh);
        double* d_val = dev(D->val);
        int *d_order = dev(P.order), *d_pb = dev(P.pbeg), *d_pe = dev(P.pend), *d_lr = dev(P.lrow),
            *d_lf = dev(P.lfirst);
        const int np = (int)P.pbeg.size(), nl = (int)P.lrow.size();
        // the library's kernel
        Scratch scr, s2;
        SegPlan sp;
        sp.build(d_ptr, D->n, nnz, scr, st);
        CKL(cudaStreamSynchronize(st));
        const double t_lib = time_us(st, reps, [&] {
            s2.reset();
            spmm(d_ptr, d_idx, d_val, D->n, sp, nnz, panel, lp, lp, out_ref, lp, s2, st);
        });
        printf("[%s] long rows %d pieces %d; hot rows flagged hold %.1f%% of entries\n", D->name, nl, np, 100 * hf);
        printf("  %-34s %8.1f us  frac %.3f\n", "library spmm", t_lib, alg / t_lib / 1e3 / hbm);
        std::vector<double> ref((size_t)D->n * lp), got((size_t)D->n * lp);
        CKL(cudaMemcpy(ref.data(), out_ref, ref.size() * 8, cudaMemcpyDeviceToHost));
        struct V {
            const char* name;
            KFn fn;
            int pol, S, js, dyn, ord;
        };
        std::vector<int> ident(P.order);
        std::sort(ident.begin(), ident.end());
        int* d_ident = dev(ident);
        std::vector<V> vs;
#define ADD(NM, NB, POL, JS, MINB, S, DYN, ORD) vs.push_back(V{NM, kfn<NB, POL, JS, MINB>(), POL, S, JS, DYN, ORD})
        if (J == 2) {
            ADD("static natural NB4 mb5", 4, 0, 2, 5, 1, 0, 0);
            ADD("static LPT NB4 mb5", 4, 0, 2, 5, 1, 0, 1);
            ADD("static LPT NB4 mb4", 4, 0, 2, 4, 1, 0, 1);
            ADD("dyn natural NB4 mb5", 4, 0, 2, 5, 1, 1, 0);
            ADD("dyn LPT NB4 mb5", 4, 0, 2, 5, 1, 1, 1);
            ADD("dyn LPT NB8 mb4", 8, 0, 2, 4, 1, 1, 1);
            ADD("dyn LPT NB8 mb3", 8, 0, 2, 3, 1, 1, 1);
            ADD("dyn LPT NB2 mb6", 2, 0, 2, 6, 1, 1, 1);
        } else {
            ADD("static natural NB4 mb2", 4, 0, 4, 2, 1, 0, 0);
            ADD("static natural NB4 mb3", 4, 0, 4, 3, 1, 0, 0);
            ADD("static natural NB4 mb4", 4, 0, 4, 4, 1, 0, 0);
            ADD("static LPT NB4 mb2", 4, 0, 4, 2, 1, 0, 1);
            ADD("dyn natural NB4 mb2", 4, 0, 4, 2, 1, 1, 0);
            ADD("dyn LPT NB4 mb2", 4, 0, 4, 2, 1, 1, 1);
            ADD("dyn natural NB2 mb3", 2, 0, 4, 3, 1, 1, 0);
            ADD("dyn natural NB8 mb2", 8, 0, 4, 2, 1, 1, 0);
        }
#undef ADD
        for (const V& v : vs) {
            if (v.js * v.S < J) continue;
            int bps = 0;
            CKL(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (const void*)v.fn, 256, 0));
            const int grid = v.dyn ? bps * sms : std::min(16 * sms, (D->n * 64 + 255) / 256);
            const int* ix = v.pol ? d_idxh : d_idx;
            const int* od = v.ord ? d_order : d_ident;
            auto run_main = [&] {
                if (v.dyn) CKL(cudaMemsetAsync(counter, 0, 64 * sizeof(int), st));
                v.fn<<<grid, 256, 0, st>>>(d_ptr, ix, d_val, od, (int)P.order.size(), d_pb, d_pe, np, panel, lp, lp,
                                           out, lp, partial, counter, v.S, 1, v.dyn);
            };
            auto run_fix = [&] {
                if (nl) fixup_kernel<<<nl, 128, 0, st>>>(d_lr, d_lf, nl, partial, lp, lp, out, lp);
            };
            CKL(cudaMemsetAsync(out, 0, (size_t)D->n * lp * 8, st));
            const double tm = time_us(st, reps, run_main);
            const double tf = time_us(st, reps, run_fix);
            CKL(cudaMemcpy(got.data(), out, got.size() * 8, cudaMemcpyDeviceToHost));
            size_t ndiff = 0;
            double maxrel = 0;
            for (size_t i = 0; i < got.size(); ++i) {
                if (got[i] != ref[i]) {
                    ++ndiff;
                    maxrel = std::max(maxrel, std::fabs(got[i] - ref[i]) / (std::fabs(ref[i]) + 1e-300));
                }
            }
            printf("  %-28s main %8.1f us + fixup %6.1f us  frac(main) %.3f  (%d blk/SM)  diff %zu maxrel %.1e\n",
                   v.name, tm, tf, alg / tm / 1e3 / hbm, bps, ndiff, maxrel);
        }
    }
    printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
