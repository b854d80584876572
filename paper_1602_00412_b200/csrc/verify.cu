// verify.cu -- the spectral-norm verifier as one persistent cooperative kernel.
//
// Reference: verify_spectral (core/src/shrink.cpp:75-102) runs `steps` power-method
// steps on diff_op(x) = (2/Delta)(A'^T A' x - B'^T B' x) (shrink.cpp:121-126) from a
// random unit vector (la_core.cpp:174-189), tracking log|y| and exiting early on
// annihilation (accept) or on growth past 1 (reject). Every step depends on the last and
// has a global norm, so a host loop would pay a launch + round trip per step. Here all
// steps run in one cooperative grid; block b owns a contiguous chunk of rows of A' (for
// u = A'x) and a contiguous chunk of columns (for y and the rows of B'^T). Per step:
//   phase A: u = A' x                                     (CSR, warp per row)  | barrier
//   phase B: y_c = scale (A'^T u - B'^T t)_c for own columns (CSC + B'^T row), and, from the
//            same B'^T rows still in registers, the partials of next t = B' y and |y|^2
//                                                                              | barrier
//   phase C: every block reduces |y|^2 and t in the same fixed order, so all blocks take
//            the same accept / reject / continue decision with no further sync.
// B'^T is therefore streamed once per step (it is the bulk: d x ell FP64), not twice.
// x = y / |y| is never materialised: it is y scaled by 1/|y| on the fly (the reference
// divides; the two differ by at most one ulp per entry).
#include <map>
#include <mutex>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sparse.cuh"
#include "verify.cuh"

namespace sfdg {

namespace {

constexpr int kVThreads = 512;
constexpr int kVWarps = kVThreads / 32;
constexpr int kMaxQ = 8;  // ell <= 256 = 32 lanes x 8

struct GridBar {
    unsigned* count;
    unsigned* gen;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Generation barrier: the last arriving block resets the count and bumps the generation;
// the others spin on an acquire load.
__device__ __forceinline__ void grid_sync(const GridBar& b, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(b.gen);
        __threadfence();
        if (atomicAdd(b.count, 1u) == nblocks - 1) {
            atomicExch(b.count, 0u);
            __threadfence();
            atomicAdd(b.gen, 1u);
        } else {
            while (ld_acquire(b.gen) == g) __nanosleep(32);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum of the nb per-block partials in a fixed order: every block gets the identical value.
__device__ __forceinline__ double grid_total(const double* part, unsigned nb, double* sh) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < nb; b += 32) s += __ldcg(part + b);
        s = warp_sum(s);
        if (threadIdx.x == 0) sh[0] = s;
    }
    __syncthreads();
    const double t = sh[0];
    __syncthreads();
    return t;
}

// t[j] = scale * sum_b tp[b][j] for all j < L, reduced identically in every block: kSplit
// threads per entry each sum a fixed stride of blocks (all loads in flight at once), then
// the kSplit partials are combined in a fixed order.
constexpr int kSplit = 4;
__device__ __forceinline__ void reduce_t(const double* tp, unsigned nb, int L, double scale, double* tloc,
                                         double* scratch /* kSplit * 256 */) {
    for (int e = threadIdx.x; e < L * kSplit; e += kVThreads) {
        const int j = e / kSplit, sidx = e % kSplit;
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
        int u = 0;
        for (unsigned b = sidx; b < nb; b += kSplit, u = (u + 1) & 7) acc[u] += __ldcg(tp + (size_t)b * L + j);
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < 8; ++v) s += acc[v];
        scratch[sidx * 256 + j] = s;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < L; j += kVThreads) {
        double s = 0.0;
        for (int sidx = 0; sidx < kSplit; ++sidx) s += scratch[sidx * 256 + j];
        tloc[j] = s * scale;
    }
    __syncthreads();
}

// Per-warp partials (registers) -> block partial (fixed warp order) -> tp[blockIdx] and
// part[blockIdx] (the |.|^2 slot).
__device__ __forceinline__ void block_partials(double (&tn)[kMaxQ], double ns, int L, double (*wpart)[257],
                                               double* tp, double* part) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q)
        if (lane + 32 * q < L) wpart[wib][lane + 32 * q] = tn[q];
    if (lane == 0) wpart[wib][256] = ns;
    __syncthreads();
    for (int j = threadIdx.x; j <= 256; j += kVThreads) {
        if (j < L || j == 256) {
            double s = 0.0;
            for (int w = 0; w < kVWarps; ++w) s += wpart[w][j];
            if (j < L) tp[(size_t)blockIdx.x * L + j] = s;
            else part[blockIdx.x] = s;
        }
    }
}

// Sum of four per-lane partials across the warp in 6 shuffles (transposed butterfly):
// afterwards lanes 8u .. 8u+7 hold the total of partial u.
__device__ __forceinline__ double warp_sum4(const double (&v)[4]) {
    const int lane = threadIdx.x & 31;
    const bool h16 = lane & 16, h8 = lane & 8;
    double a0 = h16 ? v[2] : v[0], a1 = h16 ? v[3] : v[1];
    a0 += __shfl_xor_sync(0xffffffffu, h16 ? v[0] : v[2], 16);
    a1 += __shfl_xor_sync(0xffffffffu, h16 ? v[1] : v[3], 16);
    double c = h8 ? a1 : a0;
    c += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
    c += __shfl_xor_sync(0xffffffffu, c, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;
}

// CL = true: the grid is ONE thread-block cluster (8 or 16 CTAs) and the step barriers are
// hardware cluster barriers (release/acquire at cluster scope, covering the global-memory
// exchanges) instead of the software grid barrier. A cluster is scheduled atomically, so
// verifications of different flushes can run concurrently without the co-residency hazard
// of two spinning grids.
template <int Q, bool CL>
__global__ void __launch_bounds__(kVThreads) verify_kernel(VerifyArgs a) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char vsm[];
    __shared__ double sh[8];
    __shared__ double tloc[256];             // current t = B' x
    __shared__ double wpart[kVWarps][257];   // per-warp partials of the next t, and |.|^2
    const unsigned nb = gridDim.x;
    const GridBar bar{a.bar, a.bar + 1};
    auto step_sync = [&]() {
        if constexpr (CL) cluster_barrier();
        else grid_sync(bar, nb);
    };
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int L = a.ell;
    // Cost-balanced contiguous ranges (every step waits for the slowest block at each grid
    // barrier): rows by 4 nnz + 4 per row, columns by the per-flush cost prefix a.ccost
    // (long columns count their pieces, not their entries: B0 sums those over the grid).
    __shared__ int64_t s_rng[6];
    if (threadIdx.x == 0) {
        const int64_t tr = 4 * (int64_t)a.row_ptr[a.m] + 4 * a.m;
        auto rfind = [&](int64_t target) {
            int64_t lo = 0, hi = a.m;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (4 * (int64_t)a.row_ptr[mid] + 4 * mid < target) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
        s_rng[0] = rfind(tr * blockIdx.x / nb);
        s_rng[1] = blockIdx.x + 1 == nb ? a.m : rfind(tr * (blockIdx.x + 1) / nb);
        if (a.ccost) {
            const int64_t tc = a.ccost[a.d];
            auto cfind = [&](int64_t target) {
                int64_t lo = 0, hi = a.d;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (a.ccost[mid] < target) lo = mid + 1;
                    else hi = mid;
                }
                return lo;
            };
            s_rng[2] = cfind(tc * blockIdx.x / nb);
            s_rng[3] = blockIdx.x + 1 == nb ? a.d : cfind(tc * (blockIdx.x + 1) / nb);
        } else {
            const int64_t cper = (a.d + nb - 1) / nb;
            s_rng[2] = min((int64_t)a.d, (int64_t)blockIdx.x * cper);
            s_rng[3] = min((int64_t)a.d, s_rng[2] + cper);
        }
        // this block's long columns: a contiguous range of the ascending long-column list
        int64_t lo = 0, hi = 0;
        if (a.has_long) {
            const int nl = a.counts[0];
            auto lfind = [&](int64_t c) {
                int l = 0, h = nl;
                while (l < h) {
                    const int mid = (l + h) >> 1;
                    if (a.long_cols[mid] < c) l = mid + 1;
                    else h = mid;
                }
                return (int64_t)l;
            };
            lo = lfind(s_rng[2]);
            hi = lfind(s_rng[3]);
        }
        s_rng[4] = lo;
        s_rng[5] = hi;
    }
    __syncthreads();
    const int64_t r0 = s_rng[0], r1 = s_rng[1], c0 = s_rng[2], c1 = s_rng[3];
    const int64_t lc0 = s_rng[4], lc1 = s_rng[5];
    // The block's slices of A' (CSR rows r0..r1, CSC columns c0..c1) do not change across
    // the power-method steps: stage them in shared memory when they fit, so each step pays
    // one dependent round trip (the x / u gather) instead of three.
    const int nr = (int)max((int64_t)0, r1 - r0), nc = (int)max((int64_t)0, c1 - c0);
    const int rbase = nr > 0 ? a.row_ptr[r0] : 0, knr = nr > 0 ? a.row_ptr[r1] - rbase : 0;
    const int cbase = nc > 0 ? a.col_ptr[c0] : 0, knc = nc > 0 ? a.col_ptr[c1] - cbase : 0;
    const size_t need = 12 * ((size_t)knr + knc) + 4 * ((size_t)nr + nc + 2);
    const bool staged = need <= (size_t)a.stage_bytes;
    const int *RP = a.row_ptr + r0, *CP = a.col_ptr + c0, *RI = a.row_idx + cbase;
    const uint32_t* CI = a.col + rbase;
    const double *RV = a.val + rbase, *CV = a.cval + cbase;
    int rsub = rbase, csub = cbase;
    // Resident: the block's B'^T rows (nc x L, 8 nc L bytes) stay in shared memory, so the
    // per-step stream of B'^T (the bulk of a step's bytes) comes from SMEM instead of L2.
    const size_t need_csr = (need + 15) & ~(size_t)15;
    const bool resident = a.resident && staged && need_csr + 8 * (size_t)nc * L <= (size_t)a.stage_bytes;
    const double* BT = a.bt;
    int64_t ldbt = a.ldb, bt0 = 0;  // row c of B'^T at BT + (c - bt0) * ldbt
    if (resident) {
        double* s_b = reinterpret_cast<double*>(vsm + need_csr);
        for (int e = threadIdx.x; e < nc * L; e += kVThreads) {
            const int c = e / L, j = e - c * L;
            s_b[e] = a.bt[(c0 + c) * a.ldb + j];
        }
        BT = s_b;
        ldbt = L;
        bt0 = c0;
    }
    if (staged) {
        double* s_rv = reinterpret_cast<double*>(vsm);
        double* s_cv = s_rv + knr;
        uint32_t* s_ci = reinterpret_cast<uint32_t*>(s_cv + knc);
        int* s_ri = reinterpret_cast<int*>(s_ci + knr);
        int* s_rp = s_ri + knc;
        int* s_cp = s_rp + nr + 1;
        for (int i = threadIdx.x; i < knr; i += kVThreads) {
            s_rv[i] = RV[i];
            s_ci[i] = CI[i];
        }
        for (int i = threadIdx.x; i < knc; i += kVThreads) {
            s_cv[i] = CV[i];
            s_ri[i] = RI[i];
        }
        for (int i = threadIdx.x; i <= nr; i += kVThreads) s_rp[i] = RP[i] - rbase;
        for (int i = threadIdx.x; i <= nc; i += kVThreads) s_cp[i] = CP[i] - cbase;
        RP = s_rp;
        CP = s_cp;
        RI = s_ri;
        CI = s_ci;
        RV = s_rv;
        CV = s_cv;
        rsub = csub = 0;
        __syncthreads();
    }

    // ---- init: |x0|^2 (la_core.cpp:177-186) and the partials of B' x0 over own columns
    {
        double tn[kMaxQ];
#pragma unroll
        for (int q = 0; q < kMaxQ; ++q) tn[q] = 0.0;
        double ns = 0.0;
        for (int64_t c = c0 + wib; c < c1; c += kVWarps) {
            const double xc = a.x0[c];
            ns = fma(xc, xc, ns);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int j = lane + 32 * q;
                if (j < L) tn[q] = fma(BT[(c - bt0) * ldbt + j], xc, tn[q]);
            }
        }
        block_partials(tn, ns, L, wpart, a.tpart, a.part);
    }
    step_sync();
    const double nsq0 = grid_total(a.part, nb, sh);
    if (!(nsq0 > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            atomicOr(a.err, ERR_RNG_U1_ZERO);  // all-zero draw: would need a redraw
            a.out[0] = 0.0;
        }
        return;
    }
    double xscale = 1.0 / sqrt(nsq0);
    reduce_t(a.tpart, nb, L, xscale, tloc, &wpart[0][0]);  // t = B' x0 / |x0|
    const double* xsrc = a.x0;
    double log_mag = 0.0;
    int verdict = -1;  // -1 running, 0 reject, 1 accept
    int step = 0;
    for (; step < a.steps; ++step) {
        double* y = a.ybuf + (size_t)(step & 1) * a.d;
        double* tp = a.tpart + (size_t)((step + 1) & 1) * nb * L;  // partials of the next t
        // ---- phase A: u = A' x over this block's rows, four rows per warp in flight
        for (int64_t rb = r0 + wib; rb < r1; rb += 4 * kVWarps) {
            int k0[4], k1[4];
            int len = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t r = rb + q * kVWarps;
                k0[q] = r < r1 ? RP[r - r0] - rsub : 0;
                k1[q] = r < r1 ? RP[r - r0 + 1] - rsub : 0;
                len = max(len, k1[q] - k0[q]);
            }
            double sp[4] = {0.0, 0.0, 0.0, 0.0};
            for (int off = lane; off < len; off += 64) {  // two gathers per row and lane in flight
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = k0[q] + off;
                    double v0 = 0.0, v1 = 0.0;
                    if (k < k1[q]) v0 = RV[k] * __ldcg(xsrc + CI[k]);
                    if (k + 32 < k1[q]) v1 = RV[k + 32] * __ldcg(xsrc + CI[k + 32]);
                    sp[q] = fma(v0 + v1, xscale, sp[q]);
                }
            }
            const double tot = warp_sum4(sp);
            const int q = lane >> 3;
            const int64_t r = rb + q * kVWarps;
            if ((lane & 7) == 0 && r < r1) a.u[r] = tot;
        }
        step_sync();
        // ---- phase B0 (skewed columns only): pieces of the long columns over the whole grid
        if (a.has_long) {
            const int np = a.counts[1];
            const int gw = blockIdx.x * kVWarps + wib, tw = nb * kVWarps;
            for (int p = gw; p < np; p += tw) {
                const int kb = a.piece_beg[p], ke = a.piece_end[p];
                double sp[4] = {0.0, 0.0, 0.0, 0.0};  // four gathers per lane in flight
                for (int k = kb + lane; k < ke; k += 128) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (k + 32 * u < ke) sp[u] = fma(a.cval[k + 32 * u], __ldcg(a.u + a.row_idx[k + 32 * u]), sp[u]);
                }
                const double t = warp_sum((sp[0] + sp[1]) + (sp[2] + sp[3]));
                if (lane == 0) a.lpart[p] = t;
            }
            step_sync();
        }
        // ---- phase B: y over own columns (four per warp in flight); next-t partials and
        // |y|^2 from the same B'^T rows
        double tl[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) tl[q] = (lane + 32 * q < L) ? tloc[lane + 32 * q] : 0.0;
        double tn[kMaxQ];
#pragma unroll
        for (int q = 0; q < kMaxQ; ++q) tn[q] = 0.0;
        double nsq = 0.0;
        bool bad = false;
        for (int64_t cb = c0 + wib; cb < c1; cb += 4 * kVWarps) {
            int k0[4], k1[4];
            bool own[4];
            int len = 0;
            double lsum[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t c = cb + q * kVWarps;
                k0[q] = c < c1 ? CP[c - c0] - csub : 0;
                k1[q] = c < c1 ? CP[c - c0 + 1] - csub : 0;
                own[q] = c < c1;
                if (a.has_long && k1[q] - k0[q] > 2 * a.piece) {  // long: the loop below
                    k1[q] = k0[q];
                    own[q] = false;
                }
                len = max(len, k1[q] - k0[q]);
            }
            double brow[4][Q];
            double dp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t c = cb + q * kVWarps;
                dp[q] = lsum[q];
#pragma unroll
                for (int w = 0; w < Q; ++w) {
                    const int j = lane + 32 * w;
                    brow[q][w] = (own[q] && j < L) ? BT[(c - bt0) * ldbt + j] : 0.0;
                    dp[q] = fma(-brow[q][w], tl[w], dp[q]);  // - (B'^T t)_c partial
                }
            }
            for (int off = lane; off < len; off += 64) {  // two gathers per column and lane in flight
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = k0[q] + off;
                    double v0 = 0.0, v1 = 0.0;
                    if (k < k1[q]) v0 = CV[k] * __ldcg(a.u + RI[k]);
                    if (k + 32 < k1[q]) v1 = CV[k + 32] * __ldcg(a.u + RI[k + 32]);
                    dp[q] += v0 + v1;
                }
            }
            const double tot = warp_sum4(dp);  // (A'^T u - B'^T t)_c on lanes 8q..8q+7
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t c = cb + q * kVWarps;
                const double yc = a.scale * __shfl_sync(0xffffffffu, tot, 8 * q);  // shrink.cpp:124
                if (own[q]) {
                    if (!isfinite(yc)) bad = true;
                    if (lane == 0) y[c] = yc;
                    nsq = fma(yc, yc, nsq);
#pragma unroll
                    for (int w = 0; w < Q; ++w) tn[w] = fma(brow[q][w], yc, tn[w]);
                }
            }
        }
        // long columns of this block: warp per column, its B0 piece partials summed by lanes
        if (a.has_long) {
            const int nl = a.counts[0], npc = a.counts[1];
            for (int64_t li = lc0 + wib; li < lc1; li += kVWarps) {
                const int64_t c = a.long_cols[li];
                const int first = a.long_first[li], last = li + 1 < nl ? a.long_first[li + 1] : npc;
                double dpv = 0.0;
                for (int p = first + lane; p < last; p += 32) dpv += __ldcg(a.lpart + p);
                double brow[Q];
#pragma unroll
                for (int w = 0; w < Q; ++w) {
                    const int j = lane + 32 * w;
                    brow[w] = j < L ? BT[(c - bt0) * ldbt + j] : 0.0;
                    dpv = fma(-brow[w], tl[w], dpv);
                }
                const double yc = a.scale * warp_sum(dpv);
                if (!isfinite(yc)) bad = true;
                if (lane == 0) y[c] = yc;
                nsq = fma(yc, yc, nsq);
#pragma unroll
                for (int w = 0; w < Q; ++w) tn[w] = fma(brow[w], yc, tn[w]);
            }
        }
        if (bad) atomicOr(a.err, ERR_NONFINITE_VERIFY);
        block_partials(tn, nsq, L, wpart, tp, a.part);
        step_sync();
        // ---- phase C: identical decision in every block (shrink.cpp:88-99)
        const double tot = grid_total(a.part, nb, sh);
        if (*((volatile int*)a.err) & ERR_NONFINITE_VERIFY) {
            verdict = 0;
            break;
        }
        if (tot == 0.0) {
            verdict = 1;
            break;
        }
        const double nrm = sqrt(tot);
        log_mag += log(nrm);
        if (log_mag > 0.0 && nrm >= 1.0) {
            verdict = 0;
            ++step;
            break;
        }
        xsrc = y;
        xscale = 1.0 / nrm;
        reduce_t(tp, nb, L, xscale, tloc, &wpart[0][0]);
    }
    if (verdict < 0) verdict = log_mag <= 0.0 ? 1 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out[0] = (double)verdict;
        a.out[1] = log_mag;
        a.out[2] = (double)step;
    }
}


// ---- the verifier as a kernel sequence (no persistent grid) -----------------------------
// One power step = three kernels: vg_rows (the decision on the previous pass, the next t = B' x,
// and u = A' x over every row, all SMs), vg_colsum (w = A'^T u over every column), vg_cols (y
// over every column from w and the streamed B'^T rows, the partials of the next t and of |y|^2
// per block). Kernel
// boundaries replace the grid barriers, so nothing spins and verifications of different
// flushes overlap freely (no serialisation); the whole sequence for a given step count is
// captured once as a CUDA graph. Per column / row the arithmetic is the persistent kernel's
// (same lane order, same warp reductions); only the grouping of the block partials differs.
// After a decision every later kernel returns at once (state->done).
struct VState {
    double scale, log_mag, xscale;
    int done, verdict, step, steps;
    double lm[2];  // log magnitude after pass k at lm[k & 1] (pass -1: 0)
};

constexpr int kGRowsThreads = 256;
constexpr int kGColsThreads = 512;
constexpr int kGColsWarps = kGColsThreads / 32;

__global__ void vg_setup_kernel(VState* st, double scale, int steps) {
    pdl_entry();
    st->scale = scale;
    st->log_mag = 0.0;
    st->xscale = 0.0;
    st->done = 0;
    st->verdict = -1;
    st->step = 0;
    st->steps = steps;
    st->lm[0] = st->lm[1] = 0.0;
}

// The accept / reject / continue decision after pass s - 1 (s = 0: after the x0 pass), from the
// per-block |.|^2 partials of that pass (shrink.cpp:88-99 / la_core.cpp:177-186). Run by warp 0
// of every block of a launch: each sums the partials in the same fixed order, so all blocks take
// the same decision without a grid barrier; block 0 commits it to the state. Returns 1 to
// continue, with the scale of the next x in *xs.
__device__ int vg_decide(const VerifyArgs& a, VState* st, int s, int nblk, double* xs) {
    const int lane = threadIdx.x & 31;
    if (*((volatile int*)&st->done)) return 0;
    double tot = 0.0;
    for (int b = lane; b < nblk; b += 32) tot += __ldcg(a.part + b);
    tot = warp_sum(tot);
    const bool commit = blockIdx.x == 0 && lane == 0;
    if (s == 0) {
        if (!(tot > 0.0)) {
            if (commit) {
                atomicOr(a.err, ERR_RNG_U1_ZERO);  // all-zero draw: would need a redraw
                st->done = 1;
                st->verdict = 0;
            }
            return 0;
        }
        *xs = 1.0 / sqrt(tot);
        return 1;
    }
    if (*((volatile int*)a.err) & ERR_NONFINITE_VERIFY) {
        if (commit) {
            st->verdict = 0;
            st->done = 1;
        }
        return 0;
    }
    if (tot == 0.0) {  // iterate annihilated (shrink.cpp:92)
        if (commit) {
            st->verdict = 1;
            st->done = 1;
        }
        return 0;
    }
    const double nrm = sqrt(tot);
    const double lm = st->lm[s & 1] + log(nrm);
    if (commit) {
        st->lm[(s - 1) & 1] = lm;
        st->log_mag = lm;
        st->step = s;
    }
    if (lm > 0.0 && nrm >= 1.0) {
        if (commit) {
            st->verdict = 0;
            st->done = 1;
        }
        return 0;
    }
    *xs = 1.0 / nrm;
    return 1;
}

// Lane-strided sum of part[first], part[first + step], ... (< last) with eight loads per lane in flight (a column of
// thousands of pieces -- c5's most frequent item has 13 700 -- is summed by one warp: a dependent
// load per iteration made that a 300 us tail). Fixed order: deterministic.
__device__ __forceinline__ double lane_strided_sum(const double* part, int first, int last, int step, int lane) {
    double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int64_t st = 32 * (int64_t)step;
    int64_t q = first + (int64_t)lane * step;
    for (; q + 7 * st < last; q += 8 * st) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + q + u * st);
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] += v[u];
    }
    for (; q < last; q += st) s[0] += __ldcg(part + q);
    return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// Step `step`: the decision after the previous pass (vg_decide, warp 0 of every block), t = B' x
// for this pass from the previous pass's block partials (entry j by warp j % 8 of block j / 8),
// and u = A' y_prev UNSCALED (x = y_prev / |y_prev|: the consumers apply the 1 / |y_prev| that
// the decision produces, so the row work does not wait for it): long-row pieces first (warp per
// piece, the last piece of a row sums them in piece order), then the short rows longest first,
// sixteen lanes per row with four entries each in flight. The x gathers go through L1
// (ld.global.nc): x is read-only for the launch and L1 starts every launch invalid, so this is
// safe in the kernel sequence (not in the persistent kernel); tools/spmv_lab.cu on the c4 flush:
// 8 lanes L2-only 32.8 us, 16 lanes through L1 14.4 us.
template <int G>
__global__ void __launch_bounds__(kGRowsThreads) vg_rows_kernel(VerifyArgs a, VState* st, int step, int nblk) {
    pdl_entry();
    __shared__ double s_xs;
    __shared__ int s_go;
    if (*((volatile int*)&st->done)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int L = a.ell;
    const bool t_block = blockIdx.x * (kGRowsThreads / 32) < L;
    if (threadIdx.x < 32) {
        double xs = 0.0;
        const int go = vg_decide(a, st, step, nblk, &xs);
        if (threadIdx.x == 0) {
            s_go = go;
            s_xs = xs;
            if (blockIdx.x == 0 && go) st->xscale = xs;
        }
    }
    if (t_block) {
        __syncthreads();
        if (!s_go) return;
        const int j = blockIdx.x * (kGRowsThreads / 32) + wib;
        if (j < L) {
            double sacc = 0.0;
            for (int b = lane; b < nblk; b += 32) sacc += __ldcg(a.tpart + (size_t)b * L + j);
            sacc = warp_sum(sacc);
            if (lane == 0) a.t[j] = sacc * s_xs;
        }
    }
    const double* x = step == 0 ? a.x0 : a.ybuf + (size_t)((step - 1) & 1) * a.d;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int np = 0, ns = (int)a.m;
    if (a.r_counts) {
        np = a.r_counts[1];
        ns = a.r_counts[2];
    }
    for (int64_t p = gw; p < np; p += nw) {
        const int kb = a.r_piece_beg[p], ke = a.r_piece_end[p];
        double sp[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = kb + lane; k < ke; k += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + 32 * u < ke) sp[u] = fma(a.val[k + 32 * u], __ldg(x + a.col[k + 32 * u]), sp[u]);
        }
        const double t = warp_sum((sp[0] + sp[1]) + (sp[2] + sp[3]));
        if (lane == 0) a.r_part[p] = t;
        __threadfence();
        const int li = a.r_piece_li[p];
        const int nl = a.r_counts[0];
        const int first = a.r_long_first[li], last = li + 1 < nl ? a.r_long_first[li + 1] : np;
        int old = 0;
        if (lane == 0) old = atomicAdd(a.r_arrive + li, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == last - first - 1) {  // every piece of this row is written: sum them in order
            __threadfence();
            // the whole warp sums the row's pieces: lane-strided, then a fixed shuffle tree
            double tot = 0.0;
            for (int q = first + lane; q < last; q += 32) tot += __ldcg(a.r_part + q);
            tot = warp_sum(tot);
            if (lane == 0) {
                a.u[a.r_long_rows[li]] = tot;
                a.r_arrive[li] = 0;  // ready for the next launch
            }
        }
    }
    // G lanes per row (32 / G rows per warp in flight), four entries per lane in flight
    const int sub = lane & (G - 1);
    const int64_t g0 = gw * (32 / G) + lane / G, ng = nw * (32 / G);
    for (int64_t gi = g0; gi < ns; gi += ng) {
        const int r = a.r_counts ? a.r_order[gi] : (int)gi;
        const int kb = a.row_ptr[r], ke = a.row_ptr[r + 1];
        double sp[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = kb + sub; k < ke; k += 4 * G) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + G * u < ke) sp[u] = fma(a.val[k + G * u], __ldg(x + a.col[k + G * u]), sp[u]);
        }
        double t = (sp[0] + sp[1]) + (sp[2] + sp[3]);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (sub == 0) a.u[r] = t;
    }
}

// w = A'^T u (unscaled) for every column: pieces of the long columns first (warp per piece, the
// last piece of a column sums them in piece order), then the short columns longest first, sixteen
// lanes per column with four entries each in flight; u through L1 (read-only in this launch).
// Each w_c is a per-column sum in a fixed order, so which warp computes it does not matter.
template <int G>
__global__ void __launch_bounds__(kGRowsThreads) vg_colsum_kernel(VerifyArgs a, const VState* __restrict__ st) {
    pdl_entry();
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int np = a.has_long ? a.counts[1] : 0;
    const int ns = a.c_order ? a.counts[2] : (int)a.d;
    // A long column's pieces in runs of vrun consecutive pieces (about 512 entries) per warp: the
    // SpMM's pieces may be as short as 64 entries (panels larger than L2), and a scalar gather per
    // entry does not pay a partial, a fence and an arrival per such piece (c5: 568 -> 290 us).
    const int vrun = max(1, 512 / max(a.piece, 1));
    for (int64_t p = gw; p < np; p += nw) {
        const int li = a.c_piece_li[p];
        const int nl = a.counts[0];
        const int first = a.long_first[li], last = li + 1 < nl ? a.long_first[li + 1] : np;
        if ((p - first) % vrun != 0) continue;  // not the head of a run
        const int pend = min((int)p + vrun, last);
        const int kb = a.piece_beg[p], ke = a.piece_end[pend - 1];
        double sp[4] = {0.0, 0.0, 0.0, 0.0};  // four gathers per lane in flight
        for (int k = kb + lane; k < ke; k += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + 32 * u < ke) sp[u] = fma(a.cval[k + 32 * u], __ldg(a.u + a.row_idx[k + 32 * u]), sp[u]);
        }
        const double t = warp_sum((sp[0] + sp[1]) + (sp[2] + sp[3]));
        if (lane == 0) a.lpart[p] = t;
        __threadfence();
        int old = 0;
        if (lane == 0) old = atomicAdd(a.c_arrive + li, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == (last - first + vrun - 1) / vrun - 1) {  // every run of this column is written: sum them in order
            __threadfence();
            const double tot = warp_sum(lane_strided_sum(a.lpart, first, last, vrun, lane));
            if (lane == 0) {
                a.w[a.long_cols[li]] = tot;
                a.c_arrive[li] = 0;  // ready for the next launch
            }
        }
    }
    const int sub = lane & (G - 1);
    const int64_t g0 = gw * (32 / G) + lane / G, ng = nw * (32 / G);
    for (int64_t gi = g0; gi < ns; gi += ng) {
        const int c = a.c_order ? a.c_order[gi] : (int)gi;
        const int kb = a.col_ptr[c], ke = a.col_ptr[c + 1];
        double sp[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = kb + sub; k < ke; k += 4 * G) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + G * u < ke) sp[u] = fma(a.cval[k + G * u], __ldg(a.u + a.row_idx[k + G * u]), sp[u]);
        }
        double t = (sp[0] + sp[1]) + (sp[2] + sp[3]);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (sub == 0) a.w[c] = t;
    }
}

// columns: y_c = scale (xscale w_c - B'^T_c t) with the B'^T rows streamed once, and from the
// same rows the block partials of the next t = B' y and of |y|^2 (init = true: the x0 pass --
// |x0|^2 and B' x0 partials, no y). Every column costs one B'^T row, so equal contiguous column
// ranges per block and a fixed warp interleave inside it (the partials' order is fixed).
// Q > 8 (256 < ell <= 512): 256 threads and two columns in flight per warp keep the B'^T
// rows, t and the partials in registers (2 x 16 + 2 x 16 doubles) and the static shared memory
// under 48 KB.
template <int Q>
__host__ __device__ constexpr int vg_cols_threads() { return Q > 8 ? 256 : kGColsThreads; }

template <int Q, bool INIT>
__global__ void __launch_bounds__(vg_cols_threads<Q>()) vg_cols_kernel(VerifyArgs a, const VState* __restrict__ st, int step) {
    pdl_entry();
    constexpr int NT = vg_cols_threads<Q>(), NW = NT / 32, QL = 32 * Q;
    constexpr int RF = Q > 8 ? 2 : 4;  // columns in flight per warp
    __shared__ double tloc[QL];
    __shared__ double wpart[NW][QL + 1];
    if (st->done) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int L = a.ell;
    const int64_t cper = (a.d + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = min((int64_t)a.d, (int64_t)blockIdx.x * cper), c1 = min((int64_t)a.d, c0 + cper);
    double* y = a.ybuf + (size_t)(step & 1) * a.d;
    const double xscale = INIT ? 1.0 : st->xscale;  // w = A'^T A' y_prev is unscaled
    if (!INIT)
        for (int j = threadIdx.x; j < L; j += NT) tloc[j] = __ldcg(a.t + j);
    __syncthreads();
    double tl[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) tl[q] = (!INIT && lane + 32 * q < L) ? tloc[lane + 32 * q] : 0.0;
    double tn[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) tn[q] = 0.0;
    double nsq = 0.0;
    bool bad = false;
    const double scale = st->scale;
    for (int64_t cb = c0 + wib; cb < c1; cb += RF * NW) {
        double brow[RF][Q];
        double wc[RF];
#pragma unroll
        for (int q = 0; q < RF; ++q) {
            const int64_t c = cb + q * NW;
            const bool own = c < c1;
            wc[q] = own ? (INIT ? a.x0[c] : __ldcg(a.w + c)) : 0.0;
#pragma unroll
            for (int w = 0; w < Q; ++w) {
                const int j = lane + 32 * w;
                brow[q][w] = (own && j < L) ? a.bt[c * a.ldb + j] : 0.0;
            }
        }
        if constexpr (INIT) {
#pragma unroll
            for (int q = 0; q < RF; ++q) {
                nsq = fma(wc[q], wc[q], nsq);
#pragma unroll
                for (int w = 0; w < Q; ++w) tn[w] = fma(brow[q][w], wc[q], tn[w]);
            }
        } else {
            double dp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < RF; ++q) {
#pragma unroll
            for (int w = 0; w < Q; ++w) dp[q] = fma(-brow[q][w], tl[w], dp[q]);
        }
        const double tot = warp_sum4(dp);  // -(B'^T t)_c on lanes 8q .. 8q+7
#pragma unroll
        for (int q = 0; q < RF; ++q) {
            const int64_t c = cb + q * NW;
            const double yc = scale * fma(wc[q], xscale, __shfl_sync(0xffffffffu, tot, 8 * q));  // shrink.cpp:124
            if (c < c1) {
                if (!isfinite(yc)) bad = true;
                if (lane == 0) y[c] = yc;
                nsq = fma(yc, yc, nsq);
#pragma unroll
                for (int w = 0; w < Q; ++w) tn[w] = fma(brow[q][w], yc, tn[w]);
            }
        }
        }
    }
    if (bad) atomicOr(a.err, ERR_NONFINITE_VERIFY);
    // block partials (fixed warp order) -> tpart[block], part[block]
#pragma unroll
    for (int q = 0; q < Q; ++q)
        if (lane + 32 * q < L) wpart[wib][lane + 32 * q] = tn[q];
    if (lane == 0) wpart[wib][QL] = nsq;
    __syncthreads();
    for (int j = threadIdx.x; j <= QL; j += NT) {
        if (j < L || j == QL) {
            double sacc = 0.0;
            for (int w = 0; w < NW; ++w) sacc += wpart[w][j];
            if (j < L) a.tpart[(size_t)blockIdx.x * L + j] = sacc;
            else a.part[blockIdx.x] = sacc;
        }
    }
}

// after the last pass: its decision, then the verdict (shrink.cpp:101)
__global__ void vg_final_kernel(VerifyArgs a, VState* st, int nblk) {
    pdl_entry();
    if (threadIdx.x < 32) {
        double xs = 0.0;
        vg_decide(a, st, st->steps, nblk, &xs);
        if (threadIdx.x == 0) {
            __threadfence_block();
            const int verdict = st->verdict >= 0 ? st->verdict : (st->log_mag <= 0.0 ? 1 : 0);
            a.out[0] = (double)verdict;
            a.out[1] = st->log_mag;
            a.out[2] = (double)st->step;
        }
    }
}

typedef void (*VgColsFn)(VerifyArgs, const VState*, int);
template <bool INIT>
VgColsFn vg_cols_fn(int ell) {
    switch ((ell + 31) / 32) {
        case 1: return vg_cols_kernel<1, INIT>;
        case 2: return vg_cols_kernel<2, INIT>;
        case 3: return vg_cols_kernel<3, INIT>;
        case 4: return vg_cols_kernel<4, INIT>;
        case 5: return vg_cols_kernel<5, INIT>;
        case 6: return vg_cols_kernel<6, INIT>;
        case 7: return vg_cols_kernel<7, INIT>;
        case 8: return vg_cols_kernel<8, INIT>;
        case 9: case 10: return vg_cols_kernel<10, INIT>;
        case 11: case 12: return vg_cols_kernel<12, INIT>;
        case 13: case 14: return vg_cols_kernel<14, INIT>;
        default: return vg_cols_kernel<16, INIT>;
    }
}
unsigned vg_cols_nthreads(int ell) { return (ell + 31) / 32 > 8 ? 256u : (unsigned)kGColsThreads; }

typedef void (*VerifyFn)(VerifyArgs);
template <bool CL>
VerifyFn verify_fn_t(int ell) {
    switch ((ell + 31) / 32) {
        case 1: return verify_kernel<1, CL>;
        case 2: return verify_kernel<2, CL>;
        case 3: return verify_kernel<3, CL>;
        case 4: return verify_kernel<4, CL>;
        case 5: return verify_kernel<5, CL>;
        case 6: return verify_kernel<6, CL>;
        case 7: return verify_kernel<7, CL>;
        default: return verify_kernel<8, CL>;
    }
}

// Per-column cost for the cost-balanced column ranges: a CSC entry is a stream read plus a
// dependent gather (4), a long column (> 2 piece entries, summed over the grid in B0) costs
// its pieces, and every column streams its B'^T row (ell / 8).
__global__ void vcost_kernel(const int* __restrict__ col_ptr, int64_t d, int ell, int piece,
                             int64_t* __restrict__ cost) {
    pdl_entry();
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < d; c += (int64_t)gridDim.x * blockDim.x) {
        const int len = col_ptr[c + 1] - col_ptr[c];
        const int eff = len > 2 * piece ? (len + piece - 1) / piece : len;
        cost[c] = 4 * (int64_t)eff + ell / 8 + 4;
    }
}

}  // namespace

void verify_column_costs(const int* d_col_ptr, int64_t d, int ell, int piece, int64_t* d_prefix, Scratch& scr,
                         cudaStream_t st) {
    int64_t* cost = scr.take<int64_t>(d + 1);
    LAUNCH(vcost_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)d, 256))), 256, 0, st, d_col_ptr, d, ell,
           piece, cost);
    CK(cudaMemsetAsync(cost + d, 0, sizeof(int64_t), st));
    exclusive_scan(cost, d_prefix, d + 1, scr, st);
}

int verify_grid_blocks(int device, int64_t d, int lp) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // Each step streams B'^T (8 d lp bytes) once over the grid. Small B' (c2: 8 MB): the power
    // method is latency bound (two grid barriers per step), so 32 blocks -- with several
    // flushes in flight the other SMs keep running SpMM / orthonormalisation (measured on c2:
    // 146 blocks 322, 74 blocks 199, 32 blocks 182 ms per stream). Large B' (c3-c5: 0.16-2 GB
    // per step) is bandwidth bound per SM: one block per 512 KB of B', up to every SM.
    const int64_t by_size = (8 * d * (int64_t)lp) / (512 * 1024);
    // past the small-B' regime every SM: the cost-balanced ranges keep the blocks even
    int nb = by_size > 32 ? sms : 32;
    if (const char* e = std::getenv("SFDG_VERIFY_BLOCKS")) nb = std::max(1, std::min(sms, std::atoi(e)));
    return nb;
}

namespace {
int stage_bytes_for(int device) {
    // the kernel's static shared memory and the device opt-in limit; one value per device
    static std::mutex mu;
    static std::map<int, int> cached;
    std::lock_guard<std::mutex> g(mu);
    auto it = cached.find(device);
    if (it != cached.end()) return it->second;
    cudaFuncAttributes attr;
    CK(cudaFuncGetAttributes(&attr, (const void*)verify_kernel<8, false>));
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    const int v = optin - (int)attr.sharedSizeBytes - 1024;
    cached[device] = v;
    return v;
}
}  // namespace

// Opt-in (SFDG_VERIFY_RESIDENT=1). Measured on c2 (SFDG_TRACE of the timed step, 1 B200): a
// resident verification takes 1233 us against 1687 us streaming (57 blocks against 32), but
// the extra SMs it holds stretch the lanes' shrink phase 5023 -> 5271 us, and the stream
// gets slower overall (170.0 against 166.0 ms); c3-c5 B'^T does not fit at all.
int verify_resident_blocks(int device, int64_t m, int64_t d, int ell, int64_t nnz, int min_blocks) {
    const char* e = std::getenv("SFDG_VERIFY_RESIDENT");
    if (!e || std::atoi(e) == 0) return 0;
    if (std::getenv("SFDG_VERIFY_BLOCKS")) return 0;  // explicit grid: streaming kernel
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const double stage = (double)stage_bytes_for(device);
    for (int nb = std::max(1, min_blocks); nb <= sms; ++nb) {
        // per block: CSR + CSC slices (12 B per entry each, +25% for uneven rows / columns),
        // their offsets, and the B'^T rows of its columns
        const double rows = std::ceil((double)m / nb), cols = std::ceil((double)d / nb);
        const double need = 1.25 * 24.0 * (double)nnz / nb + 4.0 * (rows + cols + 2) + 16 + 8.0 * cols * ell;
        if (need <= stage) return nb;
    }
    return 0;
}

int verify_cluster_size(int64_t d, int lp) {
    // Opt-in (SFDG_VERIFY_CLUSTER=8|16): one cluster per verification, so the flushes in
    // flight verify concurrently (hardware barriers, no co-residency hazard). Measured on c2
    // (ms per 100-flush stream): grid 165.8, cluster-16 168.2, cluster-8 228.9 -- a 16-CTA
    // cluster streams 512 KB of B'^T per CTA per step and waits for 16 free SMs in a GPC, which
    // cancels the concurrency. Large B' (c3-c5) needs the whole grid's bandwidth anyway.
    (void)d;
    (void)lp;
    int c = 0;
    if (const char* e = std::getenv("SFDG_VERIFY_CLUSTER")) {
        const int v = std::atoi(e);
        c = v >= 16 ? 16 : v >= 8 ? 8 : 0;
    }
    return c;
}

void verify_launch(const VerifyArgs& args_in, int nblocks, int cluster, cudaStream_t st) {
    if (args_in.ell > 32 * kMaxQ) throw invalid_argument("verify: the persistent verifier holds ell <= 256 (wider: kernel sequence)");
    ProfScope prof("verify", st);
    if (first_on_device((const void*)verify_kernel<8, false>)) {
        for (int ell = 32; ell <= 256; ell += 32) {
            allow_max_dynamic_smem(verify_fn_t<false>(ell));
            allow_max_dynamic_smem(verify_fn_t<true>(ell));
            CK(cudaFuncSetAttribute((const void*)verify_fn_t<true>(ell), cudaFuncAttributeNonPortableClusterSizeAllowed,
                                    1));
        }
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    int stage = stage_bytes_for(dev);
    if (const char* e = std::getenv("SFDG_VERIFY_STAGE")) stage = std::atoi(e) ? stage : 0;
    if (cluster == 0 && !args_in.resident && args_in.nnz > 0) {
        // no block's CSR / CSC slices will fit: launch without the dynamic shared memory, so
        // the L1 keeps its full size for the x / u gathers
        const double per_block = 1.25 * 24.0 * (double)args_in.nnz / nblocks + 4.0 * (double)(args_in.m + args_in.d + 2) / nblocks;
        if (per_block > (double)stage) stage = 0;
    }
    VerifyArgs args = args_in;
    args.stage_bytes = stage;
    if (cluster > 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cluster);
        cfg.blockDim = dim3(kVThreads);
        cfg.dynamicSmemBytes = (size_t)stage;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, verify_fn_t<true>(args.ell), args));
    } else {
        CK(cudaMemsetAsync(args.bar, 0, 2 * sizeof(unsigned), st));
        void* params[] = {(void*)&args};
        CK(cudaLaunchCooperativeKernel((const void*)verify_fn_t<false>(args.ell), dim3(nblocks), dim3(kVThreads),
                                       params, (size_t)stage, st));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

int verify_graph_blocks(int device, int64_t d) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    return (int)std::max<int64_t>(1, std::min<int64_t>(2 * sms, (d + 63) / 64));
}

size_t verify_state_bytes() { return sizeof(VState); }

void verify_sequence(const VerifyArgs& a, void* state, int nblk, int sms, cudaStream_t st) {
    VState* s = static_cast<VState*>(state);
    // one wave of the row kernel (six 256-thread blocks per SM), at least one warp per entry of t
    const unsigned rgrid = (unsigned)std::max<int64_t>((a.ell + 7) / 8, std::min<int64_t>(6 * sms, (a.m + 31) / 32));
    const unsigned rgrid2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(6 * sms, (a.d + 31) / 32));
    LAUNCH(vg_cols_fn<true>(a.ell), nblk, vg_cols_nthreads(a.ell), 0, st, a, s, 0);
    // SFDG_VG_LANES=8|16|32: lanes per row / column in the two SpMVs (A/B testing)
    static const int G = std::getenv("SFDG_VG_LANES") ? std::atoi(std::getenv("SFDG_VG_LANES")) : 16;
    auto rows_fn = G == 8 ? vg_rows_kernel<8> : G == 32 ? vg_rows_kernel<32> : vg_rows_kernel<16>;
    auto cols_fn = G == 8 ? vg_colsum_kernel<8> : G == 32 ? vg_colsum_kernel<32> : vg_colsum_kernel<16>;
    for (int step = 0; step < a.steps; ++step) {
        LAUNCH(rows_fn, rgrid, kGRowsThreads, 0, st, a, s, step, nblk);
        LAUNCH(cols_fn, rgrid2, kGRowsThreads, 0, st, a, s);
        LAUNCH(vg_cols_fn<false>(a.ell), nblk, vg_cols_nthreads(a.ell), 0, st, a, s, step);
    }
    LAUNCH(vg_final_kernel, 1, 32, 0, st, a, s, nblk);
}

void verify_setup(void* state, double scale, int steps, cudaStream_t st) {
    LAUNCH(vg_setup_kernel, 1, 1, 0, st, static_cast<VState*>(state), scale, steps);
}

}  // namespace sfdg
