// sparse.cu -- device CSR buffer A' and its products (reference: core/src/sparse.cpp).
//
//  * csc_build: CSR -> CSC by a stable LSD radix sort on the column index (8-bit
//    digits, warp-level match_any ranking). Stability keeps every column's entries in
//    row order, so W = A'^T Y gathers in exactly the order rmatvec / project_rows
//    scatter (sparse.cpp:45-69) and the result is deterministic (no FP atomics).
//  * spmm: out[r, :] = sum_k val[k] * in[idx[k], :] over an ell-wide row-major panel.
//    One warp per output row, lanes across the panel columns (double2 loads). Rows
//    longer than kPiece*2 are split into kPiece-long pieces whose partial rows are
//    summed in piece order by a fix-up kernel (deterministic load balancing for
//    Zipf-skewed columns). Used for Y = A' X (matvec, sparse.cpp:32-43) and
//    W = A'^T Y (rmatvec/project_rows, sparse.cpp:45-69).
#include <algorithm>

#include <mutex>
#include <set>
#include <cstdlib>
#include "common.cuh"
#include "sparse.cuh"

namespace sfdg {

namespace {

constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;  // 4096 elements per block

// ---------------------------------------------------------------- exclusive scan
__global__ void scan_block_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                  int64_t* __restrict__ block_sums) {
    pdl_entry();
    __shared__ int64_t warp_tot[32];
    const int64_t base = (int64_t)blockIdx.x * kScanBlock * kScanItems;
    int64_t v[kScanItems];
    int64_t tsum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + (int64_t)threadIdx.x * kScanItems + i;
        v[i] = idx < n ? in[idx] : 0;
        tsum += v[i];
    }
    // block exclusive scan of tsum
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t t = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    int64_t run = x - tsum + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + (int64_t)threadIdx.x * kScanItems + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
    if (threadIdx.x == kScanBlock - 1 && block_sums) block_sums[blockIdx.x] = run;
}

__global__ void scan_add_kernel(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ block_offs) {
    pdl_entry();
    const int64_t base = (int64_t)blockIdx.x * kScanBlock * kScanItems;
    const int64_t add = block_offs[blockIdx.x];
    for (int i = threadIdx.x; i < kScanBlock * kScanItems; i += kScanBlock) {
        const int64_t idx = base + i;
        if (idx < n) out[idx] += add;
    }
}

// ---------------------------------------------------------------- radix sort
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixItemsPerWarp = 256;  // 8 rounds of 32
constexpr int kRadixTile = kRadixWarps * kRadixItemsPerWarp;

__global__ void radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift, int ntiles,
                                  int64_t* __restrict__ hist /* [256][ntiles] */) {
    pdl_entry();
    __shared__ int cnt[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRadixTile;
    for (int i = threadIdx.x; i < kRadixTile; i += blockDim.x) {
        const int64_t k = base + i;
        if (k < n) atomicAdd(&cnt[(keys[k] >> shift) & 0xff], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[(int64_t)i * ntiles + blockIdx.x] = cnt[i];
}

__global__ void radix_scatter_kernel(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                     uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n,
                                     int shift, int ntiles, const int64_t* __restrict__ offs /* [256][ntiles] */) {
    pdl_entry();
    __shared__ int cnt[kRadixWarps][256];
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t wbase = (int64_t)blockIdx.x * kRadixTile + (int64_t)w * kRadixItemsPerWarp;
    constexpr int R = kRadixItemsPerWarp / 32;
    uint32_t key[R], val[R];
    int dig[R], lpos[R];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t k = wbase + r * 32 + lane;
        const bool ok = k < n;
        key[r] = ok ? keys_in[k] : 0u;
        val[r] = ok ? vals_in[k] : 0u;
        dig[r] = ok ? (int)((key[r] >> shift) & 0xff) : 256;
        const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
        const int rank = __popc(peers & lt);
        const int leader = __ffs(peers) - 1;
        int before = 0;
        if (ok) before = cnt[w][dig[r]];
        __syncwarp();
        if (ok && lane == leader) cnt[w][dig[r]] = before + __popc(peers);
        __syncwarp();
        lpos[r] = before + rank;
    }
    __syncthreads();
    // per digit: exclusive prefix over warps (tile-local offsets)
    for (int dg = threadIdx.x; dg < 256; dg += blockDim.x) {
        int run = 0;
#pragma unroll
        for (int ww = 0; ww < kRadixWarps; ++ww) {
            const int t = cnt[ww][dg];
            cnt[ww][dg] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (dig[r] < 256) {
            const int64_t pos = offs[(int64_t)dig[r] * ntiles + blockIdx.x] + cnt[w][dig[r]] + lpos[r];
            keys_out[pos] = key[r];
            vals_out[pos] = val[r];
        }
    }
}

__global__ void iota_kernel(uint32_t* __restrict__ v, int64_t n) {
    pdl_entry();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

// row id of every stored entry (warp per row)
__global__ void expand_rows_kernel(const int* __restrict__ row_ptr, int m, uint32_t* __restrict__ row_of) {
    pdl_entry();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < m; r += nw)
        for (int k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) row_of[k] = (uint32_t)r;
}

__global__ void csc_fill_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ row_of,
                                const double* __restrict__ val, int64_t n, int* __restrict__ row_idx,
                                double* __restrict__ cval) {
    pdl_entry();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = perm[i];
        row_idx[i] = (int)row_of[k];
        cval[i] = val[k];
    }
}

// col_ptr[c] = first position with key >= c (sorted keys)
__global__ void col_ptr_kernel(const uint32_t* __restrict__ skeys, int64_t n, int d, int* __restrict__ col_ptr) {
    pdl_entry();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= d; c += gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (skeys[mid] < (uint32_t)c) lo = mid + 1;
            else hi = mid;
        }
        col_ptr[c] = (int)lo;
    }
}

// ---------------------------------------------------------------- segment plans
// Warp-aggregated slot in bin b: one atomic per distinct bin among the active lanes (row lengths
// cluster on a few values, so per-lane atomics would serialise on a handful of addresses).
__device__ __forceinline__ int64_t bin_slot(int64_t* bins, int b) {
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, b);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == leader)
        base = atomicAdd(reinterpret_cast<unsigned long long*>(bins + b), (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    return (int64_t)base + __popc(peers & ((1u << lane) - 1u));
}

// short rows are binned by length, longest first (bin 2 piece - len), for the SpMM's row order
__global__ void plan_count_kernel(const int* __restrict__ ptr, int nrows, int piece, int64_t* __restrict__ is_long,
                                  int64_t* __restrict__ npieces, int64_t* __restrict__ bins) {
    pdl_entry();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
        const int len = ptr[r + 1] - ptr[r];
        const bool lg = len > 2 * piece;
        is_long[r] = lg ? 1 : 0;
        npieces[r] = lg ? (len + piece - 1) / piece : 0;
        if (!lg) bin_slot(bins, 2 * piece - len);
    }
}

// Pieces of the long rows in row order; the short rows scattered into their length bins (the
// order inside a bin is arbitrary: it only decides which warp computes a row).
__global__ void plan_fill_kernel(const int* __restrict__ ptr, int nrows, int piece, const int64_t* __restrict__ is_long,
                                 const int64_t* __restrict__ long_off, const int64_t* __restrict__ piece_off,
                                 int* __restrict__ long_rows, int* __restrict__ long_first, int* __restrict__ piece_beg,
                                 int* __restrict__ piece_end, int* __restrict__ piece_li,
                                 int* __restrict__ counts /* [nlong, npieces, nshort] */, int64_t* __restrict__ bin_off,
                                 int* __restrict__ order) {
    pdl_entry();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
        const int len = ptr[r + 1] - ptr[r];
        if (len > 2 * piece) {
            const int li = (int)long_off[r];
            const int pf = (int)piece_off[r];
            long_rows[li] = r;
            long_first[li] = pf;
            const int np = (len + piece - 1) / piece;
            for (int p = 0; p < np; ++p) {
                piece_beg[pf + p] = ptr[r] + p * piece;
                piece_end[pf + p] = min(ptr[r] + (p + 1) * piece, ptr[r + 1]);
                piece_li[pf + p] = li;
            }
        } else {
            order[bin_slot(bin_off, 2 * piece - len)] = r;
        }
        if (r == nrows - 1) {
            counts[0] = (int)(long_off[r] + is_long[r]);
            counts[1] = (int)(piece_off[r] + (len > 2 * piece ? (len + piece - 1) / piece : 0));
            counts[2] = nrows - counts[0];
        }
    }
}

// Pieces by the first input index they gather, in kPieceBuckets coarse buckets (counting sort;
// the order inside a bucket is arbitrary). Only which warp runs a piece, and when, changes: the
// partials are indexed by piece and summed in piece order, so results do not depend on it.
constexpr int kPieceBuckets = 1024;
__global__ void piece_order_kernel(const int* __restrict__ counts, const int* __restrict__ key,
                                   int64_t* __restrict__ bin_off, int* __restrict__ porder) {
    pdl_entry();
    const int np = counts[1];
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x)
        porder[bin_slot(bin_off, key[p])] = p;
}

// Key of a piece: the coarse bucket of the first input index it gathers.
__global__ void piece_key_kernel(const int* __restrict__ counts, const int* __restrict__ piece_beg,
                                 const int* __restrict__ idx, int range, int* __restrict__ key,
                                 int64_t* __restrict__ bins) {
    pdl_entry();
    const int np = counts[1];
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const int k = (int)min((int64_t)kPieceBuckets - 1, (int64_t)idx[piece_beg[p]] * kPieceBuckets / range);
        key[p] = k;
        bin_slot(bins, k);
    }
}

// ---------------------------------------------------------------- SpMM
// J = number of 64-column chunks (lane owns columns 2*lane + 64*j, +1). HOT: idx is relabelled
// (HotSet): entries < nh read the staged row in shared memory (hot + i * ldh), the others row
// idx - nh of `in`. The same loads in the same order either way, so the sums are identical.
template <int J, bool HOT, int NB>
__device__ __forceinline__ void gather_range(int kb, int ke, const int* __restrict__ idx, const double* __restrict__ val,
                                             const double* __restrict__ in, int ld, int ncols, int lane,
                                             double2 (&acc)[J], const double* hot, int nh, int ldh) {
    auto row = [&](int ci) -> const double* {
        if constexpr (HOT) return ci < nh ? hot + (size_t)ci * ldh : in + (size_t)(ci - nh) * ld;
        else return in + (size_t)ci * ld;
    };
    auto load = [&](const double* p) -> double2 {
        if constexpr (HOT) return *reinterpret_cast<const double2*>(p);  // generic: SMEM or global
        else return __ldg(reinterpret_cast<const double2*>(p));
    };
    for (int k0 = kb; k0 < ke; k0 += 32) {
        const int kk = k0 + lane;
        const int my_idx = kk < ke ? idx[kk] : 0;
        const double my_val = kk < ke ? val[kk] : 0.0;
        const int cnt = min(32, ke - k0);
        int e = 0;
        for (; e + NB <= cnt; e += NB) {
            const double* rp[NB];
            double cv[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                rp[u] = row(__shfl_sync(0xffffffffu, my_idx, e + u));
                cv[u] = __shfl_sync(0xffffffffu, my_val, e + u);
            }
            double2 x[NB][J];
#pragma unroll
            for (int u = 0; u < NB; ++u)
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const int c = 2 * lane + 64 * j;
                    x[u][j] = c < ncols ? load(rp[u] + c) : make_double2(0.0, 0.0);
                }
#pragma unroll
            for (int u = 0; u < NB; ++u)
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    acc[j].x = fma(cv[u], x[u][j].x, acc[j].x);
                    acc[j].y = fma(cv[u], x[u][j].y, acc[j].y);
                }
        }
        for (; e < cnt; ++e) {
            const double* r1 = row(__shfl_sync(0xffffffffu, my_idx, e));
            const double cv = __shfl_sync(0xffffffffu, my_val, e);
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int c = 2 * lane + 64 * j;
                if (c < ncols) {
                    const double2 x = load(r1 + c);
                    acc[j].x = fma(cv, x.x, acc[j].x);
                    acc[j].y = fma(cv, x.y, acc[j].y);
                }
            }
        }
    }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// The CTA's copy of the hot input rows: one 1-D TMA bulk copy (cp.async.bulk) per row into
// shared memory, completion counted in bytes on an mbarrier.
__device__ __forceinline__ void stage_hot_rows(double* hot, const int* __restrict__ cols, int nh, const double* in,
                                               int ld, int ncols, uint64_t* bar) {
    const unsigned bytes = (unsigned)ncols * 8u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                         "r"(bytes * (unsigned)nh)
                         : "memory");
        __syncwarp();
        for (int i = threadIdx.x; i < nh; i += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(hot + (size_t)i * ncols)),
                         "l"(in + (size_t)cols[i] * ld), "r"(bytes), "r"(smem_u32(bar))
                         : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}

// One launch for the whole product. Work item w < npieces is a piece of a long row: its
// partial row goes to `partial`, and the piece that finishes a row last (per-row arrival
// counter) sums that row's partials in piece order -- deterministic, no FP atomics. The other
// items are the short rows in the plan's longest-first order, written directly. Pieces come
// first, so their dependent gather chains start at the beginning of the launch instead of
// forming a tail.
// Occupancy / loads in flight (tools/spmm_lab.cu on the c2-c5 flush buffers): ell <= 128
// (J <= 2) four panel rows in flight per warp at 4 blocks per SM; wider panels two rows at 3.
// dst[c] = sum of the partial rows p = first, first + step, ... < last, in that order, eight
// rows in flight (read through L2: other SMs wrote them).
template <int J>
__device__ __forceinline__ void sum_partials(const double* partial, int ld, int first, int last, int step, int ncols,
                                             int lane, double* dst) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int c = 2 * lane + 64 * j;
        if (c < ncols) {
            double2 t = make_double2(0.0, 0.0);
            int p = first;
            for (; p + 8 * step <= last; p += 8 * step) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    v[u] = __ldcg(reinterpret_cast<const double2*>(partial + (size_t)(p + u * step) * ld + c));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    t.x += v[u].x;
                    t.y += v[u].y;
                }
            }
            for (; p < last; p += step) {
                const double2 v = __ldcg(reinterpret_cast<const double2*>(partial + (size_t)p * ld + c));
                t.x += v.x;
                t.y += v.y;
            }
            *reinterpret_cast<double2*>(dst + c) = t;
        }
    }
}

template <int J, bool HOT>
constexpr int spmm_threads() {
    return HOT ? (J <= 2 ? 1024 : 512) : 256;
}
template <int J, bool HOT>
constexpr int spmm_min_blocks() {
    return HOT ? 1 : (J <= 2 ? 4 : 3);
}
template <int J>
__host__ __device__ constexpr int spmm_batch() {
    return J <= 2 ? 4 : 2;
}

template <int J, bool HOT>
__global__ void __launch_bounds__(spmm_threads<J, HOT>(), spmm_min_blocks<J, HOT>()) spmm_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const double* __restrict__ val, int nrows,
    const int* __restrict__ piece_beg, const int* __restrict__ piece_end, const int* __restrict__ piece_li,
    const int* __restrict__ long_rows, const int* __restrict__ long_first, const int* __restrict__ counts,
    int* __restrict__ arrive, int* __restrict__ garrive, const int* __restrict__ order, int use_pieces, const double* __restrict__ in, int ld, int ncols,
    double* __restrict__ out, int ldo, double* __restrict__ partial, const int* __restrict__ hot_cols, int nh,
    const int* __restrict__ porder, int* __restrict__ ticket) {
    extern __shared__ __align__(128) double hot_sm[];
    __shared__ uint64_t hot_bar;
    if constexpr (HOT) {
        pdl_entry();
        stage_hot_rows(hot_sm, hot_cols, nh, in, ld, ncols, &hot_bar);
    }
    if constexpr (!HOT) pdl_entry();
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int np = use_pieces ? counts[1] : 0;
    const int nl = use_pieces ? counts[0] : 0;
    const int ns = counts[2];  // short rows (all rows when there are no long ones)
    constexpr int NB = spmm_batch<J>();
    // Pieces either statically strided over the grid's warps or, with a ticket counter (gathered
    // panels larger than L2), taken in order as warps become free: the pieces in flight then stay
    // a window of consecutive pieces -- with the pieces in the order of the first index they
    // gather, a window of the panel -- whatever the individual piece durations. The warp that
    // leaves the piece phase last resets the counters for the next launch.
    const bool dyn = ticket != nullptr && np > 0;
    bool grabbing = dyn;
    int sw = warp;
    for (;;) {
        int w;
        if (grabbing) {
            int t = 0;
            if (lane == 0) t = atomicAdd(ticket, 1);
            w = __shfl_sync(0xffffffffu, t, 0);
            if (w >= np) {
                grabbing = false;
                if (lane == 0 && atomicAdd(ticket + 1, 1) == nw - 1) {
                    ticket[0] = 0;
                    ticket[1] = 0;
                }
                continue;
            }
        } else {
            w = dyn ? np + sw : sw;
            if (w >= np + ns) break;
            sw += nw;
        }
        double2 acc[J];
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = make_double2(0.0, 0.0);
        if (w < np) {
            const int pc = porder ? porder[w] : w;  // the piece this warp runs
            gather_range<J, HOT, NB>(piece_beg[pc], piece_end[pc], idx, val, in, ld, ncols, lane, acc, hot_sm, nh,
                                     ncols);
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int c = 2 * lane + 64 * j;
                if (c < ncols) *reinterpret_cast<double2*>(partial + (size_t)pc * ld + c) = acc[j];
            }
            __threadfence();
            const int li = piece_li[pc];
            const int first = long_first[li], last = li + 1 < nl ? long_first[li + 1] : np;
            // Two-level sum, both levels in piece order (deterministic, no FP atomics): the piece
            // that finishes a group of kPieceGroup consecutive pieces last sums the group, and the
            // group that finishes the row last sums the group sums. A row of one group is summed
            // straight into `out`.
            const int gfirst = first + (pc - first) / kPieceGroup * kPieceGroup;
            const int glast = min(gfirst + kPieceGroup, last);
            int old = 0;
            if (lane == 0) old = atomicAdd(garrive + gfirst, 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old != glast - gfirst - 1) continue;
            __threadfence();
            if (lane == 0) garrive[gfirst] = 0;  // ready for the next launch
            const bool single = last - first <= kPieceGroup;
            const int r = long_rows[li];
            sum_partials<J>(partial, ld, gfirst, glast, 1, ncols, lane,
                            single ? out + (size_t)r * ldo : partial + (size_t)gfirst * ld);
            if (single) continue;
            __threadfence();
            if (lane == 0) old = atomicAdd(arrive + li, 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            const int ngroups = (last - first + kPieceGroup - 1) / kPieceGroup;
            if (old != ngroups - 1) continue;
            __threadfence();
            if (lane == 0) arrive[li] = 0;
            sum_partials<J>(partial, ld, first, last, kPieceGroup, ncols, lane, out + (size_t)r * ldo);
            continue;
        }
        const int r = order[w - np];
        const int kb = ptr[r], ke = ptr[r + 1];
        gather_range<J, HOT, NB>(kb, ke, idx, val, in, ld, ncols, lane, acc, hot_sm, nh, ncols);
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int c = 2 * lane + 64 * j;
            if (c < ncols) *reinterpret_cast<double2*>(out + (size_t)r * ldo + c) = acc[j];
        }
    }
}

__global__ void hot_slot_kernel(const int* __restrict__ cols, int n, int* __restrict__ slot) {
    pdl_entry();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) slot[cols[i]] = i;
}

__global__ void hot_relabel_kernel(const uint32_t* __restrict__ col, int64_t nnz, const int* __restrict__ slot, int n,
                                   int* __restrict__ idx2) {
    pdl_entry();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = col[k];
        const int sl = slot[c];
        idx2[k] = sl >= 0 ? sl : n + (int)c;
    }
}

// ---------------------------------------------------------------- validation
// Device-resident input rows (sfdg_sketcher_append_csr_device): first bad row
// (index out of range / not strictly increasing / non-finite), sparse.cpp:8-20.
__global__ void validate_rows_kernel(const int64_t* __restrict__ row_ptr, int64_t nrows, const uint32_t* __restrict__ cols,
                                     const double* __restrict__ vals, uint32_t d, unsigned long long* __restrict__ first_bad,
                                     int* __restrict__ kind) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < nrows; r += nw) {
        bool bad_idx = false, bad_val = false;
        for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) {
            const uint32_t c = cols[k];
            if (c >= d) bad_idx = true;
            if (k > row_ptr[r] && cols[k - 1] >= c) bad_idx = true;
            if (!isfinite(vals[k])) bad_val = true;
        }
        const bool bi = __any_sync(0xffffffffu, bad_idx), bv = __any_sync(0xffffffffu, bad_val);
        if ((bi || bv) && lane == 0) {
            atomicMin(first_bad, (unsigned long long)r);
            atomicOr(kind, bi ? ERR_BAD_INDEX : ERR_BAD_VALUE);
        }
    }
}

// ---------------------------------------------------------------- misc
__global__ void rebase_rows_kernel(const int64_t* __restrict__ src, int64_t base, int m, int* __restrict__ dst) {
    pdl_entry();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += gridDim.x * blockDim.x)
        dst[i] = (int)(src[i] - base);
}

}  // namespace

// ============================================================== host side

void exclusive_scan(const int64_t* d_in, int64_t* d_out, int64_t n, Scratch& scr, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t per = (int64_t)kScanBlock * kScanItems;
    const int64_t nb = (n + per - 1) / per;
    if (nb == 1) {
        LAUNCH(scan_block_kernel, 1, kScanBlock, 0, st, d_in, d_out, n, (int64_t*)nullptr);
        return;
    }
    int64_t* sums = scr.take<int64_t>(nb);
    int64_t* offs = scr.take<int64_t>(nb);
    LAUNCH(scan_block_kernel, (unsigned)nb, kScanBlock, 0, st, d_in, d_out, n, sums);
    exclusive_scan(sums, offs, nb, scr, st);
    LAUNCH(scan_add_kernel, (unsigned)nb, kScanBlock, 0, st, d_out, n, offs);
}

void DevCsr::reserve(int m_cap, int64_t nnz_cap_) {
    if (m_cap > rows_cap) {
        if (row_ptr) cudaFree(row_ptr);
        CK(cudaMalloc(&row_ptr, (size_t)(m_cap + 1) * sizeof(int)));
        rows_cap = m_cap;
    }
    if (nnz_cap_ > nnz_cap) {
        nnz_cap = std::max<int64_t>(nnz_cap_, nnz_cap * 3 / 2);
        for (void* p : {(void*)col, (void*)val, (void*)row_idx, (void*)cval})
            if (p) cudaFree(p);
        CK(cudaMalloc(&col, nnz_cap * sizeof(uint32_t)));
        CK(cudaMalloc(&val, nnz_cap * sizeof(double)));
        CK(cudaMalloc(&row_idx, nnz_cap * sizeof(int)));
        CK(cudaMalloc(&cval, nnz_cap * sizeof(double)));
    }
}

void DevCsr::release() {
    for (void* p : {(void*)row_ptr, (void*)col, (void*)val, (void*)col_ptr, (void*)row_idx, (void*)cval})
        if (p) cudaFree(p);
    row_ptr = nullptr;
    col = nullptr;
    val = nullptr;
    col_ptr = nullptr;
    row_idx = nullptr;
    cval = nullptr;
    rows_cap = 0;
    nnz_cap = 0;
    d_cap = 0;
}

void DevCsr::set_shape(int m_, int d_, int64_t nnz_) {
    if (nnz_ >= (int64_t)INT32_MAX) throw invalid_argument("buffer: more than 2^31-1 stored entries per flush");
    m = m_;
    d = d_;
    nnz = nnz_;
    reserve(m_, std::max<int64_t>(nnz_, 1));
    if (d_ + 1 > d_cap) {
        if (col_ptr) cudaFree(col_ptr);
        CK(cudaMalloc(&col_ptr, (size_t)(d_ + 1) * sizeof(int)));
        d_cap = d_ + 1;
    }
}

void rebase_row_ptr(const int64_t* d_src, int64_t base, int m, int* d_dst, cudaStream_t st) {
    LAUNCH(rebase_rows_kernel, ceil_div(m + 1, 256), 256, 0, st, d_src, base, m, d_dst);
}

// CSR -> CSC (stable in row order) + long-row plans for both orientations.
void build_transpose(DevCsr& a, Scratch& scr, cudaStream_t st) {
    ProfScope prof("csc_build", st);
    const int64_t n = a.nnz;
    const int d = a.d;
    if (n == 0) {
        CK(cudaMemsetAsync(a.col_ptr, 0, (size_t)(d + 1) * sizeof(int), st));
        return;
    }
    uint32_t* k0 = scr.take<uint32_t>(n);
    uint32_t* k1 = scr.take<uint32_t>(n);
    uint32_t* v0 = scr.take<uint32_t>(n);
    uint32_t* v1 = scr.take<uint32_t>(n);
    uint32_t* row_of = scr.take<uint32_t>(n);
    CK(cudaMemcpyAsync(k0, a.col, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    const unsigned g = (unsigned)std::min<int64_t>(8 * kSMs, (n + 255) / 256);
    LAUNCH(iota_kernel, g, 256, 0, st, v0, n);
    int bits = 0;
    while (bits < 32 && (1ull << bits) < (unsigned long long)d) ++bits;
    const int ntiles = (int)((n + kRadixTile - 1) / kRadixTile);
    int64_t* hist = scr.take<int64_t>((int64_t)256 * ntiles);
    int64_t* offs = scr.take<int64_t>((int64_t)256 * ntiles);
    for (int shift = 0; shift < bits; shift += 8) {
        LAUNCH(radix_hist_kernel, ntiles, kRadixThreads, 0, st, k0, n, shift, ntiles, hist);
        exclusive_scan(hist, offs, (int64_t)256 * ntiles, scr, st);
        LAUNCH(radix_scatter_kernel, ntiles, kRadixThreads, 0, st, k0, v0, k1, v1, n, shift, ntiles, offs);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    LAUNCH(expand_rows_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)a.m * 32, 256))), 256, 0, st,
           a.row_ptr, a.m, row_of);
    LAUNCH(csc_fill_kernel, g, 256, 0, st, v0, row_of, a.val, n, a.row_idx, a.cval);
    LAUNCH(col_ptr_kernel, ceil_div(d + 1, 256), 256, 0, st, k0, n, d, a.col_ptr);
}

int spmm_piece_length(int64_t nnz) {
    const int64_t per_warp = nnz / (16 * kSMs * 8);  // the SpMM grid: <= 16 x 148 blocks of 8 warps
    int piece = kPiece;
    while (piece < 2048 && 2 * (int64_t)piece <= per_warp / 2) piece *= 2;
    return piece;
}

int spmm_big_piece_length(int piece, int64_t nnz, int64_t in_rows, size_t panel_bytes, size_t l2_bytes) {
    // The pieces in flight are the resident warps' (kSMs x 3 blocks x 8 warps, one piece each);
    // taken by ticket in the order of the first panel row they gather, they cover a window of
    // about warps x piece / (entries per panel row) panel rows. That window has to stay in the
    // L2 next to the streamed CSR / CSC arrays and the partial rows: a quarter of the L2.
    // c5 CSC (2 GB panel, 21 entries per panel row): 64 entries, DRAM 36.7 -> 20.2 GB and 6.17 ->
    // 3.90 ms per launch; c3 (160 MB panel, 110 entries per row) keeps its 512
    // (profiles/r02f_piece_big_ab.txt). SFDG_PIECE_BIG=<entries> overrides (A/B testing).
    static const int want = std::getenv("SFDG_PIECE_BIG") ? std::atoi(std::getenv("SFDG_PIECE_BIG")) : 0;
    if (want >= 8) return want;
    if (in_rows <= 0 || panel_bytes == 0) return piece;
    const double row_bytes = (double)panel_bytes / (double)in_rows;
    const double window_rows = 0.25 * (double)l2_bytes / row_bytes;
    const double per_row = (double)nnz / (double)in_rows;
    const double fit = window_rows * per_row / (double)(kSMs * 24);
    int p = 32;
    while (2 * p <= piece && 2.0 * p <= fit) p *= 2;
    return p;
}

// SFDG_SPMM_BLOCKS=<k> (A/B testing): at most k blocks per SM in the SpMM grid (default 16)
static unsigned spmm_blocks_per_sm() {
    static const int want = std::getenv("SFDG_SPMM_BLOCKS") ? std::atoi(std::getenv("SFDG_SPMM_BLOCKS")) : 0;
    return want >= 1 ? (unsigned)want : 16u;
}

void SegPlan::build(const int* d_ptr, int nrows, int64_t nnz, Scratch& scr, cudaStream_t st, const int* d_idx,
                    int idx_range, size_t panel_bytes) {
    ProfScope prof("csc_build", st);
    rows = nrows;
    host_long = -1;
    piece = spmm_piece_length(nnz);
    int l2 = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    // A gathered panel larger than the L2: the pieces in flight (resident warps x piece entries)
    // must cover a window of the panel that fits in the L2, or the long rows' gathers all come
    // from HBM (see spmm_big_piece_length()).
    if (panel_bytes > (size_t)l2) piece = spmm_big_piece_length(piece, nnz, idx_range, panel_bytes, (size_t)l2);
    reserve_pieces(2 * (nnz / std::min(piece, kPiece)) + 2);  // any piece length >= min(piece, kPiece)
    if (garrive_fresh) {
        CK(cudaMemsetAsync(garrive, 0, cap_pieces * sizeof(int), st));
        garrive_fresh = false;
    }
    if (nrows > cap_rows) {
        for (void* p : {(void*)long_rows, (void*)long_first, (void*)arrive, (void*)order}) if (p) cudaFree(p);
        CK(cudaMalloc(&long_rows, (size_t)nrows * sizeof(int)));
        CK(cudaMalloc(&long_first, (size_t)nrows * sizeof(int)));
        CK(cudaMalloc(&arrive, (size_t)nrows * sizeof(int)));
        CK(cudaMalloc(&order, (size_t)nrows * sizeof(int)));
        CK(cudaMemsetAsync(arrive, 0, (size_t)nrows * sizeof(int), st));
        cap_rows = nrows;
    }
    host_pieces = -1;
    has_porder = false;
    if (!counts) CK(cudaMalloc(&counts, 3 * sizeof(int)));
    if (!ticket) {
        CK(cudaMalloc(&ticket, 2 * sizeof(int)));
        CK(cudaMemsetAsync(ticket, 0, 2 * sizeof(int), st));  // on the plan's stream; self-resetting afterwards
    }
    big = panel_bytes > (size_t)l2;
    CK(cudaMemsetAsync(counts, 0, 3 * sizeof(int), st));
    if (nrows == 0) return;
    int64_t* is_long = scr.take<int64_t>(nrows);
    int64_t* np = scr.take<int64_t>(nrows);
    int64_t* long_off = scr.take<int64_t>(nrows);
    int64_t* piece_off = scr.take<int64_t>(nrows);
    const int nbins = 2 * piece + 1;  // short rows have 0 .. 2 piece entries
    int64_t* bins = scr.take<int64_t>(nbins);
    int64_t* bin_off = scr.take<int64_t>(nbins);
    CK(cudaMemsetAsync(bins, 0, nbins * sizeof(int64_t), st));
    const unsigned g = std::max(1u, std::min(8u * kSMs, ceil_div(nrows, 256)));
    LAUNCH(plan_count_kernel, g, 256, 0, st, d_ptr, nrows, piece, is_long, np, bins);
    exclusive_scan(is_long, long_off, nrows, scr, st);
    exclusive_scan(np, piece_off, nrows, scr, st);
    exclusive_scan(bins, bin_off, nbins, scr, st);
    // pieces <= nnz / piece + nrows; size the piece arrays for the worst case of this call
    LAUNCH(plan_fill_kernel, g, 256, 0, st, d_ptr, nrows, piece, is_long, long_off, piece_off, long_rows, long_first,
           piece_beg, piece_end, piece_li, counts, bin_off, order);
    // Pieces in the order of the first input index they gather (porder), for panels larger
    // than the L2 (c3, c5): taken by ticket in that order (spmm()), the pieces in flight are the
    // pieces of many long rows over one window of panel rows, sized to fit the L2 by
    // spmm_big_piece_length(). With statically strided pieces of the default length the order
    // alone gave c5 CSC DRAM 41.6 -> 36.8 GB per launch (L2 hits 3 -> 10 %); the ticket and the
    // 64-entry pieces 20.2 GB (39 %), 6.17 -> 3.90 ms. An L2-resident panel (c4) gains nothing and
    // its standalone launch got slower (146 -> 156 us).
    // SFDG_PIECE_ORDER=0 / 1 forces it off / on (A/B testing).
    const char* po_env = std::getenv("SFDG_PIECE_ORDER");
    const bool pord = po_env ? std::atoi(po_env) != 0 : panel_bytes > (size_t)l2;
    has_porder = pord && d_idx && idx_range > 0 && nnz > 2 * piece;
    if (has_porder) {
        int* key = scr.take<int>(cap_pieces);
        int64_t* pb = scr.take<int64_t>(kPieceBuckets);
        int64_t* po = scr.take<int64_t>(kPieceBuckets);
        CK(cudaMemsetAsync(pb, 0, kPieceBuckets * sizeof(int64_t), st));
        const unsigned gp = std::max(1u, std::min(8u * kSMs, ceil_div((size_t)cap_pieces, 256)));
        LAUNCH(piece_key_kernel, gp, 256, 0, st, counts, piece_beg, d_idx, idx_range, key, pb);
        exclusive_scan(pb, po, kPieceBuckets, scr, st);
        LAUNCH(piece_order_kernel, gp, 256, 0, st, counts, key, po, porder);
    }
}

void SegPlan::reserve_pieces(int64_t need) {
    if (need > cap_pieces) {
        for (void* p : {(void*)piece_beg, (void*)piece_end, (void*)piece_li, (void*)porder, (void*)garrive}) if (p) cudaFree(p);
        cap_pieces = need;
        CK(cudaMalloc(&garrive, cap_pieces * sizeof(int)));
        garrive_fresh = true;  // build() zeroes it on the plan's stream; self-resetting afterwards
        CK(cudaMalloc(&piece_beg, cap_pieces * sizeof(int)));
        CK(cudaMalloc(&piece_end, cap_pieces * sizeof(int)));
        CK(cudaMalloc(&piece_li, cap_pieces * sizeof(int)));
        CK(cudaMalloc(&porder, cap_pieces * sizeof(int)));
    }
}

void SegPlan::ensure_partial(int64_t doubles) const {
    if (doubles <= partial_cap) return;
    if (partial) CK(cudaFree(partial));
    partial_cap = std::max<int64_t>(doubles, partial_cap * 3 / 2);
    CK(cudaMalloc(&partial, partial_cap * sizeof(double)));
}

void SegPlan::release() {
    if (partial) cudaFree(partial);
    partial = nullptr;
    partial_cap = 0;
    for (void* p : {(void*)long_rows, (void*)long_first, (void*)piece_beg, (void*)piece_end, (void*)piece_li,
                    (void*)arrive, (void*)order, (void*)counts, (void*)porder, (void*)garrive, (void*)ticket})
        if (p) cudaFree(p);
    ticket = nullptr;
    long_rows = long_first = piece_beg = piece_end = piece_li = arrive = order = counts = porder = garrive = nullptr;
    cap_rows = 0;
    cap_pieces = 0;
}

namespace {
// Persisting-L2 window for a gathered panel of `panel` bytes (0 = none): only when SFDG_L2_WINDOW
// asks for one and the panel is at least twice the L2, capped by the device's window and
// persisting-carve-out limits (the carve-out is set once per device).
size_t l2_window_bytes(size_t panel) {
    static const size_t want = std::getenv("SFDG_L2_WINDOW") ? (size_t)std::atoll(std::getenv("SFDG_L2_WINDOW")) << 20 : 0;
    if (want == 0 || panel == 0) return 0;
    int dev = 0, l2 = 0, maxwin = 0, maxpers = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    if (panel < 2 * (size_t)l2) return 0;
    CK(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    CK(cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, dev));
    const size_t bytes = std::min({want, (size_t)maxwin, (size_t)maxpers, panel});
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> g(mu);
    if (done.insert(dev).second) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(want, (size_t)maxpers)));
    return bytes;
}
}  // namespace

void spmm(const int* d_ptr, const int* d_idx, const double* d_val, int nrows, const SegPlan& plan, int64_t nnz,
          const double* d_in, int ld, int ncols, double* d_out, int ldo, Scratch& scr, cudaStream_t st,
          int64_t in_rows, int alg_cols, const HotSet* hot) {
    if (nrows == 0) return;
    if (ncols % 2 != 0 || ld % 2 != 0 || ldo % 2 != 0) throw invalid_argument("spmm: panel widths must be even");
    ProfScope prof("spmm", st);
    {
        const double w = alg_cols > 0 ? alg_cols : ncols, ir = in_rows >= 0 ? (double)in_rows : (double)nrows;
        prof.work(2.0 * (double)nnz * w, 12.0 * (double)nnz + 8.0 * (nrows + 1) + 8.0 * w * (ir + nrows));
    }
    const int J = (ncols + 63) / 64;
    const int use_pieces = plan.host_long != 0 ? 1 : 0;
    const int64_t pieces = plan.host_pieces >= 0 ? plan.host_pieces : 2 * (nnz / plan.piece) + 2;
    // a function of nrows only, so a captured sweep block replays unchanged for any piece count
    const unsigned grid = std::max(1u, std::min(spmm_blocks_per_sm() * kSMs, ceil_div((size_t)nrows * 2 * 32, 256)));
    if (use_pieces) plan.ensure_partial(std::max<int64_t>(pieces, 1) * ld);
    double* partial = use_pieces ? plan.partial : nullptr;
    // pieces by ticket for gathered panels larger than L2 (SFDG_SPMM_DYN=0 / 1 forces it off / on
    // for every panel: A/B testing; the sums do not depend on it)
    static const int dyn_env = std::getenv("SFDG_SPMM_DYN") ? std::atoi(std::getenv("SFDG_SPMM_DYN")) : -1;
    int* ticket = use_pieces && (dyn_env < 0 ? plan.big : dyn_env != 0) ? plan.ticket : nullptr;
    const bool use_hot = hot && hot->n > 0;
    if (use_hot) {
        int dev = 0, sms = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const size_t smem = (size_t)hot->n * ncols * sizeof(double);
        switch (J) {
#define SPMM_HOT(JJ)                                                                                                  \
    case JJ: {                                                                                                        \
        auto* fn = spmm_kernel<JJ, true>;                                                                             \
        if (first_on_device((const void*)fn)) allow_max_dynamic_smem(fn);                                            \
        LAUNCH(fn, (unsigned)sms, (spmm_threads<JJ, true>()), smem, st, d_ptr, hot->idx, d_val, nrows, plan.piece_beg, \
               plan.piece_end, plan.piece_li, plan.long_rows, plan.long_first, plan.counts, plan.arrive, plan.garrive, plan.order, use_pieces,  \
               d_in, ld, ncols, d_out, ldo, partial, hot->cols, hot->n, plan.piece_order(), ticket);                     \
        break;                                                                                                        \
    }
            SPMM_HOT(1)
            SPMM_HOT(2)
            SPMM_HOT(3)
            SPMM_HOT(4)
            SPMM_HOT(5)
            SPMM_HOT(6)
            SPMM_HOT(7)
            SPMM_HOT(8)
#undef SPMM_HOT
            default:
                throw invalid_argument("spmm: panel wider than 512 columns");
        }
        return;
    }
    // SFDG_L2_WINDOW=<MB> (A/B testing): for the gather of a panel much larger than L2 in the CSR
    // direction (rows of W by column id), keep its first MB -- the most frequent columns when the
    // ids are frequency ranked -- persisting in L2
    const size_t win = l2_window_bytes(in_rows >= 0 && hot ? (size_t)in_rows * ld * sizeof(double) : 0);
    if (win > 0) {
        switch (J) {
#define SPMM_WIN(JJ)                                                                                               \
    case JJ:                                                                                                       \
        ::sfdg::launch_kernel_l2win((spmm_kernel<JJ, false>), dim3(grid), dim3(256), 0, st, (const void*)d_in, win,  \
               d_ptr, d_idx, d_val, nrows, plan.piece_beg,                                                          \
               plan.piece_end, plan.piece_li, plan.long_rows, plan.long_first, plan.counts, plan.arrive, plan.garrive, plan.order, use_pieces, \
               d_in, ld, ncols, d_out, ldo, partial, (const int*)nullptr, 0, plan.piece_order(), ticket);            \
        g_launches.fetch_add(1, std::memory_order_relaxed);                                                      \
        return;
            SPMM_WIN(1)
            SPMM_WIN(2)
            SPMM_WIN(3)
            SPMM_WIN(4)
            SPMM_WIN(5)
            SPMM_WIN(6)
            SPMM_WIN(7)
            SPMM_WIN(8)
#undef SPMM_WIN
            default:
                throw invalid_argument("spmm: panel wider than 512 columns");
        }
    }
    switch (J) {
#define SPMM_CASE(JJ)                                                                                              \
    case JJ:                                                                                                       \
        LAUNCH((spmm_kernel<JJ, false>), grid, 256, 0, st, d_ptr, d_idx, d_val, nrows, plan.piece_beg,             \
               plan.piece_end, plan.piece_li, plan.long_rows, plan.long_first, plan.counts, plan.arrive, plan.garrive, plan.order, use_pieces, \
               d_in, ld, ncols, d_out, ldo, partial, (const int*)nullptr, 0, plan.piece_order(), ticket);            \
        break;
        SPMM_CASE(1)
        SPMM_CASE(2)
        SPMM_CASE(3)
        SPMM_CASE(4)
        SPMM_CASE(5)
        SPMM_CASE(6)
        SPMM_CASE(7)
        SPMM_CASE(8)
#undef SPMM_CASE
        default:
            throw invalid_argument("spmm: panel wider than 512 columns");
    }
}

int hot_rows_capacity(int ncols) {
    // 200 KB of the 227 KB a CTA may use (static smem and the L1 keep the rest)
    return (int)((200u * 1024u) / ((unsigned)ncols * sizeof(double)));
}

void hot_relabel(const int* d_cols_hot, int n, const uint32_t* col, int64_t nnz, int d, int* slot, int* idx2,
                 cudaStream_t st) {
    CK(cudaMemsetAsync(slot, 0xff, (size_t)d * sizeof(int), st));
    if (n > 0) LAUNCH(hot_slot_kernel, ceil_div(n, 256), 256, 0, st, d_cols_hot, n, slot);
    if (nnz > 0)
        LAUNCH(hot_relabel_kernel, std::max(1u, std::min(8u * kSMs, ceil_div((size_t)nnz, 256))), 256, 0, st, col, nnz,
               slot, n, idx2);
}

int64_t validate_rows_device(const int64_t* d_row_ptr, int64_t nrows, const uint32_t* d_cols, const double* d_vals,
                             uint32_t d, int* kind_out, Scratch& scr, cudaStream_t st) {
    unsigned long long* first = scr.take<unsigned long long>(1);
    int* kind = scr.take<int>(2);
    const unsigned long long init = ~0ull;
    CK(cudaMemcpyAsync(first, &init, sizeof init, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(kind, 0, sizeof(int), st));
    if (nrows > 0)
        LAUNCH(validate_rows_kernel, std::max(1u, std::min(16u * kSMs, ceil_div((size_t)nrows * 32, 256))), 256, 0, st,
               d_row_ptr, nrows, d_cols, d_vals, d, first, kind);
    unsigned long long h_first = 0;
    int h_kind = 0;
    CK(cudaMemcpyAsync(&h_first, first, sizeof h_first, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h_kind, kind, sizeof h_kind, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *kind_out = h_kind;
    return h_first == ~0ull ? -1 : (int64_t)h_first;
}

}  // namespace sfdg
