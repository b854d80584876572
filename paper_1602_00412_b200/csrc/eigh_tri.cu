// eigh_tri.cu -- fast symmetric eigensolver for the 2ell x 2ell (and ell x ell) Grams.
//
// Contract: the jacobi_eigh one (la_core.cpp:24-80): eigenvalues descending with their
// eigenvectors, for the symmetric Gram K of svd_top (la_core.cpp:90-103) and dense_shrink
// (shrink.cpp:34-36). Parity needs B^T B = sum_i (lambda_i - lambda_ell) v_i v_i^T to 1e-8,
// i.e. accurate eigenvalues and eigenvectors of the top ell -- not the reference's
// rotation sequence. Jacobi on one SM is latency bound (~8 ms at n = 200, eigh.cu), so:
//
//  1. tridiag_kernel (1 CTA): Householder reduction K = Q T Q^T (LAPACK dsytd2 algebra),
//     packed upper triangle in shared memory; n-2 steps of symv + rank-2 update.
//  2. bisect_kernel (warp per eigenvalue): Sturm-count multisection on T, 32 shifts per
//     step (5 bits per iteration) to full double precision.
//  3. twisted_kernel (lane pair per eigenvalue): eigenvector from the forward/backward
//     twisted factorisations in one pass; inviter_kernel (thread per eigenvalue: inverse
//     iteration with a partially pivoted tridiagonal LU, distinct deterministic start
//     vectors) redoes the eigenvalues in clusters, which need independent start vectors.
//  4. cluster_kernel (warp per cluster of eigenvalues closer than 1e-6 |T|): modified
//     Gram-Schmidt twice, then Rayleigh-Ritz with a small Jacobi inside the cluster so each
//     vector is the right eigenvector, not just a basis of the cluster's space.
//  5. backtransform_kernel: U = Q X by applying the reflectors.
// Degenerate starts mirror the reference: if K's off-diagonal norm is already below the
// tolerance the reference performs no rotation, so neither do we (diagonal + identity).
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr int kTriThreads = 1024;
constexpr int kTriSmemMax = 232;

struct TriArgs {
    const double* K;
    int n, ldk;
    double tol_sq;
    const double* d_fsq;
    double* gpacked;
    int use_smem;
    double* d;     // n diagonal of T
    double* e;     // n-1 off-diagonal of T
    double* vh;    // n x n: reflector k in row k, entries k+1.. (v_{k+1} = 1)
    double* tau;   // n
    int* trivial;  // 1 when K is already diagonal within the tolerance
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Branch-free double reciprocal: MUFU seed (rcp.approx.ftz.f64, ~2^-23) + two Newton
// steps (~1 ulp). IEEE division carries a slow-path branch per divide, which serialises
// the interleaved Sturm chains below; this keeps them independent.
__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

template <bool SMEM>
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(TriArgs a) {
    pdl_entry();
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ int tri[1024];
    __shared__ double s_tau, s_scal, s_kk;
    const int n = a.n;
    double* A = SMEM ? sm : a.gpacked;
    double* vs = SMEM ? sm + (size_t)n * (n + 1) / 2 : a.gpacked + (size_t)n * (n + 1) / 2;  // n
    double* ws = vs + n;                                                                       // n
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int j = tid; j < n; j += nt) tri[j] = j * (j + 1) / 2;
    __syncthreads();
    double off = 0.0;
    for (int j = warp; j < n; j += nw)
        for (int i = lane; i <= j; i += 32) {
            const double v = a.K[(size_t)i * a.ldk + j];
            A[tri[j] + i] = v;
            if (i != j) off += 2.0 * v * v;
        }
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {
        const double ot = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = ot * ot;
    }
    off = block_sum(off, red);
    if (!(off > tol_sq) || n == 1) {  // the reference's Jacobi would not rotate at all (la_core.cpp:33)
        for (int i = tid; i < n; i += nt) {
            a.d[i] = A[tri[i] + i];
            if (i + 1 < n) a.e[i] = 0.0;
        }
        if (tid == 0) *a.trivial = 1;
        return;
    }
    if (tid == 0) *a.trivial = 0;
    __shared__ double wred[32];
    for (int k = 0; k + 2 < n; ++k) {
        // warp 0: Householder (dlarfg) on x_j = A(k, j), j = k+1..n-1, and the vector v
        if (warp == 0) {
            double xs = 0.0;
            for (int j = k + 2 + lane; j < n; j += 32) {
                const double x = A[tri[j] + k];
                xs += x * x;
            }
            xs = warp_sum(xs);
            const double alpha = A[tri[k + 1] + k];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xs > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + xs), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            for (int j = k + 1 + lane; j < n; j += 32) {
                const double v = (j == k + 1) ? 1.0 : A[tri[j] + k] * scal;
                vs[j] = v;
                a.vh[(size_t)k * n + j] = v;
            }
            if (lane == 0) {
                s_tau = tau;
                a.d[k] = A[tri[k] + k];
                a.e[k] = beta;
                a.tau[k] = tau;
            }
        }
        __syncthreads();
        const double tau = s_tau;
        if (tau == 0.0) continue;
        // p = tau A22 v (warp per row) and per-warp partials of p^T v
        double pv = 0.0;
        for (int i = k + 1 + warp; i < n; i += nw) {
            double s = 0.0;
            for (int j = k + 1 + lane; j < n; j += 32) s += A[i <= j ? tri[j] + i : tri[i] + j] * vs[j];
            s = warp_sum(s) * tau;
            if (lane == 0) ws[i] = s;
            pv += s * vs[i];
        }
        if (lane == 0) wred[warp] = pv;
        __syncthreads();
        double kk = 0.0;
        for (int w2 = 0; w2 < nw; ++w2) kk += wred[w2];  // fixed order, same in every thread
        kk *= 0.5 * tau;
        for (int i = k + 1 + tid; i < n; i += nt) ws[i] -= kk * vs[i];
        __syncthreads();
        // A22 -= v w^T + w v^T (upper triangle)
        for (int j = k + 1 + warp; j < n; j += nw) {
            const double vj = vs[j], wj = ws[j];
            for (int i = k + 1 + lane; i <= j; i += 32) A[tri[j] + i] -= vs[i] * wj + ws[i] * vj;
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            a.d[n - 2] = A[tri[n - 2] + n - 2];
            a.e[n - 2] = A[tri[n - 1] + n - 2];
            a.tau[n - 2] = 0.0;
        }
        a.d[n - 1] = A[tri[n - 1] + n - 1];
        a.tau[n - 1] = 0.0;
    }
}

// Row-distributed Householder tridiagonalisation, one CTA or a cluster of C CTAs.
//
// The full symmetric matrix lives in shared memory, row i on CTA (i % C), local row
// i / C, owned by warp (i / C) % NW. Step k is fused with the update of step k-1:
//   S1 (owner warp of row k): c_{k-1} = tau_{k-1}/2 p_{k-1}^T v_{k-1}; apply the rank-2
//      update of step k-1 to row k; Householder (dlarfg) on row k -> v_k, tau_k; broadcast
//      v_k, tau_k, c_{k-1} into every CTA of the cluster.
//   S2 (every warp, rows i > k): a_ij -= v_i w_j + w_i v_j (step k-1, w = p - c v) and in
//      the same pass p_k,i = tau_k sum_j a_ij v_k,j; broadcast p_k,i.
// Two (cluster) barriers per step; each element is read and written once per step, with
// lanes over columns (conflict-free rows). Algebra as tridiag_kernel (dsytd2).
#ifdef SFDG_TRI_PROBE  // tools/tri_probe: per-step clock64 stamps of the single-CTA row kernel
__device__ long long g_tri_probe[8 * 1100];
#define TPROBE(i, cond) \
    if (cond) g_tri_probe[8 * k + (i)] = clock64();
#else
#define TPROBE(i, cond)
#endif
struct TriRowsArgs {
    TriArgs a;
    int C;      // CTAs in the cluster
    int rows;   // ceil(n / C): local rows per CTA
};

template <int C, int NT, int NTHR>
__global__ void __launch_bounds__(NTHR) tridiag_rows_kernel(TriRowsArgs ra) {
    pdl_entry();
    constexpr int NW = NTHR / 32;
    extern __shared__ double sm[];
    __shared__ double s_sc[2][2];  // [k & 1] = {tau_k, c_{k-1}}
    __shared__ double s_off[16];
    __shared__ double red[32];
    const TriArgs& a = ra.a;
    const int n = a.n;
    const unsigned rank = C > 1 ? cluster_rank() : 0u;
    const int tid = threadIdx.x, lane = tid & 31, wl = tid >> 5;
    const int nloc = (n - (int)rank + C - 1) / C;  // rows rank, rank + C, ...
    double* A = sm;                                // rows x n
    double* vbuf = sm + (size_t)ra.rows * n;       // 2 x n
    double* pbuf = vbuf + 2 * n;                   // 2 x n
    auto bar = [&]() {
        if (C > 1) cluster_barrier();
        else __syncthreads();
    };
    // load the owned rows; off-diagonal sum of squares over them
    double off = 0.0;
    for (int li = wl; li < nloc; li += NW) {
        const int i = (int)rank + C * li;
        for (int j = lane; j < n; j += 32) {
            const double v = a.K[(size_t)i * a.ldk + j];
            A[(size_t)li * n + j] = v;
            if (j != i) off += v * v;
        }
    }
    for (int j = tid; j < 4 * n; j += NTHR) vbuf[j] = 0.0;
    if (tid < 4) (&s_sc[0][0])[tid] = 0.0;
    off = block_sum(off, red);
    if (tid == 0)
        for (int r = 0; r < C; ++r) (C > 1 ? cluster_map(s_off, r) : s_off)[rank] = off;
    bar();
    off = 0.0;
    for (int r = 0; r < C; ++r) off += s_off[r];  // same order on every CTA
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {
        const double ot = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = ot * ot;
    }
    if (!(off > tol_sq) || n == 1) {  // the reference's Jacobi would not rotate at all (la_core.cpp:33)
        for (int li = wl; li < nloc; li += NW)
            if (lane == 0) {
                const int i = (int)rank + C * li;
                a.d[i] = A[(size_t)li * n + i];
                if (i + 1 < n) a.e[i] = 0.0;
            }
        if (rank == 0 && tid == 0) *a.trivial = 1;
        return;
    }
    if (rank == 0 && tid == 0) *a.trivial = 0;
    for (int k = 0; k + 1 < n; ++k) {
        const int cur = k & 1, prv = cur ^ 1;
        const double* vp = vbuf + prv * n;
        const double* pp = pbuf + prv * n;
        TPROBE(0, tid == 0)
        // ---- S1: owner warp of row k
        if ((int)rank == k % C && wl == (k / C) % NW) {
            double dsum = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j >= k && j < n) dsum += pp[j] * vp[j];
            }
            dsum = warp_sum(dsum);
            const double cprev = 0.5 * s_sc[prv][0] * dsum;
            const double vk = vp[k], wk = pp[k] - cprev * vp[k];
            double* Ak = A + (size_t)(k / C) * n;
            double x[NT];
            double xs = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                x[t] = 0.0;
                if (j >= k && j < n) {
                    const double vj = vp[j];
                    const double val = Ak[j] - vk * (pp[j] - cprev * vj) - wk * vj;
                    Ak[j] = val;
                    x[t] = val;
                    if (j >= k + 2) xs += val * val;
                }
            }
            xs = warp_sum(xs);
            __syncwarp();
            const double alpha = Ak[k + 1];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xs > 0.0) {  // reciprocals without the IEEE-divide slow path (~1 ulp, 55 vs 131 cycles)
                beta = -copysign(sqrt(alpha * alpha + xs), alpha);
                tau = (beta - alpha) * fast_rcp(beta);
                scal = fast_rcp(alpha - beta);
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j >= k + 1 && j < n) {
                    const double v = (j == k + 1) ? 1.0 : x[t] * scal;
                    for (int r = 0; r < C; ++r) (C > 1 ? cluster_map(vbuf, r) : vbuf)[cur * n + j] = v;
                    a.vh[(size_t)k * n + j] = v;
                }
            }
            if (lane == 0) {
                for (int r = 0; r < C; ++r) {
                    double* sc = C > 1 ? cluster_map(&s_sc[cur][0], r) : &s_sc[cur][0];
                    sc[0] = tau;
                    sc[1] = cprev;
                }
                a.d[k] = Ak[k];
                a.e[k] = beta;
                a.tau[k] = tau;
            }
            TPROBE(1, lane == 0)
        }
        bar();
        TPROBE(2, tid == 0)
        // ---- S2: rows i > k: update of step k-1, p_k = tau_k A v_k
        {
            const double tau = s_sc[cur][0], cprev = s_sc[cur][1];
            const double* vc = vbuf + cur * n;
            double rv[NT], rw[NT], rc[NT];
            const int t0 = (k + 1) >> 5;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                const bool on = t >= t0 && j > k && j < n;
                rv[t] = on ? vp[j] : 0.0;
                rw[t] = on ? pp[j] - cprev * vp[j] : 0.0;
                rc[t] = on ? vc[j] : 0.0;
            }
            int li = wl;
            {  // first local row index with global row > k owned by this warp
                const int need = (k + 1 - (int)rank + C - 1) / C;  // smallest li with rank + C li > k
                if (need > li) li += (need - li + NW - 1) / NW * NW;
            }
            // four rows per pass: independent accumulators, one 6-shuffle transposed reduction
            for (; li < nloc; li += 4 * NW) {
                double sr[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int lr = li + r * NW;
                    sr[r] = 0.0;
                    if (lr < nloc) {
                        const int i = (int)rank + C * lr;
                        const double vi = vp[i], wi = pp[i] - cprev * vp[i];
                        double* Ai = A + (size_t)lr * n;
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            const int j = 32 * t + lane;
                            if (t >= t0 && j > k && j < n) {
                                const double val = Ai[j] - vi * rw[t] - wi * rv[t];
                                Ai[j] = val;
                                sr[r] += val * rc[t];
                            }
                        }
                    }
                }
                const bool h16 = lane & 16, h8 = lane & 8;
                double a0 = h16 ? sr[2] : sr[0], a1 = h16 ? sr[3] : sr[1];
                a0 += __shfl_xor_sync(0xffffffffu, h16 ? sr[0] : sr[2], 16);
                a1 += __shfl_xor_sync(0xffffffffu, h16 ? sr[1] : sr[3], 16);
                double c0 = h8 ? a1 : a0;
                c0 += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 4);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 2);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 1);
                // lanes 0, 8, 16, 24 hold rows 0..3; lanes +1..+C-1 of each group fan out to the cluster
                const int r = lane >> 3, sub = lane & 7;
                const int lr = li + r * NW;
                if (lr < nloc) {
                    const int i = (int)rank + C * lr;
                    for (int q = sub; q < C; q += 8) (C > 1 ? cluster_map(pbuf, q) : pbuf)[cur * n + i] = c0 * tau;
                }
            }
        }
        TPROBE(3, tid == 0)
        TPROBE(4, tid == 32 * (NW - 1))
        bar();
        TPROBE(5, tid == 0)
    }
    if ((int)rank == (n - 1) % C && tid == 0) {
        a.d[n - 1] = A[(size_t)((n - 1) / C) * n + n - 1];
        a.tau[n - 1] = 0.0;
        if (n >= 2) a.tau[n - 2] = 0.0;
    }
}

// Register-resident variant of tridiag_rows_kernel (same row distribution, same algebra and
// summation order, same two barriers per step): each warp keeps its rows of the matrix in
// registers, A[s][t] = row (rank + C (wl + NW s)), columns 32 t + lane. The trailing update
// of S2 was bound by shared-memory traffic (every live element loaded and stored once per
// step, tools/tri_probe: S2 ~2.5x the S1 time at n = 100-160); here it is register FMAs.
// RPW slots x NT chunks <= 32 doubles per lane: n <= 128 on 1 CTA, n <= 256 on a 4-CTA
// cluster, n <= 512 on 16 CTAs. Shared memory only holds the v / p exchange vectors.
template <int C, int NT, int RPW>
__global__ void __launch_bounds__(512) tridiag_regs_kernel(TriRowsArgs ra) {
    pdl_entry();
    constexpr int NTHR = 512, NW = NTHR / 32;
    extern __shared__ double sm[];
    __shared__ double s_sc[2][2];  // [k & 1] = {tau_k, c_{k-1}}
    __shared__ double s_off[16];
    __shared__ double red[32];
    const TriArgs& a = ra.a;
    const int n = a.n;
    const unsigned rank = C > 1 ? cluster_rank() : 0u;
    const int tid = threadIdx.x, lane = tid & 31, wl = tid >> 5;
    const int nloc = (n - (int)rank + C - 1) / C;  // rows rank, rank + C, ...
    double* vbuf = sm;          // 2 x n
    double* pbuf = sm + 2 * n;  // 2 x n
    auto bar = [&]() {
        if (C > 1) cluster_barrier();
        else __syncthreads();
    };
    double A[RPW][NT];
    double off = 0.0;
#pragma unroll
    for (int s = 0; s < RPW; ++s) {
        const int li = wl + NW * s;
        const int i = (int)rank + C * li;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int j = 32 * t + lane;
            const bool on = li < nloc && j < n;
            const double v = on ? a.K[(size_t)i * a.ldk + j] : 0.0;
            A[s][t] = v;
            if (on && j != i) off += v * v;
        }
    }
    for (int j = tid; j < 4 * n; j += NTHR) vbuf[j] = 0.0;
    if (tid < 4) (&s_sc[0][0])[tid] = 0.0;
    off = block_sum(off, red);
    if (tid == 0)
        for (int r = 0; r < C; ++r) (C > 1 ? cluster_map(s_off, r) : s_off)[rank] = off;
    bar();
    off = 0.0;
    for (int r = 0; r < C; ++r) off += s_off[r];  // same order on every CTA
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {
        const double ot = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = ot * ot;
    }
    if (!(off > tol_sq) || n == 1) {  // the reference's Jacobi would not rotate at all (la_core.cpp:33)
#pragma unroll
        for (int s = 0; s < RPW; ++s) {
            const int li = wl + NW * s;
            const int i = (int)rank + C * li;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (li < nloc && 32 * t + lane == i) {
                    a.d[i] = A[s][t];
                    if (i + 1 < n) a.e[i] = 0.0;
                }
        }
        if (rank == 0 && tid == 0) *a.trivial = 1;
        return;
    }
    if (rank == 0 && tid == 0) *a.trivial = 0;
    for (int k = 0; k + 1 < n; ++k) {
        const int cur = k & 1, prv = cur ^ 1;
        const double* vp = vbuf + prv * n;
        const double* pp = pbuf + prv * n;
        TPROBE(0, tid == 0)
        // ---- S1: owner warp of row k (slot sk of warp (k / C) % NW on CTA k % C)
        if ((int)rank == k % C && wl == (k / C) % NW) {
            const int sk = (k / C) / NW;
            double dsum = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j >= k && j < n) dsum += pp[j] * vp[j];
            }
            dsum = warp_sum(dsum);
            const double cprev = 0.5 * s_sc[prv][0] * dsum;
            const double vk = vp[k], wk = pp[k] - cprev * vp[k];
            double x[NT];
            double xs = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                double ak = 0.0;
#pragma unroll
                for (int s = 0; s < RPW; ++s)
                    if (s == sk) ak = A[s][t];
                x[t] = 0.0;
                if (j >= k && j < n) {
                    const double vj = vp[j];
                    const double val = ak - vk * (pp[j] - cprev * vj) - wk * vj;
                    x[t] = val;
                    if (j >= k + 2) xs += val * val;
                }
            }
            xs = warp_sum(xs);
            double xa = 0.0, xd = 0.0;  // columns k + 1 and k of the updated row, on their lanes
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (t == (k + 1) >> 5) xa = x[t];
                if (t == k >> 5) xd = x[t];
            }
            const double alpha = __shfl_sync(0xffffffffu, xa, (k + 1) & 31);
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xs > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + xs), alpha);
                tau = (beta - alpha) * fast_rcp(beta);
                scal = fast_rcp(alpha - beta);
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j >= k + 1 && j < n) {
                    const double v = (j == k + 1) ? 1.0 : x[t] * scal;
                    for (int r = 0; r < C; ++r) (C > 1 ? cluster_map(vbuf, r) : vbuf)[cur * n + j] = v;
                    a.vh[(size_t)k * n + j] = v;
                }
            }
            if (lane == (k & 31)) a.d[k] = xd;
            if (lane == 0) {
                for (int r = 0; r < C; ++r) {
                    double* sc = C > 1 ? cluster_map(&s_sc[cur][0], r) : &s_sc[cur][0];
                    sc[0] = tau;
                    sc[1] = cprev;
                }
                a.e[k] = beta;
                a.tau[k] = tau;
            }
            TPROBE(1, lane == 0)
        }
        bar();
        TPROBE(2, tid == 0)
        // ---- S2: rows i > k: update of step k-1, p_k = tau_k A v_k (groups of four slots)
        {
            const double tau = s_sc[cur][0], cprev = s_sc[cur][1];
            const double* vc = vbuf + cur * n;
#pragma unroll
            for (int g = 0; g < (RPW + 3) / 4; ++g) {
                const int li_hi = wl + NW * min(4 * g + 3, RPW - 1);  // last slot of the group
                const int li_lo = wl + NW * 4 * g;
                if (li_lo >= nloc || (int)rank + C * li_hi <= k) continue;  // warp-uniform
                double vi[4], wi[4], sr[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int li = wl + NW * (4 * g + r);
                    const int i = (int)rank + C * li;
                    const bool live = 4 * g + r < RPW && li < nloc && i > k;
                    vi[r] = live ? vp[i] : 0.0;
                    wi[r] = live ? pp[i] - cprev * vp[i] : 0.0;
                    sr[r] = 0.0;
                }
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int j = 32 * t + lane;
                    if (j > k && j < n) {
                        const double rv = vp[j], rw = pp[j] - cprev * vp[j], rc = vc[j];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int s = 4 * g + r;
                            if (s < RPW) {
                                const int li = wl + NW * s;
                                if (li < nloc && (int)rank + C * li > k) {
                                    const double val = A[s][t] - vi[r] * rw - wi[r] * rv;
                                    A[s][t] = val;
                                    sr[r] += val * rc;
                                }
                            }
                        }
                    }
                }
                const bool h16 = lane & 16, h8 = lane & 8;
                double a0 = h16 ? sr[2] : sr[0], a1 = h16 ? sr[3] : sr[1];
                a0 += __shfl_xor_sync(0xffffffffu, h16 ? sr[0] : sr[2], 16);
                a1 += __shfl_xor_sync(0xffffffffu, h16 ? sr[1] : sr[3], 16);
                double c0 = h8 ? a1 : a0;
                c0 += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 4);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 2);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 1);
                const int r = lane >> 3, sub = lane & 7;
                const int s = 4 * g + r;
                const int li = wl + NW * s;
                const int i = (int)rank + C * li;
                if (s < RPW && li < nloc && i > k)
                    for (int q = sub; q < C; q += 8) (C > 1 ? cluster_map(pbuf, q) : pbuf)[cur * n + i] = c0 * tau;
            }
        }
        TPROBE(3, tid == 0)
        TPROBE(4, tid == 32 * (NW - 1))
        bar();
        TPROBE(5, tid == 0)
    }
    // the last diagonal entry, from the register of its owner lane
#pragma unroll
    for (int s = 0; s < RPW; ++s) {
        const int li = wl + NW * s;
        const int i = (int)rank + C * li;
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (i == n - 1 && li < nloc && 32 * t + lane == n - 1) {
                a.d[n - 1] = A[s][t];
                a.tau[n - 1] = 0.0;
                if (n >= 2) a.tau[n - 2] = 0.0;
            }
    }
}

// Sturm count: eigenvalues of T smaller than x (dlaebz recurrence with pivmin guard).
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    int c = q < 0.0;
    for (int j = 1; j < n; ++j) {
        q = (d[j] - x) - e2[j - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

// Warp per eigenvalue: the top `nval` eigenvalues, written in descending order. Each lane
// runs kShifts interleaved Sturm chains (independent divides overlap), so one step splits
// the bracket into 32 * kShifts + 1 pieces (~7 bits per step instead of 5).
#ifndef SFDG_BISECT_SHIFTS
#define SFDG_BISECT_SHIFTS 2  // measured: 1 -> 49/91 us, 2 -> 48/88, 3 -> 52/96, 4 -> 106/206 (n = 100 / 200)
#endif
constexpr int kShifts = SFDG_BISECT_SHIFTS;
__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                              const int* __restrict__ trivial, double* __restrict__ lam_desc) {
    pdl_entry();
    extern __shared__ double sh[];
    double* d = sh;
    double* e2 = sh + n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        d[j] = dg[j];
        e2[j] = j + 1 < n ? eg[j] * eg[j] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // descending index
    if (t >= nval) return;
    if (*trivial) {  // diagonal: eigenvalues are the sorted diagonal (stable, descending)
        for (int i = lane; i < n; i += 32) {
            int r = 0;
            for (int j = 0; j < n; ++j) r += (d[j] > d[i] || (d[j] == d[i] && j < i));
            if (r == t) lam_desc[t] = d[i];
        }
        return;
    }
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double r = (j > 0 ? sqrt(e2[j - 1]) : 0.0) + (j + 1 < n ? sqrt(e2[j]) : 0.0);
        lo = fmin(lo, d[j] - r);
        hi = fmax(hi, d[j] + r);
        emax = fmax(emax, e2[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 1e3;
    lo -= 2.0 * 2.2e-16 * tnorm + pivmin;
    hi += 2.0 * 2.2e-16 * tnorm + pivmin;
    const int want = n - 1 - t;  // ascending index of the eigenvalue
    constexpr int P = 32 * kShifts;
    constexpr double inv = 1.0 / (P + 1);
    double a = lo, b = hi;  // count(a) <= want < count(b)
    for (int it = 0; it < 40; ++it) {
        if (b - a <= 2.0 * 2.2e-16 * fmax(fabs(a), fabs(b)) + pivmin) break;
        const double w = b - a;
        double x[kShifts], q[kShifts];
        int c[kShifts];
#pragma unroll
        for (int s = 0; s < kShifts; ++s) {
            x[s] = a + w * ((double)(lane * kShifts + s + 1) * inv);
            q[s] = d[0] - x[s];
            if (fabs(q[s]) < pivmin) q[s] = -pivmin;
            c[s] = q[s] < 0.0;
        }
        for (int j = 1; j < n; ++j) {
            const double dj = d[j], ej = e2[j - 1];
#pragma unroll
            for (int s = 0; s < kShifts; ++s) {
                q[s] = fma(-ej, fast_rcp(q[s]), dj - x[s]);
                if (fabs(q[s]) < pivmin) q[s] = -pivmin;
                c[s] += q[s] < 0.0;
            }
        }
        int f = kShifts;  // first local shift past the eigenvalue
#pragma unroll
        for (int s = kShifts - 1; s >= 0; --s)
            if (c[s] > want) f = s;
        const unsigned above = __ballot_sync(0xffffffffu, f < kShifts);
        const int L = above ? __ffs(above) - 1 : 32;
        const int fL = __shfl_sync(0xffffffffu, f, L & 31);
        const int m = L < 32 ? L * kShifts + fL : P;  // first point index with count > want
        const double na = m > 0 ? a + w * ((double)m * inv) : a;
        const double nb = m < P ? a + w * ((double)(m + 1) * inv) : b;
        a = na;
        b = nb;
    }
    if (lane == 0) lam_desc[t] = 0.5 * (a + b);
}

// Thread per eigenvalue: 3 steps of inverse iteration with a partially pivoted LU of
// (T - lambda I) (LAPACK dgttrf/dgttrs algebra); X is n x ldx (column t = vector t).
// T is staged in shared memory; the per-thread LU bands live in shared memory (or global
// for large n) interleaved by thread; the solves carry their recurrences in registers and
// multiply by stored pivot reciprocals, so the only divides are the n of the factorisation.
__global__ void inviter_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                               const double* __restrict__ lam, const int* __restrict__ trivial,
                               double* __restrict__ X, int ldx, double* __restrict__ work_g,
                               const int* __restrict__ need) {
    pdl_entry();
    extern __shared__ double sh_inv[];
    __shared__ double s_tn;
    double* d = sh_inv;
    double* e = sh_inv + n;
    const int nb = blockDim.x;
    for (int j = threadIdx.x; j < n; j += nb) {
        d[j] = dg[j];
        e[j] = j + 1 < n ? eg[j] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tn = 0.0;
        for (int j = 0; j < n; ++j) tn = fmax(tn, fabs(d[j]) + (j > 0 ? fabs(e[j - 1]) : 0.0) + fabs(e[j]));
        s_tn = tn;
    }
    __syncthreads();
    const int t = blockIdx.x * nb + threadIdx.x;
    if (t >= nval) return;
    if (need && !need[t]) return;  // already done by the twisted factorisation
    if (*trivial) {  // identity eigenvectors in the stable descending order of the diagonal
        int idx = 0;
        for (int i = 0; i < n; ++i) {
            int r = 0;
            for (int j = 0; j < n; ++j) r += (d[j] > d[i] || (d[j] == d[i] && j < i));
            if (r == t) idx = i;
        }
        for (int i = 0; i < n; ++i) X[(size_t)i * ldx + t] = (i == idx) ? 1.0 : 0.0;
        return;
    }
    // interleaved per-thread arrays: element j of thread s at [j * S + s]
    const bool glob = work_g != nullptr;
    const int S = glob ? gridDim.x * nb : nb;
    const int slot = glob ? t : threadIdx.x;
    double* base = glob ? work_g : sh_inv + 2 * n;
    double* Ui = base;                      // 1 / diag(U)
    double* U1 = base + (size_t)n * S;      // 1st super
    double* U2 = base + 2 * (size_t)n * S;  // 2nd super (0 unless a swap)
    double* Lm = base + 3 * (size_t)n * S;  // multipliers
    double* x = base + 4 * (size_t)n * S;
#define AT(arr, j) arr[(size_t)(j) * S + slot]
    const double tiny = 2.2e-16 * fmax(s_tn, 1e-300);
    const double l = lam[t];
    unsigned swapw = 0;  // row-swap flags of the current 32-row word
    double a = d[0] - l;
    double b = n > 1 ? e[0] : 0.0;
    unsigned* flags = reinterpret_cast<unsigned*>(base + 5 * (size_t)n * S);  // ceil(n/32) words per thread
    for (int j = 0; j + 1 < n; ++j) {
        const double c = e[j];
        const double dn = d[j + 1] - l;
        const double bn = j + 2 < n ? e[j + 1] : 0.0;
        double u0;
        if (fabs(a) >= fabs(c)) {
            const double r = a != 0.0 ? fast_rcp(a) : 0.0;
            const double m = c * r;
            u0 = a;
            AT(U1, j) = b;
            AT(U2, j) = 0.0;
            AT(Lm, j) = m;
            a = dn - m * b;
            b = bn;
        } else {
            const double m = a * fast_rcp(c);
            u0 = c;
            AT(U1, j) = dn;
            AT(U2, j) = bn;
            AT(Lm, j) = m;
            swapw |= 1u << (j & 31);
            a = b - m * dn;
            b = -m * bn;
        }
        if (fabs(u0) < tiny) u0 = u0 < 0.0 ? -tiny : tiny;
        AT(Ui, j) = fast_rcp(u0);
        if ((j & 31) == 31) {
            flags[(size_t)(j >> 5) * S + slot] = swapw;
            swapw = 0;
        }
    }
    if (n >= 1) {
        if (((n - 2) & 31) != 31 && n >= 2) flags[(size_t)((n - 2) >> 5) * S + slot] = swapw;
        double u0 = a;
        if (fabs(u0) < tiny) u0 = u0 < 0.0 ? -tiny : tiny;
        AT(Ui, n - 1) = 1.0 / u0;
    }
    // deterministic distinct start vector
    uint64_t sd = 0x9E3779B97F4A7C15ull * (uint64_t)(t + 1);
    for (int j = 0; j < n; ++j) {
        sd ^= sd >> 12;
        sd ^= sd << 25;
        sd ^= sd >> 27;
        AT(x, j) = (double)((sd * 2685821657736338717ull) >> 11) * 0x1.0p-53 - 0.5;
    }
    double scale = 1.0;
    for (int it = 0; it < 3; ++it) {
        // forward: apply P and L (scaled by the previous normalisation). The next step's
        // operands are loaded before this step's store (software pipelining: the store/load
        // pair on x would otherwise serialise every step on shared-memory latency).
        double xj = AT(x, 0) * scale;
        unsigned fw = flags[slot];
        double xn_n = n > 1 ? AT(x, 1) * scale : 0.0, m_n = n > 1 ? AT(Lm, 0) : 0.0;
        for (int j = 0; j + 1 < n; ++j) {
            const double xn = xn_n, m = m_n;
            if (j + 2 < n) {
                xn_n = AT(x, j + 2) * scale;
                m_n = AT(Lm, j + 1);
            }
            double keep, carry;
            if ((fw >> (j & 31)) & 1u) {
                keep = xn;
                carry = xj - m * xn;
            } else {
                keep = xj;
                carry = xn - m * xj;
            }
            AT(x, j) = keep;
            xj = carry;
            if ((j & 31) == 31) fw = flags[(size_t)((j + 1) >> 5) * S + slot];
        }
        // backward: U x = y, with the squared norm on the side
        double x1 = xj * AT(Ui, n - 1);
        AT(x, n - 1) = x1;
        double nrm = x1 * x1;
        double x0 = x1, x2 = 0.0;
        if (n >= 2) {
            x0 = (AT(x, n - 2) - AT(U1, n - 2) * x1) * AT(Ui, n - 2);
            AT(x, n - 2) = x0;
            nrm += x0 * x0;
            x2 = x1;
            x1 = x0;
        }
        if (n >= 3) {
            double bx = AT(x, n - 3), b1 = AT(U1, n - 3), b2 = AT(U2, n - 3), bi = AT(Ui, n - 3);
            for (int j = n - 3; j >= 0; --j) {
                const double cx = bx, c1 = b1, c2 = b2, ci = bi;
                if (j > 0) {
                    bx = AT(x, j - 1);
                    b1 = AT(U1, j - 1);
                    b2 = AT(U2, j - 1);
                    bi = AT(Ui, j - 1);
                }
                const double v = (cx - c1 * x1 - c2 * x2) * ci;
                AT(x, j) = v;
                nrm += v * v;
                x2 = x1;
                x1 = v;
            }
        }
        scale = 1.0 / sqrt(nrm);
    }
    for (int j = 0; j < n; ++j) X[(size_t)j * ldx + t] = AT(x, j) * scale;
#undef AT
}

// Eigenvectors by twisted factorisations (Dhillon's "getvec"): for each eigenvalue l the
// stationary forward factorisation T - l I = L+ D+ L+^T and the backward one U- D- U-^T
// run at once on a lane pair (same recurrence q' = (a - l) - b^2 / q, indexed up vs down);
// the twist r = argmin |gamma_k| (gamma_k = D+_k + D-_k - (a_k - l)) then gives the vector
// z_r = 1, z_i = -L_i z_{i+1} above and z_i = -U_{i-1} z_{i-1} below. One pass, no
// iteration: with l accurate to bisection precision the residual is |gamma_r| / |z| ~ u |T|.
// kEPW eigenvalues per warp (lane 2p forward, 2p+1 backward); the factors live in shared
// memory, four n-vectors per eigenvalue.
constexpr int kEPW = 16;
__global__ void twisted_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                               const double* __restrict__ lam, const int* __restrict__ trivial,
                               double* __restrict__ X, int ldx, int* __restrict__ need) {
    pdl_entry();
    extern __shared__ double tw_s[];
    double* a = tw_s;          // n diagonal
    double* b2 = tw_s + n;     // n-1 squared off-diagonals
    double* bo = tw_s + 2 * n; // n-1 off-diagonals
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        a[j] = dg[j];
        const double e = j + 1 < n ? eg[j] : 0.0;
        bo[j] = e;
        b2[j] = e * e;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int pr = lane >> 1, dir = lane & 1;
    const int t = (blockIdx.x * nw + w) * kEPW + pr;
    const bool act = pr < kEPW && t < nval;
    if (*trivial) {  // identity vectors in the stable descending order of the diagonal
        if (act && dir == 0) {
            int idx = 0;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int j = 0; j < n; ++j) r += (a[j] > a[i] || (a[j] == a[i] && j < i));
                if (r == t) idx = i;
            }
            for (int i = 0; i < n; ++i) X[(size_t)i * ldx + t] = (i == idx) ? 1.0 : 0.0;
        }
        return;
    }
    // per-eigenvalue factor storage: D (n) and 1/D (n) for this lane's direction
    double* base = tw_s + 3 * n + (size_t)(w * kEPW + (pr < kEPW ? pr : 0)) * 4 * n;
    double* D = base + (size_t)dir * 2 * n;  // D+ (dir 0) or D- (dir 1)
    double* R = D + n;                       // 1/D+ or 1/D-
    double tn = 0.0, emax = 0.0;
    for (int j = 0; j < n; ++j) {
        tn = fmax(tn, fabs(a[j]) + (j > 0 ? fabs(bo[j - 1]) : 0.0) + fabs(bo[j]));
        emax = fmax(emax, b2[j]);
    }
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 1e3;
    const double l = act ? lam[t] : 0.0;
    // both factorisations: step s computes index j from j -/+ 1
    {
        int j = dir ? n - 1 : 0;
        double q = a[j] - l;
        if (fabs(q) < pivmin) q = -pivmin;
        D[j] = q;
        for (int s = 0; s + 1 < n; ++s) {
            const int jn = dir ? n - 2 - s : s + 1;
            const int o = dir ? n - 2 - s : s;  // off-diagonal between j and jn
            const double r = fast_rcp(q);
            R[j] = r;
            q = fma(-b2[o], r, a[jn] - l);
            if (fabs(q) < pivmin) q = -pivmin;
            D[jn] = q;
            j = jn;
        }
        R[j] = fast_rcp(q);
    }
    __syncwarp();
    // twist: argmin |gamma_k| over the pair (lane 2p: k < n/2, lane 2p+1: k >= n/2)
    const double* Dp = base;
    const double* Dm = base + 2 * n;
    int kbest = -1;
    double gbest = 1e300;
    const int k0 = dir ? n / 2 : 0, k1 = dir ? n : n / 2;
    for (int k = k0; k < k1; ++k) {
        const double g = fabs(Dp[k] + Dm[k] - (a[k] - l));
        if (g < gbest) {
            gbest = g;
            kbest = k;
        }
    }
    {
        const double go = __shfl_xor_sync(0xffffffffu, gbest, 1);
        const int ko = __shfl_xor_sync(0xffffffffu, kbest, 1);
        if (go < gbest || (go == gbest && ko >= 0 && (kbest < 0 || ko < kbest))) {
            gbest = go;
            kbest = ko;
        }
    }
    const int r = kbest < 0 ? 0 : kbest;
    __syncwarp();
    // z into the D+ slot (no longer needed): up from r on lane 2p, down from r on lane 2p+1
    double* z = base;
    const double* Rp = base + n;
    const double* Rm = base + 3 * n;
    double nrm = 0.0;
    {
        double zc = 1.0;
        const int len = dir ? n - 1 - r : r;
        for (int s = 0; s < n; ++s) {
            if (s < len) {
                const int i = dir ? r + 1 + s : r - 1 - s;
                // z_i = -L_i z_{i+1} = -b_i/D+_i z_{i+1}  |  z_i = -U_{i-1} z_{i-1} = -b_{i-1}/D-_i z_{i-1}
                zc = dir ? -bo[i - 1] * Rm[i] * zc : -bo[i] * Rp[i] * zc;
                nrm = fma(zc, zc, nrm);
                z[i] = zc;  // lane 2p writes i < r, lane 2p+1 writes i > r: disjoint
            }
        }
    }
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
    nrm += 1.0;  // z_r
    if (dir == 0) z[r] = 1.0;
    __syncwarp();
    const double inv = 1.0 / sqrt(nrm);
    if (act)
        for (int i = dir; i < n; i += 2) X[(size_t)i * ldx + t] = z[i] * inv;
    // eigenvalues in a cluster (gap <= the cluster kernel's 1e-6 |T|) need distinct start
    // vectors for the Rayleigh-Ritz step, and an overflowed twist needs a redo: both go to
    // inverse iteration (inviter_kernel with this mask)
    if (act && dir == 0) {
        const double ctol = 1e-6 * tn;
        const bool clus = (t > 0 && lam[t - 1] - l <= ctol) || (t + 1 < nval && l - lam[t + 1] <= ctol);
        need[t] = (clus || !isfinite(inv) || !(nrm < 1e300)) ? 1 : 0;
    }
}

// Warp per cluster start: orthonormalise the cluster's vectors (MGS twice) and resolve the
// individual eigenvectors by Rayleigh-Ritz (cyclic Jacobi on the c x c projected matrix).
constexpr int kMaxCluster = 32;
__global__ void cluster_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                               double* __restrict__ lam, const int* __restrict__ trivial, double* __restrict__ X,
                               int ldx, int* __restrict__ fallback) {
    pdl_entry();
    __shared__ double Cm[1][kMaxCluster * kMaxCluster];
    __shared__ double Vm[1][kMaxCluster * kMaxCluster];
    const int lane = threadIdx.x & 31, w = 0;
    const int t0 = blockIdx.x;
    if (t0 >= nval || *trivial) return;
    double tn = 0.0;
    for (int j = 0; j < n; ++j) tn = fmax(tn, fabs(dg[j]) + (j > 0 ? fabs(eg[j - 1]) : 0.0) + (j + 1 < n ? fabs(eg[j]) : 0.0));
    const double ctol = 1e-6 * tn;  // inverse iteration orthogonality ~ u |T| / gap <= 2e-10 outside clusters
    if (t0 > 0 && lam[t0 - 1] - lam[t0] <= ctol) return;  // not a cluster start
    int c = 1;
    while (t0 + c < nval && lam[t0 + c - 1] - lam[t0 + c] <= ctol) ++c;
    if (c == 1) return;
    if (c > kMaxCluster) {
        if (lane == 0) atomicExch(fallback, 1);  // eigh() then runs the Jacobi solver instead
        return;
    }
    // MGS, two passes. The cluster's inverse-iteration vectors must span its invariant
    // subspace: when one of them is (nearly) dependent on the earlier ones -- e.g. equal
    // eigenvalues from different diagonal blocks of a split T all converge to the same
    // vector -- the normalised remainder is rounding noise, not an eigenvector. That case is
    // handed to the Jacobi solver (eigh() runs it when *fallback is set).
    for (int pass = 0; pass < 2; ++pass)
        for (int a = 0; a < c; ++a) {
            double s0 = 0.0;
            if (pass == 0) {
                for (int j = lane; j < n; j += 32) s0 += X[(size_t)j * ldx + t0 + a] * X[(size_t)j * ldx + t0 + a];
                s0 = warp_sum(s0);
            }
            for (int b = 0; b < a; ++b) {
                double s = 0.0;
                for (int j = lane; j < n; j += 32) s += X[(size_t)j * ldx + t0 + a] * X[(size_t)j * ldx + t0 + b];
                s = warp_sum(s);
                for (int j = lane; j < n; j += 32) X[(size_t)j * ldx + t0 + a] -= s * X[(size_t)j * ldx + t0 + b];
                __syncwarp();
            }
            double s = 0.0;
            for (int j = lane; j < n; j += 32) s += X[(size_t)j * ldx + t0 + a] * X[(size_t)j * ldx + t0 + a];
            s = warp_sum(s);
            if (pass == 0 && !(s > 1e-6 * s0)) {  // lost > 99.9% of its norm: dependent
                if (lane == 0) atomicExch(fallback, 1);
                return;
            }
            s = 1.0 / sqrt(s);
            for (int j = lane; j < n; j += 32) X[(size_t)j * ldx + t0 + a] *= s;
            __syncwarp();
        }
    // C = X_c^T T X_c
    double* C = Cm[w];
    double* V = Vm[w];
    for (int a = 0; a < c; ++a)
        for (int b = a; b < c; ++b) {
            double s = 0.0;
            for (int j = lane; j < n; j += 32) {
                double tx = dg[j] * X[(size_t)j * ldx + t0 + b];
                if (j > 0) tx += eg[j - 1] * X[(size_t)(j - 1) * ldx + t0 + b];
                if (j + 1 < n) tx += eg[j] * X[(size_t)(j + 1) * ldx + t0 + b];
                s += X[(size_t)j * ldx + t0 + a] * tx;
            }
            s = warp_sum(s);
            if (lane == 0) {
                C[a * c + b] = s;
                C[b * c + a] = s;
            }
        }
    for (int e = lane; e < c * c; e += 32) V[e] = (e / c == e % c) ? 1.0 : 0.0;
    __syncwarp();
    // cyclic Jacobi on C (lane 0; c <= 48)
    if (lane == 0) {
        for (int sweep = 0; sweep < 30; ++sweep) {
            double offn = 0.0, dn = 0.0;
            for (int p = 0; p < c; ++p)
                for (int q = 0; q < c; ++q) (p == q ? dn : offn) += C[p * c + q] * C[p * c + q];
            if (offn <= 1e-30 * dn) break;
            for (int p = 0; p + 1 < c; ++p)
                for (int q = p + 1; q < c; ++q) {
                    const double apq = C[p * c + q];
                    if (apq == 0.0) continue;
                    const double th = (C[q * c + q] - C[p * c + p]) / (2.0 * apq);
                    const double tt = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                    const double cc = 1.0 / sqrt(tt * tt + 1.0), ss = tt * cc;
                    for (int i = 0; i < c; ++i) {
                        const double x1 = C[i * c + p], x2 = C[i * c + q];
                        C[i * c + p] = cc * x1 - ss * x2;
                        C[i * c + q] = ss * x1 + cc * x2;
                    }
                    for (int j = 0; j < c; ++j) {
                        const double x1 = C[p * c + j], x2 = C[q * c + j];
                        C[p * c + j] = cc * x1 - ss * x2;
                        C[q * c + j] = ss * x1 + cc * x2;
                    }
                    for (int i = 0; i < c; ++i) {
                        const double x1 = V[i * c + p], x2 = V[i * c + q];
                        V[i * c + p] = cc * x1 - ss * x2;
                        V[i * c + q] = ss * x1 + cc * x2;
                    }
                }
        }
        // order the Ritz pairs descending (insertion sort of columns)
        for (int i = 1; i < c; ++i)
            for (int j = i; j > 0 && C[j * c + j] > C[(j - 1) * c + (j - 1)]; --j) {
                const double tmp = C[j * c + j];
                C[j * c + j] = C[(j - 1) * c + j - 1];
                C[(j - 1) * c + j - 1] = tmp;
                for (int r = 0; r < c; ++r) {
                    const double t2 = V[r * c + j];
                    V[r * c + j] = V[r * c + j - 1];
                    V[r * c + j - 1] = t2;
                }
            }
    }
    __syncwarp();
    // X_c <- X_c V, Ritz values back into lam
    for (int j = lane; j < n; j += 32) {
        double row[kMaxCluster];
        for (int a = 0; a < c; ++a) row[a] = X[(size_t)j * ldx + t0 + a];
        for (int b = 0; b < c; ++b) {
            double s = 0.0;
            for (int a = 0; a < c; ++a) s += row[a] * V[a * c + b];
            X[(size_t)j * ldx + t0 + b] = s;
        }
    }
    if (lane == 0)
        for (int a = 0; a < c; ++a) lam[t0 + a] = C[a * c + a];
}

// U = Q X with Q = H_0 H_1 ... H_{n-3}: apply reflectors last-to-first. Warp per column
// of X, the column in registers (lane owns rows lane + 32 t); the reflectors are staged
// through shared memory in chunks of R rows (coalesced), one block barrier per chunk.
template <int NT>
__global__ void __launch_bounds__(256) backtransform_kernel(const double* __restrict__ vh,
                                                            const double* __restrict__ tau, int n, int nval,
                                                            const int* __restrict__ trivial, double* __restrict__ X,
                                                            int ldx, int R) {
    pdl_entry();
    if (*trivial) return;
    extern __shared__ double vs[];  // R x n reflector rows, then R taus
    double* ts = vs + (size_t)R * n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = blockIdx.x * (blockDim.x >> 5) + w;
    const bool active = col < nval;
    double x[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int j = 32 * t + lane;
        x[t] = (active && j < n) ? X[(size_t)j * ldx + col] : 0.0;
    }
    for (int hi = n - 3; hi >= 0; hi -= R) {  // chunk of reflectors k = lo .. hi
        const int lo = max(0, hi - R + 1);
        __syncthreads();
        // one flat, independent load per element (the chunk arrives in a few L2 round trips)
        const int cnt = (hi - lo + 1) * n;
        const double* src = vh + (size_t)lo * n;
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) vs[e] = src[e];
        for (int r = threadIdx.x; r <= hi - lo; r += blockDim.x) ts[r] = tau[lo + r];
        __syncthreads();
        if (!active) continue;
        for (int k = hi; k >= lo; --k) {
            const double tk = ts[k - lo];
            if (tk == 0.0) continue;
            const double* v = vs + (size_t)(k - lo) * n;
            double s0 = 0.0, s1 = 0.0;  // two chains: the dot's FMA latency halves
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j > k && j < n) {
                    if (t & 1) s1 = fma(v[j], x[t], s1);
                    else s0 = fma(v[j], x[t], s0);
                }
            }
            const double s = warp_sum(s0 + s1) * tk;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = 32 * t + lane;
                if (j > k && j < n) x[t] -= s * v[j];
            }
        }
    }
    if (!active) return;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int j = 32 * t + lane;
        if (j < n) X[(size_t)j * ldx + col] = x[t];
    }
}

template <int NT>
void launch_backtransform(const double* vh, const double* tau, int n, int nval, const int* trivial, double* X,
                          int ldx, cudaStream_t st) {
    if (first_on_device((const void*)(backtransform_kernel<NT>))) {
        allow_max_dynamic_smem(backtransform_kernel<NT>);
    }
    const int R = std::max(1, std::min(n, (int)((96 * 1024) / (sizeof(double) * (n + 1)))));
    const size_t smem = (size_t)R * (n + 1) * sizeof(double);
    LAUNCH(backtransform_kernel<NT>, ceil_div(nval, 8), 256, smem, st, vh, tau, n, nval, trivial, X, ldx, R);
}

void backtransform(const double* vh, const double* tau, int n, int nval, const int* trivial, double* X, int ldx,
                   cudaStream_t st) {
    const int nt = (n + 31) / 32;
    if (nt <= 4) launch_backtransform<4>(vh, tau, n, nval, trivial, X, ldx, st);
    else if (nt <= 8) launch_backtransform<8>(vh, tau, n, nval, trivial, X, ldx, st);
    else if (nt <= 16) launch_backtransform<16>(vh, tau, n, nval, trivial, X, ldx, st);
    else launch_backtransform<32>(vh, tau, n, nval, trivial, X, ldx, st);
}

// Single-CTA fused tridiagonalisation on the packed lower triangle (row i holds columns
// 0..i at i(i+1)/2), for matrices whose full square would need a cluster (n ~ 167..220):
// the whole step stays inside one SM, with block barriers (~26 ns) instead of cluster
// barriers (~240 ns, tools/probe_cbar) and no DSMEM broadcasts. Step k (algebra of
// tridiag_rows_kernel / dsytd2, the update of step k-1 applied lazily):
//   S0 (all threads): p_{k-1,j} = tau_{k-1} (rowdot_j + sum_w colpart_w,j), fixed order.
//   S1 (warp 0): c_{k-1} = tau_{k-1}/2 p_{k-1}^T v_{k-1}, w_{k-1} = p_{k-1} - c v_{k-1};
//      apply update k-1 to column k; Householder (dlarfg) on column k -> v_k, tau_k.
//   S2 (every warp, rows i > k, lanes over columns k < j <= i): a_ij -= v_i w_j + w_i v_j
//      (update k-1) and, from the updated value, the row part sum_j a_ij v_kj of p_k,i
//      (4-row transposed warp reduction) and the column part a_ij v_ki of p_k,j (per-lane
//      registers, one colpart row per warp) -- the symmetric matvec over the packed triangle.
// Three block barriers per step; each stored element is read and written once per step.
struct TriPackedLayout {
    size_t L, wpart, rd, pf, wv, vb, total;  // offsets in doubles
};
__host__ __device__ inline TriPackedLayout tri_packed_layout(int n, int nw) {
    TriPackedLayout o;
    o.L = 0;
    o.wpart = ((size_t)n * (n + 1) / 2 + 1) & ~(size_t)1;  // 16-byte aligned rows
    o.rd = o.wpart + (size_t)nw * n;
    o.pf = o.rd + n;
    o.wv = o.pf + n;
    o.vb = o.wv + n;  // 2 x n
    o.total = o.vb + 2 * (size_t)n;
    return o;
}

template <int NT, int NTHR>
__global__ void __launch_bounds__(NTHR) tridiag_packed_kernel(TriArgs a) {
    pdl_entry();
    constexpr int NW = NTHR / 32;
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ double s_tau;
    const int n = a.n;
    const TriPackedLayout lay = tri_packed_layout(n, NW);
    double* L = sm + lay.L;
    double* wpart = sm + lay.wpart;
    double* rd = sm + lay.rd;
    double* pf = sm + lay.pf;
    double* wv = sm + lay.wv;
    double* vb = sm + lay.vb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto tri = [](int i) { return i * (i + 1) / 2; };
    double off = 0.0;
    for (int i = warp; i < n; i += NW) {
        double* Li = L + tri(i);
        for (int j = lane; j <= i; j += 32) {
            const double v = a.K[(size_t)i * a.ldk + j];
            Li[j] = v;
            if (j != i) off += 2.0 * v * v;
        }
    }
    for (int j = tid; j < n; j += NTHR) {
        pf[j] = 0.0;
        wv[j] = 0.0;
        rd[j] = 0.0;
        vb[j] = 0.0;
        vb[n + j] = 0.0;
    }
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {
        const double ot = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = ot * ot;
    }
    off = block_sum(off, red);
    if (!(off > tol_sq) || n == 1) {  // the reference's Jacobi would not rotate at all (la_core.cpp:33)
        for (int i = tid; i < n; i += NTHR) {
            a.d[i] = L[tri(i) + i];
            if (i + 1 < n) a.e[i] = 0.0;
        }
        if (tid == 0) *a.trivial = 1;
        return;
    }
    if (tid == 0) *a.trivial = 0;
    double tau_prev = 0.0;
    for (int k = 0; k + 1 < n; ++k) {
        double* vp = vb + (k & 1 ? 0 : n);  // v_{k-1}
        double* vc = vb + (k & 1 ? n : 0);  // v_k
        // ---- S0: p_{k-1} for j >= k
        if (k > 0) {
            for (int j = k + tid; j < n; j += NTHR) {
                double s = rd[j];
#pragma unroll 4
                for (int w = 0; w < NW; ++w) s += wpart[(size_t)w * n + j];
                pf[j] = s * tau_prev;
            }
        }
        __syncthreads();
        // ---- S1 (warp 0): w_{k-1}, column k, reflector k
        if (warp == 0) {
            double pj[NT], vj[NT];
            double dsum = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = k + lane + 32 * t;
                pj[t] = i < n ? pf[i] : 0.0;
                vj[t] = i < n ? vp[i] : 0.0;
                dsum = fma(pj[t], vj[t], dsum);
            }
            dsum = warp_sum(dsum);
            const double c = 0.5 * tau_prev * dsum;
            double wj[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = k + lane + 32 * t;
                wj[t] = pj[t] - c * vj[t];
                if (i < n) wv[i] = wj[t];
            }
            const double wk = __shfl_sync(0xffffffffu, wj[0], 0);  // w_{k-1,k}
            const double vk = __shfl_sync(0xffffffffu, vj[0], 0);  // v_{k-1,k}
            double x[NT];
            double xs = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = k + lane + 32 * t;
                x[t] = 0.0;
                if (i < n) {
                    double* p = L + tri(i) + k;
                    const double val = *p - vj[t] * wk - wj[t] * vk;
                    *p = val;
                    x[t] = val;
                    if (i >= k + 2) xs = fma(val, val, xs);
                }
            }
            xs = warp_sum(xs);
            const double alpha = __shfl_sync(0xffffffffu, x[0], 1);
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xs > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + xs), alpha);
                tau = (beta - alpha) * fast_rcp(beta);
                scal = fast_rcp(alpha - beta);
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = k + lane + 32 * t;
                if (i < n) {
                    const double v = i == k ? 0.0 : (i == k + 1) ? 1.0 : x[t] * scal;
                    vc[i] = v;
                    if (i > k) a.vh[(size_t)k * n + i] = v;
                }
            }
            if (lane == 0) {
                s_tau = tau;
                a.d[k] = x[0];
                a.e[k] = beta;
                a.tau[k] = tau;
            }
        }
        __syncthreads();
        // ---- S2: rows i > k
        {
            const double tau = s_tau;
            double rv[NT], rw[NT], rc[NT], cp[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = k + 1 + lane + 32 * t;
                const bool on = j < n;
                rv[t] = on ? vp[j] : 0.0;
                rw[t] = on ? wv[j] : 0.0;
                rc[t] = on ? vc[j] : 0.0;
                cp[t] = 0.0;
            }
            for (int i0 = k + 1 + warp; i0 < n; i0 += 4 * NW) {
                double sr[4];
                const int ilast = min(n - 1, i0 + 3 * NW);
                const int tcnt = (ilast - k - 1) / 32 + 1;  // column chunks the longest row needs
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = i0 + r * NW;
                    sr[r] = 0.0;
                    if (i < n) {
                        const double vi = vp[i], wi = wv[i], ci = vc[i];
                        double* Li = L + tri(i);
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            if (t < tcnt) {
                                const int j = k + 1 + lane + 32 * t;
                                if (j <= i) {
                                    const double val = Li[j] - vi * rw[t] - wi * rv[t];
                                    Li[j] = val;
                                    sr[r] = fma(val, rc[t], sr[r]);
                                    if (j < i) cp[t] = fma(val, ci, cp[t]);
                                }
                            }
                        }
                    }
                }
                const bool h16 = lane & 16, h8 = lane & 8;
                double a0 = h16 ? sr[2] : sr[0], a1 = h16 ? sr[3] : sr[1];
                a0 += __shfl_xor_sync(0xffffffffu, h16 ? sr[0] : sr[2], 16);
                a1 += __shfl_xor_sync(0xffffffffu, h16 ? sr[1] : sr[3], 16);
                double c0 = h8 ? a1 : a0;
                c0 += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 4);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 2);
                c0 += __shfl_xor_sync(0xffffffffu, c0, 1);
                const int i = i0 + (lane >> 3) * NW;
                if ((lane & 7) == 0 && i < n) rd[i] = c0;
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = k + 1 + lane + 32 * t;
                if (j < n) wpart[(size_t)warp * n + j] = cp[t];
            }
            tau_prev = tau;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.d[n - 1] = L[tri(n - 1) + n - 1];
        a.tau[n - 1] = 0.0;
    }
}

template <int NT, int NTHR>
void launch_packed(const TriArgs& a, size_t smem, cudaStream_t st) {
    auto* fn = tridiag_packed_kernel<NT, NTHR>;
    if (first_on_device((const void*)(fn))) {
        allow_max_dynamic_smem(fn);
    }
    static const int excl = getenv("SFDG_TRIDIAG_EXCLUSIVE") ? atoi(getenv("SFDG_TRIDIAG_EXCLUSIVE")) : 1;
    if (excl) {
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, (const void*)fn));
        smem = std::max(smem, (size_t)fa.maxDynamicSharedSizeBytes);
    }
    LAUNCH(fn, 1, NTHR, smem, st, a);
}

// The fused packed kernel (opt-in, SFDG_TRIDIAG=f, n <= ~226). Measured on the B200
// (tools/kbench, eigh top-100): n = 200 1090 us against 944 us for the 2-CTA cluster row
// kernel, n = 100 414 us against 320 us for the 1-CTA row kernel -- the third barrier and
// the S0 reduction per step cost more than the cluster barrier they replace, so the row
// kernels stay the default.
bool launch_tridiag_packed(const TriArgs& a, cudaStream_t st) {
    static const char* env = getenv("SFDG_TRIDIAG");
    if (!(env && env[0] == 'f')) return false;
    const int n = a.n;
    if (n < 2) return false;
    const int nt = (n + 31) / 32;
    if (nt > 8) return false;
    const size_t s16 = tri_packed_layout(n, 16).total * sizeof(double);
    const size_t s8 = tri_packed_layout(n, 8).total * sizeof(double);
    if (s16 <= 224 * 1024) launch_packed<8, 512>(a, s16, st);
    else if (s8 <= 224 * 1024) launch_packed<8, 256>(a, s8, st);
    else return false;
    return true;
}

template <int C, int NT, int NTHR>
void launch_rows(const TriRowsArgs& ra, size_t smem, cudaStream_t st) {
    auto* fn = tridiag_rows_kernel<C, NT, NTHR>;
    if (first_on_device((const void*)(fn))) {
        allow_max_dynamic_smem(fn);
        CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    // Exclusive SMs: asking for all the shared memory an SM has keeps other kernels' blocks
    // (the lanes' SpMMs) off the SMs this latency-bound chain kernel runs on.
    static const int excl = getenv("SFDG_TRIDIAG_EXCLUSIVE") ? atoi(getenv("SFDG_TRIDIAG_EXCLUSIVE")) : 1;
    if (excl) {
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, (const void*)fn));
        smem = std::max(smem, (size_t)fa.maxDynamicSharedSizeBytes);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ra.C);
    cfg.blockDim = dim3(NTHR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ra.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, fn, ra));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int C, int NT, int RPW>
void launch_regs(const TriRowsArgs& ra, cudaStream_t st) {
    auto* fn = tridiag_regs_kernel<C, NT, RPW>;
    if (first_on_device((const void*)(fn))) {
        allow_max_dynamic_smem(fn);
        CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    size_t smem = 4 * (size_t)ra.a.n * sizeof(double);
    static const int excl = getenv("SFDG_TRIDIAG_EXCLUSIVE") ? atoi(getenv("SFDG_TRIDIAG_EXCLUSIVE")) : 1;
    if (excl) {  // keep other kernels' blocks off these SMs (latency-bound chain kernel)
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, (const void*)fn));
        smem = std::max(smem, (size_t)fa.maxDynamicSharedSizeBytes);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, fn, ra));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Register-resident row kernel for 128 < n <= 512 (SFDG_TRIDIAG=c selects the shared-memory
// row kernel below, which it reproduces bit for bit; SFDG_TRIDIAG=r forces it for n <= 128
// too). Measured (tools/kbench, eigh top-100): n = 200 881 us against 930 us for the 2-CTA
// shared-memory kernel; n = 100 312 us against 302 us, so small n keeps the shared-memory
// kernel. tools/tri_probe shows why the gain is small: the trailing update costs the same
// ~3000-4600 cycles per step from registers as from shared memory -- the step is bound by
// dependent-instruction latency with 4 warps per scheduler, not by shared-memory traffic.
bool launch_tridiag_regs(const TriArgs& a, cudaStream_t st) {
    static const char* env = getenv("SFDG_TRIDIAG");
    if (env && (env[0] == 'c' || env[0] == 'p' || env[0] == 'f')) return false;
    const int n = a.n;
    TriRowsArgs ra{a, 1, n};
    if (n <= 128) {
        if (!(env && env[0] == 'r')) return false;
        launch_regs<1, 4, 8>(ra, st);
    } else if (n <= 256) {
        ra.C = 4;
        launch_regs<4, 8, 4>(ra, st);
    } else if (n <= 512) {
        ra.C = 16;
        launch_regs<16, 16, 2>(ra, st);
    } else return false;
    return true;
}

// Row-distributed tridiagonalisation when the full matrix fits the shared memory of a
// cluster of <= 16 CTAs (n <= ~670); false -> the caller uses the packed kernel.
bool launch_tridiag_rows(const TriArgs& a, cudaStream_t st) {
    static const char* env = getenv("SFDG_TRIDIAG");
    if (env && env[0] == 'p') return false;  // packed single-CTA kernel (A/B testing)
    const int n = a.n;
    const int nt = (n + 31) / 32;
    static const int min_c = getenv("SFDG_TRIDIAG_MINC") ? atoi(getenv("SFDG_TRIDIAG_MINC")) : 1;  // A/B testing
    for (int C = 1; C <= 16; C *= 2) {
        if (C < min_c) continue;
        const int rows = (n + C - 1) / C;
        const size_t smem = ((size_t)rows * n + 4 * (size_t)n) * sizeof(double);
        if (smem > 220 * 1024) continue;
        TriRowsArgs ra{a, C, rows};
        if (C == 1 && nt <= 4) launch_rows<1, 4, 512>(ra, smem, st);
        else if (C == 1 && nt <= 8) launch_rows<1, 8, 512>(ra, smem, st);
        else if (C == 2 && nt <= 8) launch_rows<2, 8, 512>(ra, smem, st);
        else if (C == 4 && nt <= 8) launch_rows<4, 8, 512>(ra, smem, st);
        else if (C == 4 && nt <= 12) launch_rows<4, 12, 256>(ra, smem, st);
        else if (C == 8 && nt <= 12) launch_rows<8, 12, 256>(ra, smem, st);
        else if (C == 8 && nt <= 16) launch_rows<8, 16, 256>(ra, smem, st);
        else if (C == 16 && nt <= 16) launch_rows<16, 16, 256>(ra, smem, st);
        else if (C == 16 && nt <= 21) launch_rows<16, 21, 256>(ra, smem, st);
        else return false;
        return true;
    }
    return false;
}

}  // namespace

// Top `nval` eigenpairs (descending) of the symmetric K (n x n). values (nval),
// vectors (n x ldv, column t). Sets *fallback when a cluster was too large for the
// Rayleigh-Ritz step (eigh() then runs the Jacobi solver); tolerances as in eigh().
void eigh_tri(const double* K, int n, int ldk, double off_tol, const double* d_fsq, int nval, double* values,
              double* vectors, int ldv, int* fallback, Scratch& scr, cudaStream_t st) {
    if (n <= 0) return;
    if (n > 1024) throw invalid_argument("eigh: n > 1024 unsupported");
    TriArgs a{};
    a.K = K;
    a.n = n;
    a.ldk = ldk;
    a.tol_sq = off_tol * off_tol;
    a.d_fsq = d_fsq;
    const bool use_smem = n <= kTriSmemMax;
    const size_t packed = (size_t)n * (n + 1) / 2;
    a.gpacked = use_smem ? nullptr : scr.take<double>((int64_t)packed + 2 * n);
    a.use_smem = use_smem;
    a.d = scr.take<double>(n);
    a.e = scr.take<double>(n);
    a.vh = scr.take<double>((int64_t)n * n);
    a.tau = scr.take<double>(n);
    a.trivial = scr.take<int>(1);
    const int64_t inv_slots = (int64_t)ceil_div(nval, 64) * 64;
    double* work = scr.take<double>(inv_slots * (5 * (int64_t)n + (n + 31) / 32 + 1));
    if (first_on_device((const void*)(tridiag_kernel<true>))) {
        allow_max_dynamic_smem(tridiag_kernel<true>);
        allow_max_dynamic_smem(inviter_kernel);
        allow_max_dynamic_smem(twisted_kernel);
    }
    {
        ProfScope prof("eigh_tridiag", st);
        if (!launch_tridiag_packed(a, st) && !launch_tridiag_regs(a, st) && !launch_tridiag_rows(a, st)) {
            const size_t smem = use_smem ? (packed + 2 * (size_t)n) * sizeof(double) : 0;
            if (use_smem) LAUNCH(tridiag_kernel<true>, 1, kTriThreads, smem, st, a);
            else LAUNCH(tridiag_kernel<false>, 1, kTriThreads, 0, st, a);
        }
    }
    {
        ProfScope prof("eigh_bisect", st);
        LAUNCH(bisect_kernel, ceil_div(nval, 4), 128, 2 * (size_t)n * sizeof(double), st, a.d, a.e, n, nval,
               a.trivial, values);
    }
    {
        ProfScope prof("eigh_vectors", st);
        // twisted factorisations (one warp per kEPW eigenvalues, 4n doubles each) when they fit
        static const bool twisted = !(getenv("SFDG_EIGVEC") && getenv("SFDG_EIGVEC")[0] == 'i');
        const size_t tsmem = (3 * (size_t)n + (size_t)kEPW * 4 * n) * sizeof(double);
        // per thread: 5n doubles of LU bands + ceil(n/32) flag words; T staged (2n doubles)
        const int ith = 8;
        const size_t per = 5 * (size_t)n * sizeof(double) + (size_t)((n + 31) / 32) * sizeof(unsigned);
        const size_t ismem = 2 * (size_t)n * sizeof(double) + ith * per;
        int* need = nullptr;
        if (twisted && tsmem <= 200 * 1024) {
            need = scr.take<int>(nval);
            LAUNCH(twisted_kernel, ceil_div(nval, kEPW), 32, tsmem, st, a.d, a.e, n, nval, values, a.trivial,
                   vectors, ldv, need);
        }
        if (ismem <= 96 * 1024)
            LAUNCH(inviter_kernel, ceil_div(nval, ith), ith, ismem, st, a.d, a.e, n, nval, values, a.trivial, vectors,
                   ldv, (double*)nullptr, (const int*)need);
        else
            LAUNCH(inviter_kernel, ceil_div(nval, 64), 64, 2 * (size_t)n * sizeof(double), st, a.d, a.e, n, nval,
                   values, a.trivial, vectors, ldv, work, (const int*)need);
        LAUNCH(cluster_kernel, nval, 32, 0, st, a.d, a.e, n, nval, values, a.trivial, vectors, ldv, fallback);
        backtransform(a.vh, a.tau, n, nval, a.trivial, vectors, ldv, st);
    }
}

}  // namespace sfdg
