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
//  3. inviter_kernel (thread per eigenvalue): inverse iteration with a partially pivoted
//     tridiagonal LU, distinct deterministic start vectors.
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

// Warp per eigenvalue: the top `nval` eigenvalues, written in descending order.
__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                              const int* __restrict__ trivial, double* __restrict__ lam_desc) {
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
        if (lane == 0) {
            // t-th largest with stable tie order: value with rank t
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int j = 0; j < n; ++j) r += (d[j] > d[i] || (d[j] == d[i] && j < i));
                if (r == t) lam_desc[t] = d[i];
            }
        }
        return;
    }
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int j = 0; j < n; ++j) {
        const double r = (j > 0 ? sqrt(e2[j - 1]) : 0.0) + (j + 1 < n ? sqrt(e2[j]) : 0.0);
        lo = fmin(lo, d[j] - r);
        hi = fmax(hi, d[j] + r);
        emax = fmax(emax, e2[j]);
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 1e3;
    lo -= 2.0 * 2.2e-16 * tnorm + pivmin;
    hi += 2.0 * 2.2e-16 * tnorm + pivmin;
    const int want = n - 1 - t;  // ascending index of the eigenvalue
    double a = lo, b = hi;       // count(a) <= want < count(b)
    for (int it = 0; it < 80; ++it) {
        if (b - a <= 2.0 * 2.2e-16 * fmax(fabs(a), fabs(b)) + pivmin) break;
        const double x = a + (b - a) * (double)(lane + 1) / 33.0;
        const int c = sturm_count(d, e2, n, x, pivmin);
        const unsigned above = __ballot_sync(0xffffffffu, c > want);  // lanes whose x is past the eigenvalue
        const int first = above ? __ffs(above) - 1 : 32;
        const double na = first > 0 ? a + (b - a) * (double)first / 33.0 : a;
        const double nb = first < 32 ? a + (b - a) * (double)(first + 1) / 33.0 : b;
        a = na;
        b = nb;
    }
    if (lane == 0) lam_desc[t] = 0.5 * (a + b);
}

// Thread per eigenvalue: 3 steps of inverse iteration with a partially pivoted LU of
// (T - lambda I) (LAPACK dgttrf/dgttrs algebra); X is n x ldx (column t = vector t).
__global__ void inviter_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                               const double* __restrict__ lam, const int* __restrict__ trivial,
                               double* __restrict__ X, int ldx, double* __restrict__ work_g) {
    extern __shared__ double work_s[];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nval) return;
    // per-thread LU bands + vector: shared memory when they fit (n <= 320), else global
    double* work = work_g ? work_g : work_s;
    const int slot = work_g ? t : threadIdx.x;
    if (*trivial) {  // identity eigenvectors in the stable descending order of the diagonal
        int idx = 0;
        for (int i = 0; i < n; ++i) {
            int r = 0;
            for (int j = 0; j < n; ++j) r += (dg[j] > dg[i] || (dg[j] == dg[i] && j < i));
            if (r == t) idx = i;
        }
        for (int i = 0; i < n; ++i) X[(size_t)i * ldx + t] = (i == idx) ? 1.0 : 0.0;
        return;
    }
    double* U0 = work + (size_t)slot * 5 * n;  // diag of U
    double* U1 = U0 + n;                    // 1st super
    double* U2 = U1 + n;                    // 2nd super
    double* Lm = U2 + n;                    // multipliers
    double* x = Lm + n;
    double tn = 0.0;
    for (int j = 0; j < n; ++j) tn = fmax(tn, fabs(dg[j]) + (j > 0 ? fabs(eg[j - 1]) : 0.0) + (j + 1 < n ? fabs(eg[j]) : 0.0));
    const double tiny = 2.2e-16 * fmax(tn, 1e-300);
    const double l = lam[t];
    // factor (T - l I) = P L U ; pivot flags packed in the sign of Lm via a separate array
    // (we store swaps in U2 >= 0 convention: keep a small local bitmask per 64 rows)
    unsigned long long swaps[16];  // n <= 1024
    for (int i = 0; i < 16; ++i) swaps[i] = 0ull;
    double a = dg[0] - l;  // current diagonal
    double b = n > 1 ? eg[0] : 0.0;  // current super
    for (int j = 0; j + 1 < n; ++j) {
        const double c = eg[j];               // sub-diagonal below a
        const double dn = dg[j + 1] - l;      // next diagonal
        const double bn = j + 2 < n ? eg[j + 1] : 0.0;  // next super
        if (fabs(a) >= fabs(c)) {
            const double m = (a != 0.0) ? c / a : 0.0;
            U0[j] = a;
            U1[j] = b;
            U2[j] = 0.0;
            Lm[j] = m;
            a = dn - m * b;
            b = bn;
        } else {
            const double m = a / c;
            U0[j] = c;
            U1[j] = dn;
            U2[j] = bn;
            Lm[j] = m;
            swaps[j >> 6] |= 1ull << (j & 63);
            a = b - m * dn;
            b = -m * bn;
        }
    }
    U0[n - 1] = a;
    for (int j = 0; j < n; ++j)
        if (fabs(U0[j]) < tiny) U0[j] = U0[j] < 0.0 ? -tiny : tiny;
    // deterministic distinct start vector
    uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(t + 1);
    for (int j = 0; j < n; ++j) {
        s ^= s >> 12;
        s ^= s << 25;
        s ^= s >> 27;
        x[j] = (double)((s * 2685821657736338717ull) >> 11) * 0x1.0p-53 - 0.5;
    }
    for (int it = 0; it < 3; ++it) {
        // forward: apply P and L
        for (int j = 0; j + 1 < n; ++j) {
            const bool sw = (swaps[j >> 6] >> (j & 63)) & 1ull;
            if (sw) {
                const double tmp = x[j];
                x[j] = x[j + 1];
                x[j + 1] = tmp - Lm[j] * x[j];
            } else {
                x[j + 1] -= Lm[j] * x[j];
            }
        }
        // backward: U x = y
        x[n - 1] /= U0[n - 1];
        if (n >= 2) x[n - 2] = (x[n - 2] - U1[n - 2] * x[n - 1]) / U0[n - 2];
        for (int j = n - 3; j >= 0; --j) x[j] = (x[j] - U1[j] * x[j + 1] - U2[j] * x[j + 2]) / U0[j];
        double nrm = 0.0;
        for (int j = 0; j < n; ++j) nrm += x[j] * x[j];
        nrm = 1.0 / sqrt(nrm);
        for (int j = 0; j < n; ++j) x[j] *= nrm;
    }
    for (int j = 0; j < n; ++j) X[(size_t)j * ldx + t] = x[j];
}

// Warp per cluster start: orthonormalise the cluster's vectors (MGS twice) and resolve the
// individual eigenvectors by Rayleigh-Ritz (cyclic Jacobi on the c x c projected matrix).
constexpr int kMaxCluster = 32;
__global__ void cluster_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int nval,
                               double* __restrict__ lam, const int* __restrict__ trivial, double* __restrict__ X,
                               int ldx, int* __restrict__ fallback) {
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
    // MGS, two passes
    for (int pass = 0; pass < 2; ++pass)
        for (int a = 0; a < c; ++a) {
            for (int b = 0; b < a; ++b) {
                double s = 0.0;
                for (int j = lane; j < n; j += 32) s += X[(size_t)j * ldx + t0 + a] * X[(size_t)j * ldx + t0 + b];
                s = warp_sum(s);
                for (int j = lane; j < n; j += 32) X[(size_t)j * ldx + t0 + a] -= s * X[(size_t)j * ldx + t0 + b];
                __syncwarp();
            }
            double s = 0.0;
            for (int j = lane; j < n; j += 32) s += X[(size_t)j * ldx + t0 + a] * X[(size_t)j * ldx + t0 + a];
            s = 1.0 / sqrt(warp_sum(s));
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

// U = Q X with Q = H_0 H_1 ... H_{n-3}: apply reflectors last-to-first. One CTA per
// 32 columns of X; the reflector loop is sequential, each step a dot + axpy per column.
__global__ void backtransform_kernel(const double* __restrict__ vh, const double* __restrict__ tau, int n, int nval,
                                     const int* __restrict__ trivial, double* __restrict__ X, int ldx) {
    if (*trivial) return;
    extern __shared__ double colbuf[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = blockIdx.x * (blockDim.x >> 5) + w;  // warp per column, kept in shared memory
    if (col >= nval) return;
    double* x = colbuf + (size_t)w * n;
    for (int j = lane; j < n; j += 32) x[j] = X[(size_t)j * ldx + col];
    __syncwarp();
    for (int k = n - 3; k >= 0; --k) {
        const double tk = tau[k];
        if (tk == 0.0) continue;
        const double* v = vh + (size_t)k * n;
        double s = 0.0;
        for (int j = k + 1 + lane; j < n; j += 32) s += v[j] * x[j];
        s = warp_sum(s) * tk;
        for (int j = k + 1 + lane; j < n; j += 32) x[j] -= s * v[j];
        __syncwarp();
    }
    for (int j = lane; j < n; j += 32) X[(size_t)j * ldx + col] = x[j];
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
    double* work = scr.take<double>((int64_t)nval * 5 * n);
    static bool attr = false;
    if (!attr) {
        allow_max_dynamic_smem(tridiag_kernel<true>);
        allow_max_dynamic_smem(inviter_kernel);
        allow_max_dynamic_smem(backtransform_kernel);
        attr = true;
    }
    {
        ProfScope prof("eigh_tridiag", st);
        const size_t smem = use_smem ? (packed + 2 * (size_t)n) * sizeof(double) : 0;
        if (use_smem) LAUNCH(tridiag_kernel<true>, 1, kTriThreads, smem, st, a);
        else LAUNCH(tridiag_kernel<false>, 1, kTriThreads, 0, st, a);
    }
    {
        ProfScope prof("eigh_bisect", st);
        LAUNCH(bisect_kernel, ceil_div(nval, 8), 256, 2 * (size_t)n * sizeof(double), st, a.d, a.e, n, nval, a.trivial,
               values);
    }
    {
        ProfScope prof("eigh_vectors", st);
        const int ith = 8;  // threads per block: 8 x 5n doubles of LU bands in shared memory
        const size_t ismem = (size_t)ith * 5 * n * sizeof(double);
        if (ismem <= 96 * 1024)
            LAUNCH(inviter_kernel, ceil_div(nval, ith), ith, ismem, st, a.d, a.e, n, nval, values, a.trivial, vectors,
                   ldv, (double*)nullptr);
        else
            LAUNCH(inviter_kernel, ceil_div(nval, 64), 64, 0, st, a.d, a.e, n, nval, values, a.trivial, vectors, ldv,
                   work);
        LAUNCH(cluster_kernel, nval, 32, 0, st, a.d, a.e, n, nval, values, a.trivial, vectors, ldv, fallback);
        LAUNCH(backtransform_kernel, ceil_div(nval, 8), 256, 8 * (size_t)n * sizeof(double), st, a.vh, a.tau, n, nval,
               a.trivial, vectors, ldv);
    }
}

}  // namespace sfdg
