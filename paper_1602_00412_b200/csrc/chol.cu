// chol.cu -- CholeskyQR factor + apply with the reference's column-drop rule.
//
// Reference: orthonormalize (core/src/la_core.cpp:130-165) runs modified Gram-Schmidt
// with one re-orthogonalisation pass and zeroes a column whose residual norm falls
// below 1e-12 * (largest input column norm). On the GPU the same span is produced by
// CholeskyQR2: G = Y^T Y (DMMA, dense.cu), G = R^T R here, Y <- Y R^-1, twice. The
// Cholesky pivot R_jj^2 is exactly column j's squared residual after projecting out the
// kept columns 0..j-1, so the MGS drop rule becomes a pivot test. A Gram-formed pivot
// carries O(k u G_jj) cancellation error, so a pivot below kRelDrop * G_jj is treated as
// numerically dependent and dropped as well.
//
//  * chol_factor_kernel (1 CTA): R (upper, k x k) with a one-barrier-per-pivot right-
//    looking loop (warp 0 carries the pivot chain, the other warps the trailing update),
//    plus the inverse of every 8 x 8 diagonal block of R.
//  * trsm_apply_kernel (many CTAs): Q = Y R^-1 without ever forming R^-1: each warp owns
//    16 rows and forward-substitutes them block column by block column with DMMA
//    (X_b = (Y_b - X_<b R_<b,b) inv(R_bb)); rows are independent, so no CTA barrier.
//  * Second pass (polar): after one CholeskyQR pass, G = Q^T Q = I + E with tiny E, and
//    T = I - E/2 gives (QT)^T(QT) = I - 3/4 E^2 + O(E^3) with the same span. The kernel
//    emits T for gemm_nn when max|E| <= kPolarMax and otherwise falls back to the
//    Cholesky path, so accuracy never depends on the guess.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr double kRelDrop = 1e-13;  // ~ 4 k u for k <= 256
constexpr double kPolarMax = 1e-6;  // |E|^2 <= 1e-12 relative -> far below the 1e-8 gate
constexpr int kCholThreads = 512;
constexpr int kSmemMaxK = 160;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// out: R (k x k row-major, upper; dropped rows = e_j), dinv8 (k x 8: inverse of the
// 8 x 8 diagonal block containing row i, row i of that inverse, zero columns for dropped),
// stats[0] = min relative pivot, [1] = dropped count, [2] = max|G - I|,
// [3] = max R_jj / min R_jj over kept columns, [4] = 1 when the polar path was taken.
__global__ void __launch_bounds__(kCholThreads) chol_factor_kernel(const double* __restrict__ G, int k, int ldg,
                                                                   double* __restrict__ Rout, double* __restrict__ dinv8,
                                                                   double* __restrict__ T, int ldt,
                                                                   double* __restrict__ stats, int* __restrict__ err,
                                                                   int err_bit, double* __restrict__ gscratch,
                                                                   int use_smem, int polar, int* __restrict__ udrop) {
    pdl_entry();
    extern __shared__ double sm[];
    const int lda = use_smem ? k + 4 : k;
    double* A = use_smem ? sm : gscratch;
    double* d0 = A + (size_t)k * lda;  // original diagonal
    __shared__ double s_thr, s_emax;
    __shared__ int s_bad, s_dropped;
    __shared__ double red[32];
    __shared__ int s_drop[512];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;

    if (tid == 0) {
        s_bad = 0;
        s_dropped = 0;
    }
    for (int j = tid; j < k; j += nt) s_drop[j] = 0;
    __syncthreads();
    double mx = 0.0, emax = 0.0;
    for (int i = warp; i < k; i += nw)
        for (int j = i + lane; j < k; j += 32) {
            const double v = G[(size_t)i * ldg + j];
            if (!isfinite(v)) s_bad = 1;
            A[(size_t)i * lda + j] = v;
            if (i == j) {
                d0[i] = v;
                mx = fmax(mx, v);
            }
        }
    __syncthreads();
    if (polar) {  // max |G - I| over the kept (nonzero-diagonal) columns
        for (int i = warp; i < k; i += nw)
            for (int j = i + lane; j < k; j += 32) {
                if (d0[i] == 0.0 || d0[j] == 0.0) continue;
                emax = fmax(emax, fabs(A[(size_t)i * lda + j] - (i == j ? 1.0 : 0.0)));
            }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    if (lane == 0) {
        red[warp] = mx;
        red[16 + warp] = emax;
    }
    __syncthreads();
    if (tid == 0) {
        double m = 0.0, em = 0.0;
        for (int w = 0; w < nw; ++w) {
            m = fmax(m, red[w]);
            em = fmax(em, red[16 + w]);
        }
        const double drop_tol = 1e-12 * sqrt(m);  // la_core.cpp:141
        s_thr = drop_tol * drop_tol;
        s_emax = em;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) atomicOr(err, err_bit);
        if (polar)
            for (int e = tid; e < k * k; e += nt) T[(size_t)(e / k) * ldt + e % k] = 0.0;
        for (int e = tid; e < k * k; e += nt) Rout[e] = (e / k == e % k) ? 1.0 : 0.0;
        for (int e = tid; e < k * 8; e += nt) dinv8[e] = 0.0;
        if (tid == 0) {
            stats[0] = 0.0;
            stats[3] = 1e300;
            stats[4] = 0.0;
            stats[5] = 1e300;
            stats[6] = 0.0;
        }
        if (udrop)
            for (int j = tid; j < k; j += nt) udrop[j] = 0;
        return;
    }
    if (polar && s_emax <= kPolarMax) {
        // T = I - E/2 on kept columns, zero rows/columns for dropped ones (Q_j = 0 stays 0)
        for (int i = warp; i < k; i += nw)
            for (int j = lane; j < k; j += 32) {
                double v = 0.0;
                if (d0[i] != 0.0 && d0[j] != 0.0) {
                    const double g = i <= j ? A[(size_t)i * lda + j] : A[(size_t)j * lda + i];
                    v = (i == j ? 1.0 : 0.0) - 0.5 * (g - (i == j ? 1.0 : 0.0));
                }
                T[(size_t)i * ldt + j] = v;
            }
        if (tid == 0) {
            stats[0] = 1.0;
            stats[1] = 0.0;
            stats[2] = s_emax;
            stats[3] = 1.0;
            stats[4] = 1.0;
            stats[6] = 0.0;
        }
        if (udrop)
            for (int j = tid; j < k; j += nt) udrop[j] = 0;
        return;
    }

    // ---- right-looking Cholesky, one barrier per pivot
    auto pivot_row = [&](int j) {  // warp 0 only
        const double piv = A[(size_t)j * lda + j];
        const bool keep = isfinite(piv) && piv > s_thr && piv > kRelDrop * d0[j] && piv > 0.0;
        const double r = keep ? sqrt(piv) : 1.0;
        const double ri = 1.0 / r;
        for (int c = j + 1 + lane; c < k; c += 32) {
            double* a = A + (size_t)j * lda + c;
            *a = keep ? *a * ri : 0.0;
        }
        if (lane == 0) {
            A[(size_t)j * lda + j] = r;
            if (!keep) {
                s_drop[j] = 1;
                s_dropped += 1;
            }
        }
        __syncwarp();
    };
    if (use_smem && k % 8 == 0 && k <= 128) {
        // Blocked right-looking Cholesky: warp 0 factors an 8-row panel entirely in
        // registers (pivots via shuffles, no barrier), then all warps apply the rank-8
        // trailing update R_p^T R_p with DMMA on 8 x 8 tiles. Two barriers per 8 pivots.
        const int g = lane >> 2, t4 = lane & 3;
        for (int jb = 0; jb < k; jb += 8) {
            if (warp == 0) {
                double p[8][4];
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = jb + lane + 32 * q;
                        p[r][q] = c < k ? A[(size_t)(jb + r) * lda + c] : 0.0;
                    }
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = jb + jj;
                    const double piv = __shfl_sync(0xffffffffu, p[jj][0], jj);
                    const bool keep = isfinite(piv) && piv > s_thr && piv > kRelDrop * d0[j] && piv > 0.0;
                    const double r = keep ? sqrt(piv) : 1.0;
                    const double ri = 1.0 / r;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = jb + lane + 32 * q;
                        if (c > j) p[jj][q] = keep ? p[jj][q] * ri : 0.0;
                        else if (c == j) p[jj][q] = r;
                    }
                    if (!keep && lane == 0) {
                        s_drop[j] = 1;
                        s_dropped += 1;
                    }
#pragma unroll
                    for (int ii = jj + 1; ii < 8; ++ii) {
                        const double coef = __shfl_sync(0xffffffffu, p[jj][0], ii);  // R[j][jb + ii]
#pragma unroll
                        for (int q = 0; q < 4; ++q) p[ii][q] -= coef * p[jj][q];
                    }
                }
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = jb + lane + 32 * q;
                        if (c < k && c >= jb + r) A[(size_t)(jb + r) * lda + c] = p[r][q];
                    }
            }
            __syncthreads();
            const int t0 = jb / 8 + 1, nrem = k / 8 - t0;
            const int ntiles = nrem * (nrem + 1) / 2;
            for (int tile = warp; tile < ntiles; tile += nw) {
                int ti = 0, rem = tile;
                while (rem >= nrem - ti) {
                    rem -= nrem - ti;
                    ++ti;
                }
                const int i0 = (t0 + ti) * 8, c0 = (t0 + ti + rem) * 8;
                double v0 = 0.0, v1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 8; ks += 4) {
                    const double av = A[(size_t)(jb + ks + t4) * lda + i0 + g];
                    const double bv = A[(size_t)(jb + ks + t4) * lda + c0 + g];
                    dmma884(v0, v1, av, bv);
                }
                double* dst = A + (size_t)(i0 + g) * lda + c0 + 2 * t4;
                dst[0] -= v0;
                dst[1] -= v1;
            }
            __syncthreads();
        }
    } else {
    if (warp == 0) pivot_row(0);
    __syncthreads();
    for (int j = 0; j + 1 < k; ++j) {
        const bool kept = !s_drop[j];
        const double* rj = A + (size_t)j * lda;
        if (warp == 0) {
            if (kept) {
                const double rji = rj[j + 1];
                for (int c = j + 1 + lane; c < k; c += 32) A[(size_t)(j + 1) * lda + c] -= rji * rj[c];
            }
            __syncwarp();
            pivot_row(j + 1);
        } else if (kept) {
            for (int i = j + 1 + warp; i < k; i += nw - 1) {  // rows j+2.. (warp w >= 1)
                const double rji = rj[i];
                if (rji == 0.0) continue;
                double* ai = A + (size_t)i * lda;
                for (int c = i + lane; c < k; c += 32) ai[c] -= rji * rj[c];
            }
        }
        __syncthreads();
    }
    }
    // ---- outputs: R, and the inverse of every 8 x 8 diagonal block (one thread per
    // column of each block solves the 8 x 8 triangular system by back substitution)
    for (int i = warp; i < k; i += nw)
        for (int c = lane; c < k; c += 32) Rout[(size_t)i * k + c] = c >= i ? A[(size_t)i * lda + c] : 0.0;
    for (int t = tid; t < k; t += nt) {
        const int c = t;  // column c of block b = c / 8
        const int b0 = (c / 8) * 8, b1 = min(b0 + 8, k);
        double x[8];
        for (int i = 0; i < 8; ++i) x[i] = 0.0;
        if (!s_drop[c]) {
            for (int i = c; i >= b0; --i) {
                double s = (i == c) ? 1.0 : 0.0;
                for (int l = i + 1; l <= c; ++l) s -= A[(size_t)i * lda + l] * x[l - b0];
                x[i - b0] = s / A[(size_t)i * lda + i];
            }
        }
        // dinv8 row i (i in block) column (c - b0): inv(R_bb)[i][c]
        for (int i = b0; i < b1; ++i) dinv8[(size_t)i * 8 + (c - b0)] = x[i - b0];
    }
    __syncthreads();
    if (tid == 0) {
        double mn = 1.0, rmax = 0.0, rmin = 1e300;
        for (int j = 0; j < k; ++j)
            if (!s_drop[j] && d0[j] > 0.0) {
                const double r = A[(size_t)j * lda + j];
                mn = fmin(mn, r * r / d0[j]);
                rmax = fmax(rmax, r);
                rmin = fmin(rmin, r);
            }
        stats[0] = mn;
        stats[1] = (double)s_dropped;
        stats[2] = s_emax;
        stats[3] = rmin > 0.0 && rmin < 1e300 ? rmax / rmin : 1.0;
        stats[4] = 0.0;
        stats[5] = fmax(stats[5], stats[3]);  // running max over the calls sharing `stats`
    }
    // Uncertain drops: columns of non-negligible norm dropped by the relative pivot test
    // alone. The Gram cannot tell whether their residual is above the reference's absolute
    // threshold (exact_orth_kernel can); udrop[j] marks them, stats[6] counts them and
    // stats[7] accumulates the count over the calls sharing `stats`.
    if (warp == 0) {
        int cnt = 0;
        for (int j = lane; j < k; j += 32) {
            const int u = s_drop[j] && d0[j] > s_thr;
            if (udrop) udrop[j] = u;
            cnt += u;
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) {
            stats[6] = (double)cnt;
            stats[7] += (double)cnt;
        }
    }
}

// Q = Y R^-1 (m x k, ld). Each warp owns 16 rows (two 8-row DMMA tiles) and forward-
// substitutes them block column by block column: acc = Y_b - X_<b R_<b,b ; X_b = acc inv(R_bb).
// Rows are independent, so after the cp.async staging of R, inv(R_bb) and the row tile there
// is no CTA barrier. When the second-pass polar path was taken (stats[4] == 1) the kernel
// is a no-op (gemm_nn applies T instead).
__device__ __forceinline__ void cpa8(double* smem, const double* gmem, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0));
}
constexpr int kTrsmThreads = 256;
constexpr int kTrsmSmemK = 128;
__global__ void __launch_bounds__(kTrsmThreads) trsm_apply_kernel(const double* __restrict__ Y, int m, int k, int ld,
                                                                  const double* __restrict__ R,
                                                                  const double* __restrict__ dinv8,
                                                                  double* __restrict__ X, int ldx,
                                                                  const double* __restrict__ stats, int rows) {
    pdl_entry();
    if (stats && stats[4] != 0.0) return;
    extern __shared__ double sm[];
    const int kp = (k + 7) / 8 * 8;
    const bool rsm = kp <= kTrsmSmemK;  // R staged in shared memory, else read through L1
    const int ldr = rsm ? kp + 4 : k;   // conflict-free B-fragment reads (ldr % 16 == 4 or 12)
    const int ldy = kp + 4;
    double* Rs = sm;                                 // kp x ldr (when rsm)
    double* Ds = Rs + (rsm ? (size_t)kp * ldr : 0);  // kp x 12
    double* Xs = Ds + (size_t)kp * 12;               // rows x ldy : Y tile, overwritten by X
    const double* Rr = rsm ? Rs : R;
    const int r0 = blockIdx.x * rows;
    if (rsm)
        for (int e = threadIdx.x; e < kp * kp; e += blockDim.x) {
            const int i = e / kp, c = e % kp;
            const bool ok = i < k && c < k;
            cpa8(Rs + (size_t)i * ldr + c, ok ? R + (size_t)i * k + c : R, ok);
        }
    for (int e = threadIdx.x; e < kp * 8; e += blockDim.x) {
        const int i = e / 8, c = e % 8;
        cpa8(Ds + (size_t)i * 12 + c, i < k ? dinv8 + (size_t)i * 8 + c : dinv8, i < k);
    }
    for (int e = threadIdx.x; e < rows * kp; e += blockDim.x) {
        const int i = e / kp, c = e % kp;
        const bool ok = r0 + i < m && c < k;
        cpa8(Xs + (size_t)i * ldy + c, ok ? Y + (size_t)(r0 + i) * ld + c : Y, ok);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (rsm)  // pad rows/cols beyond k: identity so padded columns stay exactly zero
        for (int i = k + threadIdx.x; i < kp; i += blockDim.x) Rs[(size_t)i * ldr + i] = 1.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nb = kp / 8;
    const int ntile = rows / 8;
    for (int mt = w; mt < ntile; mt += blockDim.x / 32) {
        double* xr = Xs + (size_t)(mt * 8) * ldy;  // this warp's 8-row tile
        for (int b = 0; b < nb; ++b) {
            double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;  // two chains: X_<b R_<b,b
            int kk = 0;
            for (; kk + 4 < 8 * b; kk += 8) {
                const int r1 = kk + t, r2 = kk + 4 + t, cc = 8 * b + g;
                const double bv1 = rsm ? Rr[(size_t)r1 * ldr + cc] : (r1 < k && cc < k ? __ldg(Rr + (size_t)r1 * ldr + cc) : 0.0);
                const double bv2 = rsm ? Rr[(size_t)r2 * ldr + cc] : (r2 < k && cc < k ? __ldg(Rr + (size_t)r2 * ldr + cc) : 0.0);
                dmma884(c0, c1, xr[(size_t)g * ldy + r1], bv1);
                dmma884(e0, e1, xr[(size_t)g * ldy + r2], bv2);
            }
            for (; kk < 8 * b; kk += 4) {
                const int r1 = kk + t, cc = 8 * b + g;
                const double bv1 = rsm ? Rr[(size_t)r1 * ldr + cc] : (r1 < k && cc < k ? __ldg(Rr + (size_t)r1 * ldr + cc) : 0.0);
                dmma884(c0, c1, xr[(size_t)g * ldy + r1], bv1);
            }
            c0 += e0;
            c1 += e1;
            // acc = Y_b - acc, as a C fragment: row g, cols 2t, 2t+1 of block b
            double* yb = xr + (size_t)g * ldy + 8 * b + 2 * t;
            const double a0 = yb[0] - c0, a1 = yb[1] - c1;
            __syncwarp();
            yb[0] = a0;
            yb[1] = a1;
            __syncwarp();
            double x0 = 0.0, x1 = 0.0;  // X_b = acc inv(R_bb)
#pragma unroll
            for (int ks = 0; ks < 8; ks += 4)
                dmma884(x0, x1, xr[(size_t)g * ldy + 8 * b + ks + t], Ds[(size_t)(8 * b + ks + t) * 12 + g]);
            __syncwarp();
            yb[0] = x0;
            yb[1] = x1;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        if (r0 + i < m) X[(size_t)(r0 + i) * ldx + c] = Xs[(size_t)i * ldy + c];
    }
}

// k > 128: R no longer fits shared memory next to the row tile, and reading its B fragments
// through L1/L2 serialises every DMMA on an L2 round trip (19 ms for 1e6 x 256 at c5). Here
// the CTA walks the block columns b in lockstep and stages only the panel R[0 : 8b+8, 8b :
// 8b+8] it needs (double-buffered with cp.async while the previous block column computes).
constexpr int kPanelLd = 12;  // 8 columns + 4: conflict-free fragment reads
__global__ void __launch_bounds__(kTrsmThreads) trsm_panel_kernel(const double* __restrict__ Y, int m, int k, int ld,
                                                                  const double* __restrict__ R,
                                                                  const double* __restrict__ dinv8,
                                                                  double* __restrict__ X, int ldx,
                                                                  const double* __restrict__ stats, int rows) {
    pdl_entry();
    if (stats && stats[4] != 0.0) return;
    extern __shared__ double sm[];
    const int kp = (k + 7) / 8 * 8;
    const int ldy = kp + 4;
    double* Ps = sm;                                  // 2 x kp x kPanelLd : panels of R
    double* Ds = Ps + 2 * (size_t)kp * kPanelLd;      // kp x 12
    double* Xs = Ds + (size_t)kp * 12;                // rows x ldy
    const int r0 = blockIdx.x * rows;
    auto stage_panel = [&](int b, int buf) {
        double* P = Ps + (size_t)buf * kp * kPanelLd;
        const int nr = 8 * b + 8;
        for (int e = threadIdx.x; e < nr * 8; e += blockDim.x) {
            const int i = e / 8, c = e % 8, cc = 8 * b + c;
            const bool ok = i < k && cc < k;
            cpa8(P + (size_t)i * kPanelLd + c, ok ? R + (size_t)i * k + cc : R, ok);
        }
    };
    for (int e = threadIdx.x; e < kp * 8; e += blockDim.x) {
        const int i = e / 8, c = e % 8;
        cpa8(Ds + (size_t)i * 12 + c, i < k ? dinv8 + (size_t)i * 8 + c : dinv8, i < k);
    }
    for (int e = threadIdx.x; e < rows * kp; e += blockDim.x) {
        const int i = e / kp, c = e % kp;
        const bool ok = r0 + i < m && c < k;
        cpa8(Xs + (size_t)i * ldy + c, ok ? Y + (size_t)(r0 + i) * ld + c : Y, ok);
    }
    stage_panel(0, 0);
    asm volatile("cp.async.commit_group;\n" ::);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nb = kp / 8;
    const int ntile = rows / 8;
    for (int b = 0; b < nb; ++b) {
        if (b + 1 < nb) stage_panel(b + 1, (b + 1) & 1);
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);  // panel b (and the tiles) landed
        __syncthreads();
        const double* P = Ps + (size_t)(b & 1) * kp * kPanelLd;
        for (int mt = w; mt < ntile; mt += blockDim.x / 32) {
            double* xr = Xs + (size_t)(mt * 8) * ldy;
            double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
            int kk = 0;
            for (; kk + 4 < 8 * b; kk += 8) {
                dmma884(c0, c1, xr[(size_t)g * ldy + kk + t], P[(size_t)(kk + t) * kPanelLd + g]);
                dmma884(e0, e1, xr[(size_t)g * ldy + kk + 4 + t], P[(size_t)(kk + 4 + t) * kPanelLd + g]);
            }
            for (; kk < 8 * b; kk += 4) dmma884(c0, c1, xr[(size_t)g * ldy + kk + t], P[(size_t)(kk + t) * kPanelLd + g]);
            c0 += e0;
            c1 += e1;
            double* yb = xr + (size_t)g * ldy + 8 * b + 2 * t;
            const double a0 = yb[0] - c0, a1 = yb[1] - c1;
            __syncwarp();
            yb[0] = a0;
            yb[1] = a1;
            __syncwarp();
            double x0 = 0.0, x1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ks += 4)
                dmma884(x0, x1, xr[(size_t)g * ldy + 8 * b + ks + t], Ds[(size_t)(8 * b + ks + t) * 12 + g]);
            __syncwarp();
            yb[0] = x0;
            yb[1] = x1;
            __syncwarp();
        }
        __syncthreads();  // the buffer of panel b is refilled two iterations later
    }
    for (int e = threadIdx.x; e < rows * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        if (r0 + i < m) X[(size_t)(r0 + i) * ldx + c] = Xs[(size_t)i * ldy + c];
    }
}


// ---- exact_orth_kernel: the reference's Gram-Schmidt decisions (la_core.cpp:130-165)
// One 8-CTA cluster; CTA r owns rows [r * chunk, (r + 1) * chunk). Column reductions go
// through the CTAs' shared memory: each CTA writes its partial vector, a cluster barrier,
// then every CTA sums the 8 partials in rank order (identical totals everywhere).
// Per column j: sweep A (h = Q_<j^T t), sweep B (t -= Q_<j h, h2 = Q_<j^T t), sweep C
// (t -= Q_<j h2, |t|^2): classical Gram-Schmidt twice, accurate to O(u |t|) like the
// reference's re-orthogonalised MGS.
constexpr int kXC = 8;
constexpr int kXThreads = 512;
constexpr int kXWarps = kXThreads / 32;
constexpr int kXMaxK = 512;
// dynamic shared memory: per-warp partials, two cluster exchange vectors, the totals
size_t exact_orth_smem(int k) { return (size_t)(kXWarps + 3) * (size_t)((k + 31) / 32 * 32) * sizeof(double); }

__global__ void __cluster_dims__(kXC, 1, 1) __launch_bounds__(kXThreads)
    exact_orth_kernel(const double* __restrict__ Y, int ldy, double* __restrict__ Q, int ldq, int m, int k,
                      const int* __restrict__ udrop, const double* __restrict__ stats, double* __restrict__ tmp,
                      int force) {
    pdl_entry();
    if (!force && !(stats[6] > 0.0)) return;  // uniform over the cluster
    extern __shared__ double xsm[];
    const int KM = (k + 31) / 32 * 32;
    double* wred = xsm;                        // [kXWarps][KM]
    double* part = wred + (size_t)kXWarps * KM;  // [2][KM]
    double* h = part + 2 * (size_t)KM;           // [KM]
    const unsigned rank = cluster_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = (m + kXC - 1) / kXC;
    const int r0 = min(m, (int)rank * chunk), r1 = min(m, r0 + chunk);
    int pb = 0;

    // per-lane column accumulators acc[c] <-> column 32 c + lane  ->  h[0, n) (cluster totals)
    auto reduce = [&](const double* acc, int n) {
        const int nc = (n + 31) / 32;
        for (int c = 0; c < nc; ++c)
            if (32 * c + lane < n) wred[(size_t)warp * KM + 32 * c + lane] = acc[c];
        __syncthreads();
        for (int p = tid; p < n; p += kXThreads) {
            double v = 0.0;
            for (int w = 0; w < kXWarps; ++w) v += wred[(size_t)w * KM + p];
            part[(size_t)pb * KM + p] = v;
        }
        cluster_barrier();
        for (int p = tid; p < n; p += kXThreads) {
            double v = 0.0;
            for (unsigned r = 0; r < kXC; ++r) v += cluster_map(part + (size_t)pb * KM, r)[p];
            h[p] = v;
        }
        pb ^= 1;
        __syncthreads();
    };
    // (sum_p<j h_p Q_ip) for row i, lanes over p; every lane gets the total
    auto hq = [&](int i, int j) {
        double s = 0.0;
        for (int p = lane; p < j; p += 32) s += h[p] * Q[(size_t)i * ldq + p];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    };
    // residual of target column t (t(i) = tgt[i * ts]) against Q_<j; returns |t|
    auto residual = [&](double* tgt, size_t ts, int j) {
        double acc[kXMaxK / 32];
        const int nc = (j + 31) / 32;
        if (j > 0) {
            for (int c = 0; c < kXMaxK / 32; ++c) acc[c] = 0.0;
            for (int i = r0 + warp; i < r1; i += kXWarps) {  // sweep A
                const double t = tgt[(size_t)i * ts];
                for (int c = 0; c < nc; ++c) {
                    const int p = 32 * c + lane;
                    if (p < j) acc[c] += Q[(size_t)i * ldq + p] * t;
                }
            }
            reduce(acc, j);
            for (int c = 0; c < kXMaxK / 32; ++c) acc[c] = 0.0;
            for (int i = r0 + warp; i < r1; i += kXWarps) {  // sweep B
                const double t = tgt[(size_t)i * ts] - hq(i, j);
                __syncwarp();
                if (lane == 0) tgt[(size_t)i * ts] = t;
                for (int c = 0; c < nc; ++c) {
                    const int p = 32 * c + lane;
                    if (p < j) acc[c] += Q[(size_t)i * ldq + p] * t;
                }
            }
            reduce(acc, j);
        }
        double nrm = 0.0;
        for (int i = r0 + warp; i < r1; i += kXWarps) {  // sweep C
            const double t = j > 0 ? tgt[(size_t)i * ts] - hq(i, j) : tgt[(size_t)i * ts];
            __syncwarp();
            if (lane == 0) {
                tgt[(size_t)i * ts] = t;
                nrm += t * t;
            }
        }
        for (int c = 0; c < kXMaxK / 32; ++c) acc[c] = 0.0;
        acc[0] = nrm;  // lane 0 of each warp carries the warp's share
        reduce(acc, 1);
        return sqrt(h[0]);
    };

    // drop_tol = 1e-12 * max_j |y_j| over the input columns (la_core.cpp:135-141)
    {
        double acc[kXMaxK / 32];
        for (int c = 0; c < kXMaxK / 32; ++c) acc[c] = 0.0;
        const int nc = (k + 31) / 32;
        for (int i = r0 + warp; i < r1; i += kXWarps)
            for (int c = 0; c < nc; ++c) {
                const int p = 32 * c + lane;
                if (p < k) {
                    const double v = Y[(size_t)i * ldy + p];
                    acc[c] += v * v;
                }
            }
        reduce(acc, k);
    }
    __shared__ double s_tol;
    __shared__ int s_redo;
    if (tid == 0) {
        double mx = 0.0;
        for (int p = 0; p < k; ++p) mx = fmax(mx, h[p]);
        s_tol = 1e-12 * sqrt(mx);
        s_redo = force;
    }
    __syncthreads();
    const double tol = s_tol;

    // confirm CholeskyQR's uncertain drops against the threshold
    if (!s_redo)
        for (int j = 0; j < k; ++j) {
            if (!udrop[j]) continue;
            for (int i = r0 + tid; i < r1; i += kXThreads) tmp[i] = Y[(size_t)i * ldy + j];
            __syncthreads();
            const double nrm = residual(tmp, 1, j);
            if (!(nrm < tol || nrm == 0.0)) {  // the reference keeps column j
                if (tid == 0) s_redo = 1;
                __syncthreads();
                break;
            }
        }
    __syncthreads();
    if (s_redo) {
        // Gram-Schmidt with re-orthogonalisation on a copy of Y (la_core.cpp:143-163)
        for (int i = r0 + warp; i < r1; i += kXWarps)
            for (int p = lane; p < k; p += 32) Q[(size_t)i * ldq + p] = Y[(size_t)i * ldy + p];
        __syncthreads();
        for (int j = 0; j < k; ++j) {
            const double nrm = residual(Q + j, (size_t)ldq, j);
            const bool keep = !(nrm < tol || nrm == 0.0);
            const double inv = keep ? 1.0 / nrm : 0.0;
            for (int i = r0 + tid; i < r1; i += kXThreads) {
                double* q = Q + (size_t)i * ldq + j;
                *q = keep ? *q * inv : 0.0;
            }
            __syncthreads();
        }
    }
    cluster_barrier();  // no CTA leaves while a peer may still read its partials
}
}  // namespace

namespace {

// ---- Q = Y R^-1 as inverse + GEMM (the default for k % 8 == 0) -----------------------------
// The substitution kernels above walk k / 8 dependent block columns per 8-row tile, a DMMA
// latency chain that leaves the FP64 pipe mostly idle (c4: 161 us for 5e4 x 128). Instead:
// trinv_kernel forms T = R^-1 once per factorisation (one CTA, warp b owns block column b and
// back-substitutes its 8 x 8 blocks bottom-up: T_bb = inv(R_bb) from dinv8, T_ab =
// -inv(R_aa) sum_{a<c<=b} R_ac T_cb), then tsmm_kernel applies X = Y T as a triangular GEMM on
// DMMA. A dropped column j has a zero column in dinv8, hence zero column j and zero row j in T
// (R's dropped row is e_j), exactly the substitution's X_j = 0 with Y_j not contributing.
// Same span, same drop decisions; the products round differently (~u kappa(R)), which the
// second CholeskyQR pass absorbs like any other rounding.
template <bool SM>
__global__ void __launch_bounds__(1024) trinv_kernel(const double* __restrict__ R, int k,
                                                     const double* __restrict__ dinv8, double* __restrict__ T,
                                                     int ldt, const double* __restrict__ stats) {
    pdl_entry();
    if (stats && stats[4] != 0.0) return;  // polar second pass: nothing to apply
    extern __shared__ double tsm[];        // SM: block column b's tiles (rows 0..b) at 64 b (b+1) / 2
    const int nb = k / 8;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {  // lower triangle (block-wise) = 0
        const int i = e / k, j = e % k;
        if (i / 8 > j / 8) T[(size_t)i * ldt + j] = 0.0;
    }
    for (int b = w; b < nb; b += nw) {
        // tile (a, b): 8 x 8 row-major
        auto tile = [&](int a) -> double* { return SM ? tsm + 32 * b * (b + 1) + 64 * a : T + (size_t)(8 * a) * ldt + 8 * b; };
        const int tld = SM ? 8 : ldt;
        auto tload = [&](const double* p) { return SM ? *p : __ldcg(p); };
        {
            double* tb = tile(b);
            for (int e = lane; e < 64; e += 32) tb[(e >> 3) * tld + (e & 7)] = dinv8[(size_t)(8 * b + (e >> 3)) * 8 + (e & 7)];
        }
        __syncwarp();
        for (int a = b - 1; a >= 0; --a) {
            double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;  // acc = sum_c R_ac T_cb, two chains
            for (int c = a + 1; c <= b; ++c) {
                const double* tc = tile(c);
                dmma884(c0, c1, __ldg(R + (size_t)(8 * a + g) * k + 8 * c + t), tload(tc + t * tld + g));
                dmma884(e0, e1, __ldg(R + (size_t)(8 * a + g) * k + 8 * c + 4 + t), tload(tc + (4 + t) * tld + g));
            }
            c0 += e0;
            c1 += e1;
            // acc as the B operand of inv(R_aa) acc: through the tile's own slot (row g, cols 2t..)
            double* ta = tile(a);
            ta[g * tld + 2 * t] = c0;
            ta[g * tld + 2 * t + 1] = c1;
            __syncwarp();
            double x0 = 0.0, x1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ks += 4)
                dmma884(x0, x1, dinv8[(size_t)(8 * a + g) * 8 + ks + t], tload(ta + (ks + t) * tld + g));
            __syncwarp();
            ta[g * tld + 2 * t] = -x0;
            ta[g * tld + 2 * t + 1] = -x1;
            __syncwarp();
        }
        if (SM)
            for (int e = lane; e < 64 * (b + 1); e += 32) {
                const int a = e >> 6, i = (e >> 3) & 7, j = e & 7;
                T[(size_t)(8 * a + i) * ldt + 8 * b + j] = tsm[32 * b * (b + 1) + e];
            }
    }
}

// X (m x n) = Y (m x n) T (n x n), T upper block-triangular (8 x 8 blocks), n % 8 == 0, n <= 256.
// CTA: 64 rows x all n columns, 8 warps; warp w owns the 8-column blocks w, 15 - w, 16 + w,
// 31 - w (a snake, so the triangle's work is even across warps) for all 8 row tiles. T and Y
// stream through shared memory in 16-deep k-chunks (cp.async, two stages); a block skips the
// chunks below its diagonal.
constexpr int kMmRows = 64, kMmKc = 16, kMmYld = kMmKc + 4;
__device__ __forceinline__ void cpa16(double* smem, const double* gmem, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 16 : 0));
}
template <int NBW>
__global__ void __launch_bounds__(256, NBW <= 2 ? 2 : 1) tsmm_kernel(const double* __restrict__ Y, int m, int n, int ld,
                                                      const double* __restrict__ T, int ldt, double* __restrict__ X,
                                                      int ldx, const double* __restrict__ stats) {
    pdl_entry();
    if (stats && stats[4] != 0.0) return;
    extern __shared__ double mm[];
    const int tld = n + 4;  // conflict-free B-fragment reads (n % 16 == 0 or 8 -> tld % 16 == 4 or 12)
    const size_t stage_sz = (size_t)kMmRows * kMmYld + (size_t)kMmKc * tld;
    const int r0 = blockIdx.x * kMmRows;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nb = n / 8;
    int blk[NBW];
#pragma unroll
    for (int q = 0; q < NBW; ++q) {
        const int b = 8 * q + ((q & 1) ? 7 - w : w);
        blk[q] = b < nb ? b : -1;
    }
    auto load = [&](int stage, int kc) {
        double* Ys = mm + stage * stage_sz;
        double* Ts = Ys + kMmRows * kMmYld;
        for (int e = threadIdx.x; e < kMmRows * (kMmKc / 2); e += 256) {
            const int r = e / (kMmKc / 2), c = 2 * (e % (kMmKc / 2));
            const bool ok = r0 + r < m;
            cpa16(Ys + r * kMmYld + c, ok ? Y + (size_t)(r0 + r) * ld + kc + c : Y, ok);
        }
        for (int e = threadIdx.x; e < kMmKc * (n / 2); e += 256) {
            const int r = e / (n / 2), c = 2 * (e % (n / 2));
            cpa16(Ts + r * tld + c, T + (size_t)(kc + r) * ldt + c, true);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    double acc[8][NBW][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < NBW; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
    int stage = 0;
    load(0, 0);
    for (int kc = 0; kc < n; kc += kMmKc) {
        if (kc + kMmKc < n) {
            load(stage ^ 1, kc + kMmKc);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const double* Ys = mm + stage * stage_sz;
        const double* Ts = Ys + kMmRows * kMmYld;
#pragma unroll
        for (int ks = 0; ks < kMmKc; ks += 4) {
            double a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = Ys[(8 * i + g) * kMmYld + ks + t];
#pragma unroll
            for (int q = 0; q < NBW; ++q) {
                if (blk[q] < 0 || kc + ks > 8 * blk[q] + 7) continue;  // below the diagonal: T = 0
                const double bq = Ts[(ks + t) * tld + 8 * blk[q] + g];
#pragma unroll
                for (int i = 0; i < 8; ++i) dmma884(acc[i][q][0], acc[i][q][1], a[i], bq);
            }
        }
        __syncthreads();
        stage ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = r0 + 8 * i + g;
        if (row >= m) continue;
#pragma unroll
        for (int q = 0; q < NBW; ++q)
            if (blk[q] >= 0)
                *reinterpret_cast<double2*>(X + (size_t)row * ldx + 8 * blk[q] + 2 * t) =
                    make_double2(acc[i][q][0], acc[i][q][1]);
    }
}

}  // namespace

void chol_factor(const double* G, int k, int ldg, double* R, double* dinv8, double* T, int ldt, double* stats,
                 int* d_err, int err_bit, Scratch& scr, cudaStream_t st, bool polar, int* udrop) {
    if (k <= 0) return;
    if (k > 512) throw invalid_argument("chol_factor: k > 512 unsupported");
    ProfScope prof(polar ? "chol_polar" : "chol", st);
    prof.work((double)k * k * k / 3.0, 16.0 * (double)k * k);
    const bool use_smem = k <= kSmemMaxK;
    double* gscr = nullptr;
    size_t smem = 2 * (size_t)k * sizeof(double);
    if (use_smem) {
        smem += (size_t)k * (k + 4) * sizeof(double);
    } else {
        gscr = scr.take<double>((int64_t)k * k + 2 * k);
        smem = 0;
    }
    if (first_on_device((const void*)(chol_factor_kernel))) {
        allow_max_dynamic_smem(chol_factor_kernel);
        allow_max_dynamic_smem(trsm_apply_kernel);
    }
    LAUNCH(chol_factor_kernel, 1, kCholThreads, smem, st, G, k, ldg, R, dinv8, T, ldt, stats, d_err, err_bit, gscr,
           use_smem ? 1 : 0, polar ? 1 : 0, udrop);
}

void trsm_apply(const double* Y, int m, int k, int ld, const double* R, const double* dinv8, double* X, int ldx,
                const double* stats, cudaStream_t st, double* tinv) {
    if (m <= 0 || k <= 0) return;
    const int kp = (k + 7) / 8 * 8;
    if (kp > 512) throw invalid_argument("trsm_apply: k > 512 unsupported");
    ProfScope prof("trsm", st);
    prof.work((double)m * k * k, 16.0 * (double)m * k);  // X = Y R^-1: k^2 / 2 multiply-adds per row
    static const bool subst = std::getenv("SFDG_TRSM") && std::string(std::getenv("SFDG_TRSM")) == "subst";
    if (tinv && k % 8 == 0 && k <= 256 && ld % 2 == 0 && ldx % 2 == 0 && !subst) {
        const int nb = k / 8;
        const size_t tsmem = (size_t)32 * nb * (nb + 1) * sizeof(double);
        const bool in_smem = tsmem <= 200 * 1024;
        const unsigned threads = (unsigned)std::min(1024, 32 * nb);
        if (first_on_device((const void*)(trinv_kernel<true>))) {
            allow_max_dynamic_smem(trinv_kernel<true>);
            allow_max_dynamic_smem(tsmm_kernel<2>);
            allow_max_dynamic_smem(tsmm_kernel<4>);
        }
        if (in_smem) LAUNCH(trinv_kernel<true>, 1, threads, tsmem, st, R, k, dinv8, tinv, k, stats);
        else LAUNCH(trinv_kernel<false>, 1, threads, 0, st, R, k, dinv8, tinv, k, stats);
        const size_t msmem = 2 * ((size_t)kMmRows * kMmYld + (size_t)kMmKc * (k + 4)) * sizeof(double);
        if (nb <= 16) LAUNCH(tsmm_kernel<2>, ceil_div(m, kMmRows), 256, msmem, st, Y, m, k, ld, tinv, k, X, ldx, stats);
        else LAUNCH(tsmm_kernel<4>, ceil_div(m, kMmRows), 256, msmem, st, Y, m, k, ld, tinv, k, X, ldx, stats);
        return;
    }
    if (kp > kTrsmSmemK) {  // R streamed through shared memory one block-column panel at a time
        if (first_on_device((const void*)(trsm_panel_kernel))) {
            allow_max_dynamic_smem(trsm_panel_kernel);
        }
        int rows = 128;
        auto pbytes = [&](int r) {
            return (2 * (size_t)kp * kPanelLd + (size_t)kp * 12 + (size_t)r * (kp + 4)) * sizeof(double);
        };
        while (rows > 16 && pbytes(rows) > 220 * 1024) rows /= 2;
        LAUNCH(trsm_panel_kernel, ceil_div(m, rows), kTrsmThreads, pbytes(rows), st, Y, m, k, ld, R, dinv8, X, ldx,
               stats, rows);
        return;
    }
    const size_t rs = (size_t)kp * (kp + 4);
    int rows = 128;
    auto bytes = [&](int r) { return (rs + (size_t)kp * 12 + (size_t)r * (kp + 4)) * sizeof(double); };
    while (rows > 16 && bytes(rows) > 220 * 1024) rows /= 2;
    LAUNCH(trsm_apply_kernel, ceil_div(m, rows), kTrsmThreads, bytes(rows), st, Y, m, k, ld, R, dinv8, X, ldx, stats,
           rows);
}

void exact_orth(const double* Y, int ldy, double* Q, int ldq, int m, int k, const int* udrop, const double* stats,
                double* tmp, cudaStream_t st, bool force) {
    if (m <= 0 || k <= 0) return;
    if (k > kXMaxK) throw invalid_argument("exact_orth: k > 512 unsupported");
    ProfScope prof("exact_orth", st);
    if (first_on_device((const void*)exact_orth_kernel)) allow_max_dynamic_smem(exact_orth_kernel);
    LAUNCH(exact_orth_kernel, kXC, kXThreads, exact_orth_smem(k), st, Y, ldy, Q, ldq, m, k, udrop, stats, tmp,
           force ? 1 : 0);
}

}  // namespace sfdg
