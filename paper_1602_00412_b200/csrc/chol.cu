// chol.cu -- CholeskyQR factor step with the reference's column-drop rule.
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
// Second pass (mode kPolar): after one CholeskyQR pass, G = Q^T Q = I + E with tiny E.
// Then T = I - E/2 gives (QT)^T(QT) = I - 3/4 E^2 + O(E^3): orthonormal to O(|E|^2)
// with the same span, without a sequential factorisation. When max|E| > kPolarMax the
// kernel falls back to the full Cholesky path, so accuracy never depends on the guess.
//
// One CTA; the k x k Gram lives in shared memory (k <= 160) or L2-resident scratch.
// Layout: upper triangle = R, strictly lower triangle = off-diagonal of Rinv^T, dinv[k].
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr double kRelDrop = 1e-13;  // ~ 4 k u for k <= 256
constexpr double kPolarMax = 1e-6;  // |E|^2 <= 1e-12 relative -> far below the 1e-8 gate
constexpr int kCholThreads = 512;
constexpr int kSmemMaxK = 160;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kCholThreads) chol_rinv_kernel(const double* __restrict__ G, int k, int ldg,
                                                                 double* __restrict__ Rinv, int ldr,
                                                                 double* __restrict__ stats, int* __restrict__ err,
                                                                 int err_bit, double* __restrict__ gscratch,
                                                                 int use_smem, int polar) {
    extern __shared__ double sm[];
    const int lda = use_smem ? k + 1 : k;
    double* A = use_smem ? sm : gscratch;
    double* d0 = A + (size_t)k * lda;  // original diagonal
    double* dinv = d0 + k;             // 1 / R_jj (0 for dropped)
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
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, j = e % k;
        const double v = G[(size_t)i * ldg + j];
        if (!isfinite(v)) s_bad = 1;
        if (j >= i) A[(size_t)i * lda + j] = v;
        if (i == j) {
            d0[i] = v;
            mx = fmax(mx, v);
        }
    }
    __syncthreads();
    if (polar) {  // max |G - I| over the kept (nonzero-diagonal) columns
        for (int e = tid; e < k * k; e += nt) {
            const int i = e / k, j = e % k;
            if (j < i || d0[i] == 0.0 || d0[j] == 0.0) continue;
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
        for (int e = tid; e < k * k; e += nt) Rinv[(size_t)(e / k) * ldr + e % k] = 0.0;
        if (tid == 0) atomicOr(err, err_bit);
        return;
    }

    if (polar && s_emax <= kPolarMax) {
        // T = I - E/2 on kept columns, zero rows/columns for dropped ones (Q_j = 0 stays 0)
        for (int e = tid; e < k * k; e += nt) {
            const int i = e / k, j = e % k;
            double v = 0.0;
            if (d0[i] != 0.0 && d0[j] != 0.0) {
                const double g = i <= j ? A[(size_t)i * lda + j] : A[(size_t)j * lda + i];
                v = (i == j ? 1.0 : 0.0) - 0.5 * (g - (i == j ? 1.0 : 0.0));
            }
            Rinv[(size_t)i * ldr + j] = v;
        }
        if (tid == 0) {
            stats[0] = 1.0;
            stats[1] = 0.0;
            stats[2] = s_emax;
        }
        return;
    }

    // ---- right-looking Cholesky, one barrier per column. Warp 0 owns the pivot chain:
    // it updates row j+1 with row j, then pivots and scales row j+1, while the other
    // warps update rows j+2.. with row j.
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
            dinv[j] = keep ? ri : 0.0;
            if (!keep) {
                s_drop[j] = 1;
                s_dropped += 1;
            }
        }
        __syncwarp();
    };
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
            // rows i >= j+2, columns c >= i: flattened over the trailing block
            const int base = j + 2, rem = k - base;
            for (int e = tid - 32; e < rem * rem; e += nt - 32) {
                const int i = base + e / rem, c = base + e % rem;
                if (c >= i) A[(size_t)i * lda + c] -= rj[i] * rj[c];
            }
        }
        __syncthreads();
    }

    // ---- Rinv = R^-1. Column c of Rinv by back substitution, one warp per column,
    // x_i (i < c) stored in the strictly lower triangle row c: A[c][i].
    const int qend = ((k + nw - 1) / nw) * nw;
    for (int q = warp; q < qend; q += nw) {
        const int round = q / nw, pos = q % nw;
        const int c = (round & 1) ? round * nw + (nw - 1 - pos) : q;  // snake order balances cost
        if (c >= k) continue;
        const double xc = dinv[c];
        for (int i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int l = i + 1 + lane; l <= c; l += 32) {
                const double xl = (l == c) ? xc : A[(size_t)c * lda + l];
                s = fma(A[(size_t)i * lda + l], xl, s);
            }
            s = warp_sum(s);
            if (lane == 0) A[(size_t)c * lda + i] = -s * dinv[i];
            __syncwarp();
        }
    }
    __syncthreads();
    // Dropped j: dinv[j] = 0 zeroes column j (Q_j = 0, la_core.cpp:158-159) and row j
    // of R is zero, so no kept column sees y_j.
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, c = e % k;
        double v = 0.0;
        if (i == c) v = dinv[c];
        else if (i < c) v = s_drop[c] ? 0.0 : A[(size_t)c * lda + i];
        Rinv[(size_t)i * ldr + c] = v;
    }
    if (tid == 0) {
        double mn = 1.0;
        for (int j = 0; j < k; ++j)
            if (!s_drop[j] && d0[j] > 0.0) {
                const double r = A[(size_t)j * lda + j];
                mn = fmin(mn, r * r / d0[j]);
            }
        stats[0] = mn;
        stats[1] = (double)s_dropped;
        stats[2] = s_emax;
    }
}

}  // namespace

void chol_rinv(const double* G, int k, int ldg, double* Rinv, int ldr, double* stats, int* d_err, int err_bit,
               Scratch& scr, cudaStream_t st, bool polar) {
    if (k <= 0) return;
    if (k > 512) throw invalid_argument("chol_rinv: k > 512 unsupported");
    ProfScope prof(polar ? "chol_polar" : "chol", st);
    const bool use_smem = k <= kSmemMaxK;
    double* gscr = nullptr;
    size_t smem = 3 * (size_t)k * sizeof(double);
    if (use_smem) {
        smem += (size_t)k * (k + 1) * sizeof(double);
    } else {
        gscr = scr.take<double>((int64_t)k * k + 2 * k);
        smem = 0;
    }
    static bool attr_set = false;
    if (!attr_set) {
        allow_max_dynamic_smem(chol_rinv_kernel);
        attr_set = true;
    }
    LAUNCH(chol_rinv_kernel, 1, kCholThreads, smem, st, G, k, ldg, Rinv, ldr, stats, d_err, err_bit, gscr,
           use_smem ? 1 : 0, polar ? 1 : 0);
}

}  // namespace sfdg
