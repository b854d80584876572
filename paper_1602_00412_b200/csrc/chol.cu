// chol.cu -- CholeskyQR factor step with the reference's column-drop rule.
//
// Reference: orthonormalize (core/src/la_core.cpp:130-165) runs modified Gram-Schmidt
// with one re-orthogonalisation pass and zeroes a column whose residual norm falls
// below 1e-12 * (largest input column norm). On the GPU the same span is produced by
// CholeskyQR2: G = Y^T Y (DMMA, dense.cu), G = R^T R here, Y <- Y R^-1, twice. The
// Cholesky pivot R_jj^2 is exactly column j's squared residual after projecting out the
// kept columns 0..j-1, so the MGS drop rule becomes a pivot test. A Gram-formed pivot
// carries O(k u G_jj) cancellation error, so a pivot below kRelDrop * G_jj is treated as
// numerically dependent and dropped as well (SURVEY sec 7 hard part 2).
//
// One CTA factors the k x k Gram in shared memory (k <= 128) or in L2-resident global
// scratch (k > 128), then inverts R with one warp per column (back substitution).
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr double kRelDrop = 1e-13;  // ~ 4 k u for k <= 256
constexpr int kCholThreads = 1024;

__global__ void __launch_bounds__(kCholThreads) chol_rinv_kernel(const double* __restrict__ G, int k, int ldg,
                                                                 double* __restrict__ Rinv, int ldr,
                                                                 double* __restrict__ stats, int* __restrict__ err,
                                                                 int err_bit, double* __restrict__ gscratch,
                                                                 int use_smem) {
    extern __shared__ double sm[];
    const int lda = use_smem ? k + 1 : k;
    double* A = use_smem ? sm : gscratch;
    double* d0 = use_smem ? sm + (size_t)k * lda : gscratch + (size_t)k * k;  // original diagonal
    __shared__ double s_r, s_thr, s_minrel;
    __shared__ int s_keep, s_bad, s_dropped;
    __shared__ double red[32];
    __shared__ int s_drop[512];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j = tid; j < k; j += nt) s_drop[j] = 0;

    if (tid == 0) {
        s_bad = 0;
        s_dropped = 0;
        s_minrel = 1.0;
    }
    __syncthreads();
    double mx = 0.0;
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, j = e % k;
        const double v = G[(size_t)i * ldg + j];
        if (!isfinite(v)) s_bad = 1;
        A[(size_t)i * lda + j] = v;
        if (i == j) {
            d0[i] = v;
            mx = fmax(mx, v);
        }
    }
    // block max of the diagonal (largest squared input column norm)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < (nt + 31) / 32; ++w) m = fmax(m, red[w]);
        const double drop_tol = 1e-12 * sqrt(m);  // la_core.cpp:141
        s_thr = drop_tol * drop_tol;
    }
    __syncthreads();
    if (s_bad) {
        for (int e = tid; e < k * k; e += nt) Rinv[(size_t)(e / k) * ldr + e % k] = 0.0;
        if (tid == 0) atomicOr(err, err_bit);
        return;
    }

    for (int j = 0; j < k; ++j) {
        if (tid == 0) {
            const double piv = A[(size_t)j * lda + j];
            const bool keep = isfinite(piv) && piv > s_thr && piv > kRelDrop * d0[j] && piv > 0.0;
            s_keep = keep;
            if (keep) {
                s_r = sqrt(piv);
                s_minrel = fmin(s_minrel, piv / d0[j]);
            } else {
                s_dropped += 1;
                s_drop[j] = 1;
            }
        }
        __syncthreads();
        const bool keep = s_keep;
        const double r = s_r;
        for (int c = j + tid; c < k; c += nt) {
            double* a = A + (size_t)j * lda + c;
            if (keep) *a = (c == j) ? r : *a / r;
            else *a = (c == j) ? 1.0 : 0.0;  // dropped: unit pivot, zero row (fixed up below)
        }
        __syncthreads();
        if (keep) {
            const int rem = k - j - 1;
            for (int e = tid; e < rem * rem; e += nt) {
                const int i = j + 1 + e / rem, c = j + 1 + e % rem;
                if (c >= i) A[(size_t)i * lda + c] -= A[(size_t)j * lda + i] * A[(size_t)j * lda + c];
            }
        }
        __syncthreads();
    }

    // Rinv: warp per column c solves R x = e_c by back substitution.
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int qend = ((k + nw - 1) / nw) * nw;
    for (int q = warp; q < qend; q += nw) {
        // snake order balances the O(c) column costs across warps
        const int round = q / nw, pos = q % nw;
        const int c = (round & 1) ? round * nw + (nw - 1 - pos) : q;
        if (c >= k) continue;
        // x_i for i > c is 0; x lives in Rinv[:, c] (global), read back by the same warp.
        for (int i = c; i >= 0; --i) {
            double s = 0.0;
            for (int l = i + 1 + lane; l <= c; l += 32) s = fma(A[(size_t)i * lda + l], Rinv[(size_t)l * ldr + c], s);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double x = ((i == c ? 1.0 : 0.0) - s) / A[(size_t)i * lda + i];
            if (lane == 0) Rinv[(size_t)i * ldr + c] = x;
            __syncwarp();
        }
        for (int i = c + 1 + lane; i < k; i += 32) Rinv[(size_t)i * ldr + c] = 0.0;
        __syncwarp();
    }
    __syncthreads();
    // Dropped columns: Q_j = 0 (la_core.cpp:158-159) -> zero column j of Rinv. Row j of
    // Rinv is already e_j^T (zero row of R), so no kept column sees y_j.
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, c = e % k;
        if (s_drop[c]) Rinv[(size_t)i * ldr + c] = 0.0;
    }
    if (tid == 0) {
        stats[0] = s_minrel;
        stats[1] = (double)s_dropped;
    }
}

}  // namespace

}  // namespace sfdg

namespace sfdg {

void chol_rinv(const double* G, int k, int ldg, double* Rinv, int ldr, double* stats, int* d_err, int err_bit,
               Scratch& scr, cudaStream_t st) {
    if (k <= 0) return;
    if (k > 512) throw invalid_argument("chol_rinv: k > 512 unsupported");
    ProfScope prof("chol", st);
    const bool use_smem = k <= 128;
    double* gscr = nullptr;
    size_t smem = 0;
    if (use_smem) {
        smem = ((size_t)k * (k + 1) + k) * sizeof(double);
    } else {
        gscr = scr.take<double>((int64_t)k * k + k);
    }
    static bool attr_set = false;
    if (!attr_set) {
        allow_max_dynamic_smem(chol_rinv_kernel);
        attr_set = true;
    }
    LAUNCH(chol_rinv_kernel, 1, kCholThreads, smem, st, G, k, ldg, Rinv, ldr, stats, d_err, err_bit, gscr,
           use_smem ? 1 : 0);
}

}  // namespace sfdg
