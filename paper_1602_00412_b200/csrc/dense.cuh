// dense.cuh -- FP64 dense kernels (see dense.cu, chol.cu, eigh.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sparse.cuh"

namespace sfdg {

// out (k x k, ldo) = X^T X, X: n x k row-major (ldx). Deterministic.
void gram_tn(const double* X, int n, int k, int ldx, double* out, int ldo, Scratch& scr, cudaStream_t st);
// C (n x c, ldc) = X (n x k, ldx) * S (k x c, lds). C must not alias X or S.
// pred (optional, device): the kernel only runs when *pred != 0.
void gemm_nn(const double* X, int n, int k, int ldx, const double* S, int c, int lds, double* C, int ldc,
             cudaStream_t st, const double* pred = nullptr);
// *d_out = sum of squares of X (rows x cols, ld); sets err_bit in *d_err on non-finite.
void sumsq(const double* X, int64_t rows, int cols, int ld, double* d_out, int* d_err, int err_bit, Scratch& scr,
           cudaStream_t st);
void transpose(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st);
// x[i] *= s for i < n.
void scale_vector(double* x, int64_t n, double s, cudaStream_t st);
void copy2d(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st);
void fill2d(double* out, int rows, int cols, int ldo, double v, cudaStream_t st);

// CholeskyQR (chol.cu). chol_factor: from the Gram G (k x k) of a tall Y, the upper
// Cholesky factor R (k x k) and the inverses of its 8 x 8 diagonal blocks (dinv8, k x 8);
// columns whose residual pivot falls below the drop rule get a zero row in R and a zero
// column in dinv8 (la_core.cpp:141,157-162). stats (8 doubles): [0] min relative pivot,
// [1] dropped columns, [2] max|G - I|, [3] max R_jj / min R_jj, [4] polar path taken,
// [5] running max of [3], [6] uncertain drops (udrop, below), [7] running sum of [6].
// polar = true (second pass): T = I - (G - I)/2 into T (k x k, ldt) when max|G - I| <=
// 1e-6, else the Cholesky path. trsm_apply: X = Y R^-1 (skipped when stats[4] != 0).
void chol_factor(const double* G, int k, int ldg, double* R, double* dinv8, double* T, int ldt, double* stats,
                 int* d_err, int err_bit, Scratch& scr, cudaStream_t st, bool polar, int* udrop = nullptr);
// tinv (k x k workspace, optional): apply as T = R^-1 formed once + a DMMA GEMM (k % 8 == 0,
// k <= 256) instead of the row-wise substitution; SFDG_TRSM=subst forces the substitution.
void trsm_apply(const double* Y, int m, int k, int ld, const double* R, const double* dinv8, double* X, int ldx,
                const double* stats, cudaStream_t st, double* tinv = nullptr);
// The reference's orthonormalize (la_core.cpp:130-165) exactly, for the columns CholeskyQR
// cannot decide: when stats[6] > 0 (or force), re-derives the drop of every uncertain column
// (udrop[j]) from its explicit residual against the CholeskyQR result Q (two classical
// Gram-Schmidt passes, the reference's absolute threshold 1e-12 max_j |y_j|); if any of them
// would be kept, Q is recomputed from Y by Gram-Schmidt with re-orthogonalisation and the
// reference's drop rule. One 8-CTA cluster (DSMEM reductions); a no-op launch otherwise.
// tmp: m doubles.
void exact_orth(const double* Y, int ldy, double* Q, int ldq, int m, int k, const int* udrop, const double* stats,
                double* tmp, cudaStream_t st, bool force = false);

// Symmetric eigensolver (eigh.cu), the jacobi_eigh contract (la_core.cpp:24-80):
// values descending (n), vectors column k (n x n, ldv). off_tol is absolute, or, when
// d_fsq != nullptr, 1e-12 * max(*d_fsq, 1) read on the device (svd_top's rule,
// la_core.cpp:103). A non-converged solve after 100 sweeps sets ERR_JACOBI_NOCONV.
// nval: only the top nval eigenpairs are required (the default n = all). The fast path is
// eigh_tri.cu (tridiagonal + bisection + inverse iteration); the Jacobi solver runs as a
// device-predicated fallback or when SFDG_EIGH=jacobi.
void eigh(const double* K, int n, int ldk, double off_tol, const double* d_fsq, double* values, double* vectors,
          int ldv, int* d_err, Scratch& scr, cudaStream_t st, int nval = 0);

}  // namespace sfdg
