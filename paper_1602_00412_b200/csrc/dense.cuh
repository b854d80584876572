// dense.cuh -- FP64 dense kernels (see dense.cu, chol.cu, eigh.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sparse.cuh"

namespace sfdg {

// out (k x k, ldo) = X^T X, X: n x k row-major (ldx). Deterministic.
void gram_tn(const double* X, int n, int k, int ldx, double* out, int ldo, Scratch& scr, cudaStream_t st);
// C (n x c, ldc) = X (n x k, ldx) * S (k x c, lds). C must not alias X or S.
void gemm_nn(const double* X, int n, int k, int ldx, const double* S, int c, int lds, double* C, int ldc,
             cudaStream_t st);
// *d_out = sum of squares of X (rows x cols, ld); sets err_bit in *d_err on non-finite.
void sumsq(const double* X, int64_t rows, int cols, int ld, double* d_out, int* d_err, int err_bit, Scratch& scr,
           cudaStream_t st);
void transpose(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st);
void copy2d(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t st);
void fill2d(double* out, int rows, int cols, int ldo, double v, cudaStream_t st);

// CholeskyQR factor step (chol.cu): from the Gram G (k x k) of a tall Y, the upper
// triangular Rinv with Y Rinv orthonormal; columns whose residual pivot falls below
// the drop rule are zeroed (la_core.cpp:141,157-162). stats[0] = min relative pivot
// of the kept columns, stats[1] = number of dropped columns, stats[2] = max|G - I|.
// polar = true (second CholeskyQR pass): T = I - (G - I)/2 when max|G - I| <= 1e-6,
// otherwise the full Cholesky path.
void chol_rinv(const double* G, int k, int ldg, double* Rinv, int ldr, double* stats, int* d_err, int err_bit,
               Scratch& scr, cudaStream_t st, bool polar = false);

// Symmetric eigensolver (eigh.cu), the jacobi_eigh contract (la_core.cpp:24-80):
// values descending (n), vectors column k (n x n, ldv). off_tol is absolute, or, when
// d_fsq != nullptr, 1e-12 * max(*d_fsq, 1) read on the device (svd_top's rule,
// la_core.cpp:103). A non-converged solve after 100 sweeps sets ERR_JACOBI_NOCONV.
void eigh(const double* K, int n, int ldk, double off_tol, const double* d_fsq, double* values, double* vectors,
          int ldv, int* d_err, Scratch& scr, cudaStream_t st);

}  // namespace sfdg
