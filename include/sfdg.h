/*
 * sfdg.h -- C ABI of the B200-native Sparse Frequent Directions sketcher.
 *
 * Drop-in boundary for the reference's C++ sketch interface
 * (/root/reference/proj/core/include/sfd/sketch.hpp:9-49,71 and shrink.hpp:26-41).
 * Plain pointers and sizes only; no exceptions cross this boundary. Every entry
 * point returns a status code that mirrors the reference's exception classes
 * (core/include/sfd/common.hpp:14-17, mapped to exit codes in tools/sfd_main.cpp:289-298):
 *
 *   SFDG_OK (0), SFDG_INVALID_ARGUMENT (1) = std::invalid_argument,
 *   SFDG_NUMERICAL_ERROR (2) = sfd::numerical_error, SFDG_CUDA_ERROR (3) = device fault.
 *
 * sfdg_last_error() returns the thread-local message of the last failure.
 *
 * Matrices are FP64 row-major like sfd::DenseMatrix (dense_matrix.hpp:10-30). Sparse
 * inputs are CSR like sfd::SparseBuffer (sparse.hpp:52-57): int64 row offsets,
 * uint32 strictly increasing column indices, FP64 values. Host pointers are read
 * before the call returns; the caller keeps ownership.
 *
 * All compute runs on the selected CUDA device (sm_100a). There is no CPU path:
 * without a usable device every compute entry point returns SFDG_CUDA_ERROR.
 */
#ifndef SFDG_H
#define SFDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFDG_OK 0
#define SFDG_INVALID_ARGUMENT 1
#define SFDG_NUMERICAL_ERROR 2
#define SFDG_CUDA_ERROR 3

/* PowerConfig (randsvd.hpp:10-14). q_override < 0 means "not set". */
typedef struct {
    double epsilon;     /* default 0.25 */
    double q_constant;  /* default 1.0  */
    int64_t q_override; /* default -1   */
} sfdg_power_config;

/* SketchConfig (sketch.hpp:9-17). */
typedef struct {
    size_t ell;
    size_t d;
    double delta; /* default 0.1 */
    sfdg_power_config power;
    uint64_t seed;
} sfdg_sketch_config;

/* Draw state of sfd::Rng (rng.hpp:12-31): std::mt19937_64(seed) after `words` raw
 * outputs, plus the cached Box-Muller spare. A fresh Rng(seed) is {seed, 0, 0, 0}. */
typedef struct {
    uint64_t seed;
    uint64_t words;
    int32_t has_spare;
    double spare;
} sfdg_rng_state;

/* VerifierState (shrink.hpp:11-16). Fresh state: {0, delta, 2.0, 0.0}. */
typedef struct {
    size_t i;
    double delta;
    double c_verify;
    double delta_spent;
} sfdg_verifier_state;

/* Accessor snapshot of SfdSketcher (sketch.hpp:35-48). */
typedef struct {
    size_t flush_count;   /* flush_count()   */
    size_t attempt_total; /* attempt_total() */
    sfdg_verifier_state verifier;
    size_t buffer_rows; /* buffer().rows()    */
    size_t buffer_nnz;  /* buffer().nnz()     */
    double buffer_frob_sq;
    sfdg_rng_state rng;
} sfdg_stats;

typedef struct sfdg_sketcher sfdg_sketcher;

const char* sfdg_last_error(void);
const char* sfdg_version(void);
/* Number of visible CUDA devices (0 on a machine without a GPU; never an error). */
int sfdg_device_count(int* count);

/* ---- SfdSketcher (sketch.hpp:22-49; sketch.cpp:9-45) -------------------------- */

/* SfdSketcher(const SketchConfig&): validates (1 <= ell <= d, 0 < delta < 1); this build also
 * requires ell <= 512 (SFDG_INVALID_ARGUMENT above: the eigensolver / CholeskyQR limits). */
int sfdg_sketcher_create(const sfdg_sketch_config* cfg, int device, sfdg_sketcher** out);
int sfdg_sketcher_destroy(sfdg_sketcher* h);

/* append(const SparseRow&) for nrows rows at once. Row r is cols/vals[row_ptr[r] ..
 * row_ptr[r+1]). Rows are committed in order exactly as repeated append() calls
 * would: the flush trigger (nnz >= ell*d || rows == d, sketch.cpp:22) is evaluated
 * after every row. A row failing validation (sparse.cpp:8-20) stops the batch with
 * SFDG_INVALID_ARGUMENT; earlier rows stay committed; *rows_done (optional) reports
 * how many were. */
int sfdg_sketcher_append_csr(sfdg_sketcher* h, const int64_t* row_ptr, const uint32_t* cols,
                             const double* vals, size_t nrows, size_t* rows_done);

/* Same, for a CSR whose cols/vals already sit in device memory of this sketcher's
 * GPU (d_cols/d_vals indexed by the host row offsets h_row_ptr). Validation and
 * the Frobenius bookkeeping run on the device. */
int sfdg_sketcher_append_csr_device(sfdg_sketcher* h, const int64_t* h_row_ptr, const uint32_t* d_cols,
                                    const double* d_vals, size_t nrows, size_t* rows_done);

/* finalize() (sketch.cpp:34-45): flushes or densify-merges the remainder, writes
 * B (ell x d, row-major) to host `out` (may be NULL). */
int sfdg_sketcher_finalize(sfdg_sketcher* h, double* out);
/* sketch(): current B (ell x d row-major) to host memory. */
int sfdg_sketcher_get_sketch(sfdg_sketcher* h, double* out);
/* Device-side B^T (d x ell, row-major, leading dimension ld >= ell) for the merge tree. */
int sfdg_sketcher_get_sketch_device(sfdg_sketcher* h, double* d_out, size_t ld);
/* flush_count(), attempt_total(), verifier(), buffer() sizes, RNG position. */
int sfdg_sketcher_stats(sfdg_sketcher* h, sfdg_stats* out);
/* buffer() contents (CSR, host): row_ptr (rows+1), cols (nnz), vals (nnz). */
int sfdg_sketcher_get_buffer(sfdg_sketcher* h, int64_t* row_ptr, uint32_t* cols, double* vals);
/* B <- merge(B, B_other) = dense_shrink(vstack(B, B_other), ell) (sketch.cpp:80-83), with
 * B_other given as B_other^T (d x ell, leading dimension ld) in device memory of this
 * sketcher's device: the receiving side of the multi-GPU merge tree, without allocation. */
int sfdg_sketcher_merge_device(sfdg_sketcher* h, const double* d_other_bt, size_t ld);
/* Returns the sketcher to its just-constructed state with a new seed (allocations kept). */
int sfdg_sketcher_reset(sfdg_sketcher* h, uint64_t seed);
/* Blocks until all queued device work of this sketcher finished. */
int sfdg_sketcher_synchronize(sfdg_sketcher* h);

/* ---- FdSketcher: dense Frequent Directions (sketch.hpp:53-67, sketch.cpp:47-78) ---
 * The paper's baseline: a 2ell x d buffer shrunk to ell rows whenever it fills. */
typedef struct sfdg_fd_sketcher sfdg_fd_sketcher;
/* FdSketcher(ell, d) (sketch.cpp:47-50); 1 <= ell <= d else SFDG_INVALID_ARGUMENT. */
int sfdg_fd_create(size_t ell, size_t d, int device, sfdg_fd_sketcher** out);
int sfdg_fd_destroy(sfdg_fd_sketcher* h);
/* append(row) for nrows dense rows (nrows x d row-major), sketch.cpp:52-63. A non-finite
 * value fails the shrink that would consume it (dense_shrink, shrink.cpp:32). */
int sfdg_fd_append(sfdg_fd_sketcher* h, const double* rows, size_t nrows);
/* Same rows given as CSR (densified on the device). */
int sfdg_fd_append_csr(sfdg_fd_sketcher* h, const int64_t* row_ptr, const uint32_t* cols, const double* vals,
                       size_t nrows);
/* finalize() (sketch.cpp:65-78): ell x d row-major into out. */
int sfdg_fd_finalize(sfdg_fd_sketcher* h, double* out);
/* shrink_count() (sketch.hpp:60). */
int sfdg_fd_shrink_count(sfdg_fd_sketcher* h, size_t* count);

/* ---- free functions (shrink.hpp:26-41, sketch.hpp:71, randsvd.hpp:18-26) ------- */

/* merge(b1, b2, ell) = dense_shrink(vstack(b1, b2), ell)  (sketch.cpp:80-83). */
int sfdg_merge(const double* b1, size_t rows1, const double* b2, size_t rows2, size_t d, size_t ell,
               double* out, int device);
/* Device-resident merge for the shard tree: inputs/outputs are B^T (d x ell, leading
 * dimension ld) on `device`; `stream` is a cudaStream_t (NULL = legacy default). */
int sfdg_merge_device(const double* d_b1t, const double* d_b2t, size_t ell, size_t d, size_t ld,
                      double* d_outt, int device, void* stream);
/* Row-sharded sketch of one stream (the multi-GPU entry). Shard g holds the
 * contiguous rows [g*ceil(n/G), (g+1)*ceil(n/G)) and is sketched with seed + g on
 * devices[g % ndev] (one host thread per shard); the shard sketches then meet in the
 * log2 tree -- at level L shard r (r % 2^(L+1) == 2^L) is peer-copied to r - 2^L, which
 * computes merge(B_lo, B_hi) (sketch.cpp:80-83) -- and `out` (ell x d) receives the root.
 * Replaces the caller-side loop of tests/acceptance.cpp:420-445 (shard, sketch, merge).
 * shard_stats (nullable) receives the G per-shard counters. */
int sfdg_sharded_sketch(const sfdg_sketch_config* cfg, const int64_t* row_ptr, const uint32_t* cols,
                        const double* vals, size_t nrows, int shards, const int* devices, int ndev, double* out,
                        sfdg_stats* shard_stats);
/* ---- ingestion (io.hpp:13-33, io.cpp:21-189) ----------------
 * Sketch a row-stream file: MatrixMarket "matrix coordinate real general" (1-based,
 * entries grouped by nondecreasing row) or, with plain_cols > 0, the plain "col:value"
 * format -- the reference's open_row_stream + run_sketch (tools/sfd_main.cpp:65-69).
 * cfg->d = 0 takes the file's column count (else it must match). The file is memory-mapped
 * and parsed by all host threads window by window while the device sketches the previous
 * window. out: ell x d (row-major); stats and *d_out optional. */
int sfdg_sketch_file(const char* path, size_t plain_cols, const sfdg_sketch_config* cfg, int device, double* out,
                     sfdg_stats* stats, size_t* d_out);
/* The parsed rows themselves (CSR, absolute row_ptr): call with NULL arrays to get the
 * sizes, then with arrays of nrows + 1, nnz, nnz entries. */
int sfdg_read_row_stream(const char* path, size_t plain_cols, size_t* nrows, size_t* d, size_t* nnz,
                         int64_t* row_ptr, uint32_t* cols, double* vals);
/* cov_err(a, sketch, rng, iterations) (bench.hpp:62-64, bench.cpp:171-183):
 * |A^T A - B^T B|_2 / |A|_F^2 by `iterations` power steps (la_core.cpp:191-211) from
 * unit_sphere_vector(d, rng); A is n x d CSR (host), B is ell x d row-major (host). The
 * whole-stream evaluation metric of SURVEY 8(f); rng advanced in place. */
int sfdg_cov_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d,
                 const double* b, size_t ell, size_t iterations, sfdg_rng_state* rng, double* out, int device);
/* exact_tail(a, k, rng) (bench.hpp:51-55, bench.cpp:68-137): the ground-truth tail
 * |A - A_k|_F^2 and the top-k singular values of the whole stream by block power iteration
 * (block k + 10 <= 512, <= 1000 sweeps, the reference's convergence tests); *sweeps_out = the
 * sweeps run (nullable). k = 0 returns |A|_F^2. rng advanced in place. */
int sfdg_exact_tail(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d, size_t k,
                    sfdg_rng_state* rng, double* sigma_out, double* tail_out, size_t* sweeps_out, int device);
/* proj_err(a, sketch, k, tail) (bench.hpp:57-60, bench.cpp:139-169): |A - A V_k V_k^T|_F^2 /
 * tail_sq with V_k the sketch's top-k right singular vectors; *has_value = 0 for the
 * reference's nullopt cases (rank <= k input, sketch without a k-dimensional span). */
int sfdg_proj_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d, const double* b,
                  size_t ell, size_t k, double tail_sq, double* out, int* has_value, int device);
/* dense_shrink(a, ell) (shrink.cpp:30-61), host in/out. */
int sfdg_dense_shrink(const double* a, size_t rows, size_t cols, size_t ell, double* out, int device);
/* sparse_shrink(buffer, ell, power, rng) (shrink.cpp:63-73); rng advanced in place. */
int sfdg_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                       size_t ell, const sfdg_power_config* power, sfdg_rng_state* rng, double* out,
                       int device);
/* boosted_sparse_shrink (shrink.cpp:104-131); verifier and rng advanced in place. */
int sfdg_boosted_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m,
                               size_t d, size_t ell, sfdg_verifier_state* verifier,
                               const sfdg_power_config* power, sfdg_rng_state* rng, double* out,
                               double* delta_hat, size_t* attempts, int device);
/* simultaneous_iteration (randsvd.cpp:18-51): orthonormal basis Z (m x k) of the
 * dominant left subspace; rng advanced in place. */
int sfdg_simultaneous_iteration(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m,
                                size_t d, size_t k, const sfdg_power_config* power, sfdg_rng_state* rng,
                                double* z_out, int device);
/* power_iteration_count (randsvd.cpp:10-16). */
int sfdg_power_iteration_count(size_t m, const sfdg_power_config* power, size_t* q);

/* A symmetric operator y = C x on R^d supplied by the caller (la_core.hpp:45 SymOp). It
 * returns 0 on success; a nonzero return aborts the verification with SFDG_INVALID_ARGUMENT.
 * x and y are d doubles: host memory, or memory of `device` when op_on_device != 0. */
typedef int (*sfdg_symop_fn)(const double* x, double* y, size_t d, void* user);
/* verify_spectral(apply, d, state, rng) (shrink.hpp:35, shrink.cpp:75-102) over a caller
 * operator: state->i += 1, delta_i = delta / (2 i^2) added to delta_spent, steps =
 * ceil(c_verify log2(d / delta_i)); x = unit_sphere_vector(d, rng) (la_core.cpp:174-189) drawn
 * from the device generator at *rng (advanced in place); then the log-domain power method with
 * the reference's exits (annihilation -> accept, |.| >= 1 while the log magnitude is positive
 * -> reject, non-finite output -> SFDG_NUMERICAL_ERROR). *accepted = 1 / 0. With
 * op_on_device the iterate never leaves the GPU (norms and rescaling on the device). */
int sfdg_verify_spectral(sfdg_symop_fn op, void* user, int op_on_device, size_t d, sfdg_verifier_state* state,
                         sfdg_rng_state* rng, int* accepted, int device);

/* ---- device kernels exposed for parity tests (la_core.hpp:23-41) --------------- */

/* gaussian_matrix(rows, cols, rng) (la_core.cpp:167-172) generated on the device. */
int sfdg_gaussian_matrix(sfdg_rng_state* rng, size_t rows, size_t cols, double* out, int device);
/* jacobi_eigh contract (la_core.cpp:24-80): eigenvalues descending + eigenvectors
 * (column k, n x n row-major) of a symmetric matrix, off-diagonal tolerance off_tol. */
int sfdg_eigh(const double* sym, size_t n, double off_tol, double* values, double* vectors, int device);
/* orthonormalize contract (la_core.cpp:130-165) via device CholeskyQR2 with the same
 * column-drop rule (n x k, n >= k). */
int sfdg_orthonormalize(const double* in, size_t n, size_t k, double* out, int device);
/* Sparse products of SparseBuffer (sparse.cpp:32-69) on the device:
 * y = A x (m x k, x: d x k), w = A^T z (d x k, z: m x k). Either output may be NULL. */
int sfdg_csr_products(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                      size_t k, const double* x, double* y, const double* z, double* w, int device);

/* Per-kernel-class device timing with CUDA events on the launching stream (off by
 * default). profile_end writes {"class": [total_ms, launches], ...} into buf. */
int sfdg_profile_begin(void);
int sfdg_profile_end(char* buf, size_t n);

/* Process-wide count of kernels this library launched (benchmark gpu_launches claim). */
uint64_t sfdg_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SFDG_H */
