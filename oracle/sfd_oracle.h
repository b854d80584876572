/*
 * sfd_oracle.h -- CPU restatement of the reference SparseFrequentDirections path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity oracle for the B200 path. Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it. The product library (paper_1602_00412_b200/libsfdg.so) never
 * links, loads or calls anything here.
 *
 * Every function restates the reference algorithm at the cited file:line of
 * /root/reference/proj (read-only, not copied). Arithmetic order follows the
 * reference loop for loop, so with the same compiler flags (-O3, no -march, no
 * FMA contraction) it is bit-identical to the reference; tests/test_oracle_pin.py
 * checks exactly that against oracle/_ref (the reference compiled from its own
 * sources) and against the committed golden fixtures in tests/golden/.
 *
 * Status codes mirror the reference exception classes (core/include/sfd/common.hpp:14-17):
 *   0 ok, 1 std::invalid_argument, 2 sfd::numerical_error.
 */
#ifndef SFD_ORACLE_H
#define SFD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_OK 0
#define OR_INVALID 1
#define OR_NUMERICAL 2

/* ---- Rng (core/include/sfd/rng.hpp:12-31, core/src/rng.cpp:9-34) ---- */
typedef struct or_rng or_rng;
or_rng* or_rng_new(uint64_t seed);
void or_rng_free(or_rng* r);
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_uniform(or_rng* r);
uint64_t or_rng_uniform_below(or_rng* r, uint64_t n);
double or_rng_normal(or_rng* r);
/* Number of normals drawn so far (offset into the normal stream). */
uint64_t or_rng_normals_drawn(const or_rng* r);
/* Full draw state: raw words consumed, cached Box-Muller spare. */
void or_rng_state(const or_rng* r, uint64_t* words, int* has_spare, double* spare);

/* ---- power_iteration_count (core/src/randsvd.cpp:10-16) ---- */
/* q_override < 0 means "no override". */
int or_power_iteration_count(size_t m, double epsilon, double q_constant, long long q_override,
                             size_t* q_out);

/* ---- dense linear algebra (core/src/la_core.cpp) ---- */
/* values (n), vectors (n x n row-major, column k = eigenvector k) */
int or_jacobi_eigh(const double* sym, size_t n, double off_tol, double* values, double* vectors);
/* singular (r), right (d x r row-major); left optional (m x r) */
int or_svd_top(const double* a, size_t m, size_t d, size_t r, double* singular, double* right,
               double* left, int* rank_deficient);
int or_orthonormalize(const double* in, size_t n, size_t k, double* out);

/* ---- shrink (core/src/shrink.cpp) ---- */
int or_dense_shrink(const double* a, size_t rows, size_t cols, size_t ell, double* out /* ell x cols */);

typedef struct {
    double epsilon;      /* default 0.25 */
    double q_constant;   /* default 1.0  */
    long long q_override;/* < 0: none    */
} or_power_cfg;

typedef struct {
    size_t i;
    double delta;
    double c_verify;
    double delta_spent;
} or_verifier;

/* CSR view: row_ptr (m+1, int64), cols (uint32), vals (f64) */
typedef struct {
    const int64_t* row_ptr;
    const uint32_t* cols;
    const double* vals;
    size_t m;
    size_t d;
} or_csr;

int or_simultaneous_iteration(const or_csr* a, size_t k, const or_power_cfg* cfg, or_rng* rng,
                              double* z_out /* m x k */);
int or_sparse_shrink(const or_csr* a, size_t ell, const or_power_cfg* cfg, or_rng* rng,
                     double* out /* ell x d */);
typedef void (*or_symop)(const double* x, double* y, size_t d, void* ctx);
int or_verify_spectral(or_symop op, void* ctx, size_t d, or_verifier* st, or_rng* rng, int* accepted);
int or_boosted_sparse_shrink(const or_csr* a, size_t ell, or_verifier* st, const or_power_cfg* cfg,
                             or_rng* rng, double* out /* ell x d */, double* delta_hat,
                             size_t* attempts);
int or_merge(const double* b1, size_t r1, const double* b2, size_t r2, size_t d, size_t ell,
             double* out);

/* ---- cov_err (core/include/sfd/bench.hpp:62-64, core/src/bench.cpp:171-183) ----
 * |A^T A - B^T B|_2 / |A|_F^2 by `iterations` power steps from unit_sphere_vector(d, rng). */
int or_cov_err(const or_csr* a, const double* sketch, size_t ell, or_rng* rng, size_t iterations, double* out);

/* ---- exact_tail (core/include/sfd/bench.hpp:51-55, core/src/bench.cpp:68-137) ----
 * |A - A_k|_F^2 and the top-k singular values; *sweeps_out = block sweeps run. */
int or_exact_tail(const or_csr* a, size_t k, or_rng* rng, double* sigma_out, double* tail_out, size_t* sweeps_out);

/* ---- proj_err (core/include/sfd/bench.hpp:57-60, core/src/bench.cpp:139-169) ---- */
int or_proj_err(const or_csr* a, const double* sketch, size_t ell, size_t k, double tail_sq, double* out,
                int* has_value);

/* ---- FdSketcher (core/include/sfd/sketch.hpp:53-67, core/src/sketch.cpp:47-78) ----
 * Whole-stream dense FD: n rows (n x d row-major) -> B (ell x d), shrink count. */
int or_fd_sketch(const double* rows, size_t n, size_t d, size_t ell, double* out, size_t* shrink_count);

/* ---- SfdSketcher (core/include/sfd/sketch.hpp:22-49, core/src/sketch.cpp:9-45) ---- */
typedef struct or_sketcher or_sketcher;
typedef struct {
    size_t ell;
    size_t d;
    double delta;
    or_power_cfg power;
    uint64_t seed;
} or_sketch_cfg;

int or_sketcher_new(const or_sketch_cfg* cfg, or_sketcher** out);
void or_sketcher_free(or_sketcher* s);
/* Appends nrows rows (CSR with row_ptr relative to row_ptr[0]). Rows are committed
 * one at a time exactly like SfdSketcher::append; on a bad row the rows before it
 * stay committed and *rows_done reports how many were. */
int or_sketcher_append_csr(or_sketcher* s, const int64_t* row_ptr, const uint32_t* cols,
                           const double* vals, size_t nrows, size_t* rows_done);
int or_sketcher_finalize(or_sketcher* s, double* out /* ell x d */);
void or_sketcher_get_sketch(const or_sketcher* s, double* out);
void or_sketcher_stats(const or_sketcher* s, size_t* flushes, size_t* attempts, size_t* verifier_i,
                       double* delta_spent, size_t* buf_rows, size_t* buf_nnz, double* buf_frob_sq,
                       uint64_t* normals_drawn);
/* densified buffer (rows x d) */
void or_sketcher_buffer_dense(const or_sketcher* s, double* out);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
