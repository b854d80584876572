/*
 * sfd_oracle.c -- plain-C restatement of the reference SFD hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see sfd_oracle.h). Never linked into the product.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Loop order and operation order follow the reference so
 * that, compiled with the reference's Release flags (-O3, no -march), results are
 * bit-identical; tests/test_oracle_pin.py pins this against oracle/_ref.
 *
 * Error model: the reference throws std::invalid_argument / sfd::numerical_error.
 * Here every public entry point runs inside an arena + setjmp frame; a thrown
 * error longjmps back to the entry point, frees the arena and returns 1 or 2.
 */
#include "sfd_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* error + arena plumbing                                                      */
/* ------------------------------------------------------------------------- */

static __thread char g_err[512];

typedef struct arena_blk {
    struct arena_blk* next;
    double pad; /* keeps the payload 16-byte aligned */
} arena_blk;

typedef struct {
    jmp_buf jb;
    arena_blk* blocks;
} frame;

static __thread frame* g_frame;

const char* or_last_error(void) { return g_err; }

static _Noreturn void raise_err(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    longjmp(g_frame->jb, code);
}
#define THROW_INVALID(...) raise_err(OR_INVALID, __VA_ARGS__)
#define THROW_NUMERICAL(...) raise_err(OR_NUMERICAL, __VA_ARGS__)

static void* az(size_t n) { /* zeroed arena allocation */
    arena_blk* b = (arena_blk*)calloc(1, sizeof(arena_blk) + (n ? n : 1));
    if (!b) THROW_NUMERICAL("oracle: out of memory");
    b->next = g_frame->blocks;
    g_frame->blocks = b;
    return (void*)(b + 1);
}

static void arena_free(frame* f) {
    arena_blk* b = f->blocks;
    while (b) {
        arena_blk* n = b->next;
        free(b);
        b = n;
    }
    f->blocks = NULL;
}

#define ENTER()                                  \
    frame fr_;                                   \
    fr_.blocks = NULL;                           \
    frame* saved_ = g_frame;                     \
    g_frame = &fr_;                              \
    int st_ = setjmp(fr_.jb);                    \
    if (st_ != 0) {                              \
        arena_free(&fr_);                        \
        g_frame = saved_;                        \
        return st_;                              \
    }                                            \
    g_err[0] = 0
#define LEAVE()           \
    arena_free(&fr_);     \
    g_frame = saved_;     \
    return OR_OK

/* ------------------------------------------------------------------------- */
/* dense matrix (core/include/sfd/dense_matrix.hpp:10-30; dense_matrix.cpp)    */
/* ------------------------------------------------------------------------- */

typedef struct {
    size_t rows, cols;
    double* data; /* row-major */
} mat;

static mat mat_new(size_t r, size_t c) {
    mat m;
    m.rows = r;
    m.cols = c;
    m.data = (double*)az(r * c * sizeof(double));
    return m;
}
#define AT(m, i, j) ((m).data[(size_t)(i) * (m).cols + (size_t)(j)])

/* dense_matrix.cpp:8-12 */
static double frob_sq(const mat* m) {
    double s = 0.0;
    for (size_t i = 0; i < m->rows * m->cols; ++i) s += m->data[i] * m->data[i];
    return s;
}
/* dense_matrix.cpp:14-18 */
static int all_finite(const mat* m) {
    for (size_t i = 0; i < m->rows * m->cols; ++i)
        if (!isfinite(m->data[i])) return 0;
    return 1;
}
/* dense_matrix.cpp:20-28 */
static mat vstack(const mat* a, const mat* b) {
    if (a->cols != b->cols && a->rows != 0 && b->rows != 0) THROW_INVALID("vstack: column mismatch");
    size_t cols = a->rows != 0 ? a->cols : b->cols;
    mat out = mat_new(a->rows + b->rows, cols);
    memcpy(out.data, a->data, a->rows * a->cols * sizeof(double));
    memcpy(out.data + a->rows * a->cols, b->data, b->rows * b->cols * sizeof(double));
    return out;
}
/* dense_matrix.cpp:30-40 */
static void dmatvec(const mat* m, const double* x, double* y) {
    for (size_t i = 0; i < m->rows; ++i) {
        const double* r = m->data + i * m->cols;
        double s = 0.0;
        for (size_t j = 0; j < m->cols; ++j) s += r[j] * x[j];
        y[i] = s;
    }
}
/* dense_matrix.cpp:42-52 */
static void dtmatvec(const mat* m, const double* y, double* x) {
    for (size_t j = 0; j < m->cols; ++j) x[j] = 0.0;
    for (size_t i = 0; i < m->rows; ++i) {
        const double* r = m->data + i * m->cols;
        const double yi = y[i];
        if (yi == 0.0) continue;
        for (size_t j = 0; j < m->cols; ++j) x[j] += yi * r[j];
    }
}

/* ------------------------------------------------------------------------- */
/* Rng: std::mt19937_64 + fixed-formula draws (rng.hpp:12-31, rng.cpp:9-34)    */
/* ------------------------------------------------------------------------- */

#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

struct or_rng {
    uint64_t mt[MT_N];
    int mti;
    double spare;
    int has_spare;
    uint64_t normals;
    uint64_t words; /* raw engine outputs consumed */
};

/* std::mt19937_64(seed) state initialisation ([rand.eng.mers], f = 6364136223846793005). */
static void mt_seed(or_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
}

static uint64_t mt_next(or_rng* r) {
    if (r->mti >= MT_N) {
        int i;
        uint64_t x;
        for (i = 0; i < MT_N - MT_M; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        for (; i < MT_N - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        x = (r->mt[MT_N - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        r->mti = 0;
    }
    r->words += 1;
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

or_rng* or_rng_new(uint64_t seed) {
    or_rng* r = (or_rng*)calloc(1, sizeof(or_rng));
    if (r) mt_seed(r, seed);
    return r;
}
void or_rng_free(or_rng* r) { free(r); }
uint64_t or_rng_next_u64(or_rng* r) { return mt_next(r); }
/* rng.hpp:19 */
double or_rng_uniform(or_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }
/* rng.cpp:9-17 (n == 0 is rejected by the caller-facing wrapper) */
uint64_t or_rng_uniform_below(or_rng* r, uint64_t n) {
    if (n == 0) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do {
        v = mt_next(r);
    } while (v >= limit);
    return v % n;
}
/* rng.cpp:19-34: Box-Muller pair, cos returned first, sin cached as the spare. */
double or_rng_normal(or_rng* r) {
    r->normals += 1;
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1;
    do {
        u1 = or_rng_uniform(r);
    } while (u1 <= 0.0);
    const double u2 = or_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}
uint64_t or_rng_normals_drawn(const or_rng* r) { return r->normals; }
void or_rng_state(const or_rng* r, uint64_t* words, int* has_spare, double* spare) {
    *words = r->words;
    *has_spare = r->has_spare;
    *spare = r->spare;
}

/* ------------------------------------------------------------------------- */
/* la_core (core/src/la_core.cpp)                                              */
/* ------------------------------------------------------------------------- */

/* la_core.cpp:14-20 */
static double off_diag_norm_sq(const mat* s) {
    double acc = 0.0;
    for (size_t i = 0; i < s->rows; ++i)
        for (size_t j = 0; j < s->cols; ++j)
            if (i != j) acc += AT(*s, i, j) * AT(*s, i, j);
    return acc;
}

typedef struct {
    double* values;
    mat vectors;
} eigh_t;

/* la_core.cpp:24-80: cyclic Jacobi; stable sort by descending diagonal. */
static eigh_t jacobi_eigh(const mat* sym, double off_tol) {
    if (sym->rows != sym->cols) THROW_INVALID("jacobi_eigh: matrix not square");
    const size_t n = sym->rows;
    mat s = mat_new(n, n);
    memcpy(s.data, sym->data, n * n * sizeof(double));
    mat v = mat_new(n, n);
    for (size_t i = 0; i < n; ++i) AT(v, i, i) = 1.0;

    const double tol_sq = off_tol * off_tol;
    const size_t max_sweeps = 100;
    size_t sweep = 0;
    while (off_diag_norm_sq(&s) > tol_sq && n > 1) {
        if (++sweep > max_sweeps) THROW_NUMERICAL("jacobi_eigh: no convergence after 100 sweeps");
        for (size_t p = 0; p + 1 < n; ++p) {
            for (size_t q = p + 1; q < n; ++q) {
                const double apq = AT(s, p, q);
                if (apq == 0.0) continue;
                const double theta = (AT(s, q, q) - AT(s, p, p)) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double sn = t * c;
                for (size_t i = 0; i < n; ++i) {
                    const double sip = AT(s, i, p);
                    const double siq = AT(s, i, q);
                    AT(s, i, p) = c * sip - sn * siq;
                    AT(s, i, q) = sn * sip + c * siq;
                }
                for (size_t j = 0; j < n; ++j) {
                    const double spj = AT(s, p, j);
                    const double sqj = AT(s, q, j);
                    AT(s, p, j) = c * spj - sn * sqj;
                    AT(s, q, j) = sn * spj + c * sqj;
                }
                for (size_t i = 0; i < n; ++i) {
                    const double vip = AT(v, i, p);
                    const double viq = AT(v, i, q);
                    AT(v, i, p) = c * vip - sn * viq;
                    AT(v, i, q) = sn * vip + c * viq;
                }
            }
        }
    }

    /* std::stable_sort(order, s(a,a) > s(b,b)): stable insertion sort. */
    size_t* order = (size_t*)az(n * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) order[i] = i;
    for (size_t i = 1; i < n; ++i) {
        size_t key = order[i];
        size_t j = i;
        while (j > 0 && AT(s, key, key) > AT(s, order[j - 1], order[j - 1])) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = key;
    }
    eigh_t out;
    out.values = (double*)az(n * sizeof(double));
    out.vectors = mat_new(n, n);
    for (size_t k = 0; k < n; ++k) {
        out.values[k] = AT(s, order[k], order[k]);
        for (size_t i = 0; i < n; ++i) AT(out.vectors, i, k) = AT(v, i, order[k]);
    }
    return out;
}

typedef struct {
    mat left;
    double* singular;
    mat right;
    int rank_deficient;
} svd_t;

/* la_core.cpp:82-128: Gram route top-r SVD of a short-fat matrix. */
static svd_t svd_top(const mat* a, size_t r) {
    if (a->rows > a->cols) THROW_INVALID("svd_top: expects m <= d");
    if (r < 1 || r > a->rows) THROW_INVALID("svd_top: rank out of range");
    if (!all_finite(a)) THROW_INVALID("svd_top: non-finite input");
    const size_t m = a->rows, d = a->cols;
    mat gram = mat_new(m, m);
    for (size_t i = 0; i < m; ++i) {
        const double* ri = a->data + i * d;
        for (size_t j = i; j < m; ++j) {
            const double* rj = a->data + j * d;
            double s = 0.0;
            for (size_t t = 0; t < d; ++t) s += ri[t] * rj[t];
            AT(gram, i, j) = s;
            AT(gram, j, i) = s;
        }
    }
    const double fsq = frob_sq(a);
    eigh_t eig = jacobi_eigh(&gram, 1e-12 * (fsq > 1.0 ? fsq : 1.0));

    svd_t out;
    out.left = mat_new(m, r);
    out.right = mat_new(d, r);
    out.singular = (double*)az(r * sizeof(double));
    out.rank_deficient = 0;
    for (size_t k = 0; k < r; ++k) {
        out.singular[k] = sqrt(eig.values[k] > 0.0 ? eig.values[k] : 0.0);
        for (size_t i = 0; i < m; ++i) AT(out.left, i, k) = AT(eig.vectors, i, k);
    }
    const double cutoff = 1e-10 * out.singular[0];
    for (size_t k = 0; k < r; ++k) {
        if (out.singular[k] < cutoff || out.singular[k] == 0.0) {
            out.rank_deficient = 1;
            continue;
        }
        for (size_t i = 0; i < m; ++i) {
            const double w = AT(out.left, i, k) / out.singular[k];
            if (w == 0.0) continue;
            const double* ri = a->data + i * d;
            for (size_t t = 0; t < d; ++t) AT(out.right, t, k) += w * ri[t];
        }
    }
    return out;
}

/* la_core.cpp:130-165: MGS with one re-orthogonalisation pass and column drop. */
static mat orthonormalize(const mat* m) {
    if (m->rows < m->cols) THROW_INVALID("orthonormalize: needs n >= k");
    const size_t n = m->rows, k = m->cols;
    double max_norm = 0.0;
    for (size_t j = 0; j < k; ++j) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += AT(*m, i, j) * AT(*m, i, j);
        const double nj = sqrt(s);
        max_norm = max_norm > nj ? max_norm : nj;
    }
    const double drop_tol = 1e-12 * max_norm;
    mat q = mat_new(n, k);
    memcpy(q.data, m->data, n * k * sizeof(double));
    for (size_t j = 0; j < k; ++j) {
        for (int pass = 0; pass < 2; ++pass) {
            for (size_t p = 0; p < j; ++p) {
                double proj = 0.0;
                for (size_t i = 0; i < n; ++i) proj += AT(q, i, p) * AT(q, i, j);
                if (proj == 0.0) continue;
                for (size_t i = 0; i < n; ++i) AT(q, i, j) -= proj * AT(q, i, p);
            }
        }
        double nn = 0.0;
        for (size_t i = 0; i < n; ++i) nn += AT(q, i, j) * AT(q, i, j);
        const double norm = sqrt(nn);
        if (norm < drop_tol || norm == 0.0) {
            for (size_t i = 0; i < n; ++i) AT(q, i, j) = 0.0;
        } else {
            for (size_t i = 0; i < n; ++i) AT(q, i, j) /= norm;
        }
    }
    return q;
}

/* la_core.cpp:167-172 */
static mat gaussian_matrix(size_t rows, size_t cols, or_rng* rng) {
    if (rows < 1 || cols < 1) THROW_INVALID("gaussian_matrix: empty shape");
    mat g = mat_new(rows, cols);
    for (size_t i = 0; i < rows * cols; ++i) g.data[i] = or_rng_normal(rng);
    return g;
}

/* la_core.cpp:174-189 */
static double* unit_sphere_vector(size_t d, or_rng* rng) {
    if (d < 1) THROW_INVALID("unit_sphere_vector: d must be positive");
    double* x = (double*)az(d * sizeof(double));
    for (;;) {
        double nrm_sq = 0.0;
        for (size_t i = 0; i < d; ++i) {
            x[i] = or_rng_normal(rng);
            nrm_sq += x[i] * x[i];
        }
        if (nrm_sq > 0.0) {
            const double inv = 1.0 / sqrt(nrm_sq);
            for (size_t i = 0; i < d; ++i) x[i] *= inv;
            return x;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* sparse buffer products (core/src/sparse.cpp)                                */
/* ------------------------------------------------------------------------- */

/* sparse.cpp:32-43 */
static void sp_matvec(const or_csr* a, const double* x, double* y) {
    for (size_t i = 0; i < a->m; ++i) {
        double s = 0.0;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) s += a->vals[k] * x[a->cols[k]];
        y[i] = s;
    }
}
/* sparse.cpp:45-55 (rows with y_i == 0 skipped) */
static void sp_rmatvec(const or_csr* a, const double* y, double* x) {
    for (size_t j = 0; j < a->d; ++j) x[j] = 0.0;
    for (size_t i = 0; i < a->m; ++i) {
        const double yi = y[i];
        if (yi == 0.0) continue;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) x[a->cols[k]] += yi * a->vals[k];
    }
}
/* sparse.cpp:57-69: P = Z^T A' (z.cols x d) */
static mat sp_project_rows(const or_csr* a, const mat* z) {
    if (z->rows != a->m) THROW_INVALID("project_rows: row mismatch");
    mat p = mat_new(z->cols, a->d);
    for (size_t i = 0; i < a->m; ++i) {
        const double* zr = z->data + i * z->cols;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
            const double v = a->vals[k];
            const uint32_t j = a->cols[k];
            for (size_t t = 0; t < z->cols; ++t) AT(p, t, j) += zr[t] * v;
        }
    }
    return p;
}

static double csr_frob_sq(const or_csr* a) { /* running sum in row order, sparse.cpp:22 */
    double f = 0.0;
    for (int64_t k = a->row_ptr[0]; k < a->row_ptr[a->m]; ++k) f += a->vals[k] * a->vals[k];
    return f;
}

/* ------------------------------------------------------------------------- */
/* randsvd (core/src/randsvd.cpp)                                              */
/* ------------------------------------------------------------------------- */

/* randsvd.cpp:10-16 */
static size_t power_iteration_count(size_t m, const or_power_cfg* cfg) {
    if (cfg->q_override >= 0) return (size_t)cfg->q_override;
    if (cfg->epsilon <= 0.0 || cfg->epsilon >= 1.0)
        THROW_INVALID("power_iteration_count: epsilon must be in (0,1)");
    const double q = cfg->q_constant * log((double)(m > 1 ? m : 1) / cfg->epsilon) / cfg->epsilon;
    const size_t qc = (size_t)ceil(q);
    return qc > 1 ? qc : 1;
}

/* randsvd.cpp:18-51 */
static mat simultaneous_iteration(const or_csr* a, size_t k, const or_power_cfg* cfg, or_rng* rng) {
    const size_t m = a->m, d = a->d;
    if (k < 1 || k > (m < d ? m : d)) THROW_INVALID("simultaneous_iteration: k out of range");
    const size_t q = power_iteration_count(m, cfg);
    mat g = gaussian_matrix(d, k, rng);
    double* col = (double*)az(d * sizeof(double));
    double* yc = (double*)az(m * sizeof(double));
    mat y = mat_new(m, k);
    for (size_t j = 0; j < k; ++j) {
        for (size_t i = 0; i < d; ++i) col[i] = AT(g, i, j);
        sp_matvec(a, col, yc);
        for (size_t i = 0; i < m; ++i) AT(y, i, j) = yc[i];
    }
    y = orthonormalize(&y);
    double* ycol = (double*)az(m * sizeof(double));
    double* w = (double*)az(d * sizeof(double));
    for (size_t sweep = 0; sweep < q; ++sweep) {
        mat next = mat_new(m, k);
        for (size_t j = 0; j < k; ++j) {
            for (size_t i = 0; i < m; ++i) ycol[i] = AT(y, i, j);
            sp_rmatvec(a, ycol, w);
            sp_matvec(a, w, yc);
            for (size_t i = 0; i < m; ++i) AT(next, i, j) = yc[i];
        }
        if (!all_finite(&next)) THROW_NUMERICAL("simultaneous_iteration: non-finite intermediate");
        y = orthonormalize(&next);
    }
    return y;
}

/* ------------------------------------------------------------------------- */
/* shrink (core/src/shrink.cpp)                                                */
/* ------------------------------------------------------------------------- */

#define RETRY_CAP 64 /* shrink.cpp:12 */
static const double kAlpha = 6.0 / 41.0; /* common.hpp:10 */

/* shrink.cpp:15-26 */
static mat shrink_from_factors(const double* singular, const mat* right, size_t ell) {
    const size_t d = right->rows;
    const double floor_sq = singular[ell - 1] * singular[ell - 1];
    mat b = mat_new(ell, d);
    for (size_t i = 0; i < ell; ++i) {
        const double dd = singular[i] * singular[i] - floor_sq;
        const double shrunk = sqrt(dd > 0.0 ? dd : 0.0);
        if (shrunk == 0.0) continue;
        for (size_t j = 0; j < d; ++j) AT(b, i, j) = shrunk * AT(*right, j, i);
    }
    return b;
}

/* shrink.cpp:30-61 */
static mat dense_shrink(const mat* a, size_t ell) {
    if (ell < 1 || ell > a->rows) THROW_INVALID("dense_shrink: ell out of range");
    if (!all_finite(a)) THROW_INVALID("dense_shrink: non-finite input");
    if (a->rows <= a->cols) {
        svd_t svd = svd_top(a, ell);
        return shrink_from_factors(svd.singular, &svd.right, ell);
    }
    if (ell > a->cols) THROW_INVALID("dense_shrink: ell exceeds column count");
    const size_t d = a->cols;
    mat gram = mat_new(d, d);
    for (size_t i = 0; i < a->rows; ++i) {
        const double* r = a->data + i * d;
        for (size_t p = 0; p < d; ++p) {
            if (r[p] == 0.0) continue;
            for (size_t q = p; q < d; ++q) AT(gram, p, q) += r[p] * r[q];
        }
    }
    for (size_t p = 0; p < d; ++p)
        for (size_t q = 0; q < p; ++q) AT(gram, p, q) = AT(gram, q, p);
    const double fsq = frob_sq(a);
    eigh_t eig = jacobi_eigh(&gram, 1e-12 * (fsq > 1.0 ? fsq : 1.0));
    double* singular = (double*)az(ell * sizeof(double));
    mat right = mat_new(d, ell);
    for (size_t k = 0; k < ell; ++k) {
        singular[k] = sqrt(eig.values[k] > 0.0 ? eig.values[k] : 0.0);
        for (size_t j = 0; j < d; ++j) AT(right, j, k) = AT(eig.vectors, j, k);
    }
    return shrink_from_factors(singular, &right, ell);
}

/* shrink.cpp:63-73 */
static mat sparse_shrink(const or_csr* a, size_t ell, const or_power_cfg* cfg, or_rng* rng) {
    if (ell < 1 || ell > a->m) THROW_INVALID("sparse_shrink: ell out of range");
    if (ell > a->d) THROW_INVALID("sparse_shrink: ell exceeds column count");
    mat z = simultaneous_iteration(a, ell, cfg, rng);
    mat p = sp_project_rows(a, &z);
    if (!all_finite(&p)) THROW_NUMERICAL("sparse_shrink: non-finite projection");
    svd_t svd = svd_top(&p, ell);
    return shrink_from_factors(svd.singular, &svd.right, ell);
}

/* shrink.cpp:75-102 */
static int verify_spectral(or_symop op, void* ctx, size_t d, or_verifier* st, or_rng* rng) {
    st->i += 1;
    const double di = (double)st->i;
    const double delta_i = st->delta / (2.0 * di * di);
    st->delta_spent += delta_i;
    const size_t steps = (size_t)ceil(st->c_verify * log2((double)d / delta_i));
    double* x = unit_sphere_vector(d, rng);
    double* y = (double*)az(d * sizeof(double));
    double log_mag = 0.0;
    for (size_t t = 0; t < steps; ++t) {
        op(x, y, d, ctx);
        double nrm_sq = 0.0;
        for (size_t i = 0; i < d; ++i) {
            if (!isfinite(y[i])) THROW_NUMERICAL("verify_spectral: non-finite operator output");
            nrm_sq += y[i] * y[i];
        }
        if (nrm_sq == 0.0) return 1;
        const double nrm = sqrt(nrm_sq);
        log_mag += log(nrm);
        if (log_mag > 0.0 && nrm >= 1.0) return 0;
        for (size_t i = 0; i < d; ++i) x[i] = y[i] / nrm;
    }
    return log_mag <= 0.0;
}

/* shrink.cpp:121-126: (2/Delta)(A'^T A' x - B'^T B' x) */
typedef struct {
    const or_csr* a;
    const mat* b;
    double scale;
    double *tm, *tl, *t2;
} diff_ctx;

static void diff_op(const double* x, double* y, size_t d, void* vctx) {
    diff_ctx* c = (diff_ctx*)vctx;
    sp_matvec(c->a, x, c->tm);
    sp_rmatvec(c->a, c->tm, y);        /* ata */
    dmatvec(c->b, x, c->tl);
    dtmatvec(c->b, c->tl, c->t2);      /* btb */
    for (size_t i = 0; i < d; ++i) y[i] = c->scale * (y[i] - c->t2[i]);
}

/* shrink.cpp:104-131 */
static mat boosted_sparse_shrink(const or_csr* a, size_t ell, or_verifier* st, const or_power_cfg* cfg,
                                 or_rng* rng, double* delta_hat_out, size_t* attempts_out) {
    if (ell < 1 || ell > a->m) THROW_INVALID("boosted_sparse_shrink: ell out of range");
    const double a_fsq = csr_frob_sq(a);
    for (size_t attempt = 1; attempt <= RETRY_CAP; ++attempt) {
        mat b = sparse_shrink(a, ell, cfg, rng);
        const double drop = a_fsq - frob_sq(&b);
        const double delta_hat = drop / (kAlpha * (double)ell);
        if (drop <= 1e-12 * a_fsq) {
            *delta_hat_out = 0.0;
            *attempts_out = attempt;
            return b;
        }
        diff_ctx c;
        c.a = a;
        c.b = &b;
        c.scale = 2.0 / delta_hat;
        c.tm = (double*)az(a->m * sizeof(double));
        c.tl = (double*)az(b.rows * sizeof(double));
        c.t2 = (double*)az(a->d * sizeof(double));
        if (verify_spectral(diff_op, &c, a->d, st, rng)) {
            *delta_hat_out = delta_hat;
            *attempts_out = attempt;
            return b;
        }
    }
    THROW_NUMERICAL("boosted_sparse_shrink: retry cap exceeded");
    return mat_new(0, 0); /* unreachable */
}

/* ------------------------------------------------------------------------- */
/* public wrappers                                                             */
/* ------------------------------------------------------------------------- */

int or_power_iteration_count(size_t m, double epsilon, double q_constant, long long q_override,
                             size_t* q_out) {
    ENTER();
    or_power_cfg c = {epsilon, q_constant, q_override};
    *q_out = power_iteration_count(m, &c);
    LEAVE();
}

int or_jacobi_eigh(const double* sym, size_t n, double off_tol, double* values, double* vectors) {
    ENTER();
    mat s = {n, n, (double*)sym};
    eigh_t e = jacobi_eigh(&s, off_tol);
    memcpy(values, e.values, n * sizeof(double));
    memcpy(vectors, e.vectors.data, n * n * sizeof(double));
    LEAVE();
}

int or_svd_top(const double* a, size_t m, size_t d, size_t r, double* singular, double* right,
               double* left, int* rank_deficient) {
    ENTER();
    mat am = {m, d, (double*)a};
    svd_t s = svd_top(&am, r);
    memcpy(singular, s.singular, r * sizeof(double));
    memcpy(right, s.right.data, d * r * sizeof(double));
    if (left) memcpy(left, s.left.data, m * r * sizeof(double));
    if (rank_deficient) *rank_deficient = s.rank_deficient;
    LEAVE();
}

int or_orthonormalize(const double* in, size_t n, size_t k, double* out) {
    ENTER();
    mat m = {n, k, (double*)in};
    mat q = orthonormalize(&m);
    memcpy(out, q.data, n * k * sizeof(double));
    LEAVE();
}

int or_dense_shrink(const double* a, size_t rows, size_t cols, size_t ell, double* out) {
    ENTER();
    mat am = {rows, cols, (double*)a};
    mat b = dense_shrink(&am, ell);
    memcpy(out, b.data, ell * cols * sizeof(double));
    LEAVE();
}

static void check_csr(const or_csr* a) {
    if (a->row_ptr[0] != 0) THROW_INVALID("csr: row_ptr[0] must be 0");
}

int or_simultaneous_iteration(const or_csr* a, size_t k, const or_power_cfg* cfg, or_rng* rng,
                              double* z_out) {
    ENTER();
    check_csr(a);
    mat z = simultaneous_iteration(a, k, cfg, rng);
    memcpy(z_out, z.data, a->m * k * sizeof(double));
    LEAVE();
}

int or_sparse_shrink(const or_csr* a, size_t ell, const or_power_cfg* cfg, or_rng* rng, double* out) {
    ENTER();
    check_csr(a);
    mat b = sparse_shrink(a, ell, cfg, rng);
    memcpy(out, b.data, ell * a->d * sizeof(double));
    LEAVE();
}

int or_verify_spectral(or_symop op, void* ctx, size_t d, or_verifier* st, or_rng* rng, int* accepted) {
    ENTER();
    *accepted = verify_spectral(op, ctx, d, st, rng);
    LEAVE();
}

int or_boosted_sparse_shrink(const or_csr* a, size_t ell, or_verifier* st, const or_power_cfg* cfg,
                             or_rng* rng, double* out, double* delta_hat, size_t* attempts) {
    ENTER();
    check_csr(a);
    mat b = boosted_sparse_shrink(a, ell, st, cfg, rng, delta_hat, attempts);
    memcpy(out, b.data, ell * a->d * sizeof(double));
    LEAVE();
}

/* sketch.cpp:80-83 */
int or_merge(const double* b1, size_t r1, const double* b2, size_t r2, size_t d, size_t ell,
             double* out) {
    ENTER();
    mat m1 = {r1, d, (double*)b1}, m2 = {r2, d, (double*)b2};
    mat st = vstack(&m1, &m2);
    mat b = dense_shrink(&st, ell);
    memcpy(out, b.data, ell * d * sizeof(double));
    LEAVE();
}

/* ------------------------------------------------------------------------- */
/* Evaluation metric: cov_err (core/src/bench.cpp:171-183) over                */
/* spectral_norm_sym (core/src/la_core.cpp:191-211).                           */
/* ------------------------------------------------------------------------- */

/* la_core.cpp:191-211: Rayleigh quotient after `iterations` normalised power steps */
static double spectral_norm_sym(or_symop op, void* ctx, size_t d, size_t iterations, or_rng* rng) {
    if (iterations < 1) THROW_INVALID("spectral_norm_sym: iterations must be >= 1");
    double* x = unit_sphere_vector(d, rng);
    double* y = (double*)az(d * sizeof(double));
    double rayleigh = 0.0;
    for (size_t it = 0; it < iterations; ++it) {
        op(x, y, d, ctx);
        double dot = 0.0, nrm_sq = 0.0;
        for (size_t i = 0; i < d; ++i) {
            if (!isfinite(y[i])) THROW_NUMERICAL("spectral_norm_sym: non-finite operator output");
            dot += x[i] * y[i];
            nrm_sq += y[i] * y[i];
        }
        rayleigh = dot;
        if (nrm_sq == 0.0) return 0.0; /* operator annihilated the iterate */
        const double inv = 1.0 / sqrt(nrm_sq);
        for (size_t i = 0; i < d; ++i) x[i] = y[i] * inv;
    }
    return rayleigh;
}

/* bench.cpp:68-137: |A - A_k|_F^2 by block power iteration (block k + 10, <= 1000 sweeps) */
int or_exact_tail(const or_csr* a, size_t k, or_rng* rng, double* sigma_out /* k */, double* tail_out,
                  size_t* sweeps_out) {
    ENTER();
    const double fsq = csr_frob_sq(a);
    *sweeps_out = 0;
    if (k == 0) {
        *tail_out = fsq;
        LEAVE();
    }
    const size_t m = a->m, d = a->d;
    if (k > (m < d ? m : d)) THROW_INVALID("exact_tail: k exceeds matrix rank bound");
    size_t block = k + 10;
    if (block > (m < d ? m : d)) block = m < d ? m : d;
    mat g = gaussian_matrix(d, block, rng);
    double* col = (double*)az(d * sizeof(double));
    double* yc = (double*)az(m * sizeof(double));
    mat y = mat_new(m, block);
    for (size_t j = 0; j < block; ++j) {
        for (size_t i = 0; i < d; ++i) col[i] = AT(g, i, j);
        sp_matvec(a, col, yc);
        for (size_t i = 0; i < m; ++i) AT(y, i, j) = yc[i];
    }
    y = orthonormalize(&y);
    double* prev = (double*)az(k * sizeof(double));
    for (size_t i = 0; i < k; ++i) prev[i] = -1.0;
    double prev_energy = -1.0;
    double* ycol = (double*)az(m * sizeof(double));
    double* wc = (double*)az(d * sizeof(double));
    double* est = (double*)az(k * sizeof(double));
    for (size_t sweep = 0; sweep < 1000; ++sweep) {
        mat w = mat_new(d, block);
        mat next = mat_new(m, block);
        for (size_t j = 0; j < block; ++j) {
            for (size_t i = 0; i < m; ++i) ycol[i] = AT(y, i, j);
            sp_rmatvec(a, ycol, wc);
            for (size_t i = 0; i < d; ++i) AT(w, i, j) = wc[i];
            sp_matvec(a, wc, yc);
            for (size_t i = 0; i < m; ++i) AT(next, i, j) = yc[i];
        }
        mat small = mat_new(block, block);
        for (size_t p = 0; p < block; ++p)
            for (size_t q = p; q < block; ++q) {
                double s = 0.0;
                for (size_t i = 0; i < d; ++i) s += AT(w, i, p) * AT(w, i, q);
                AT(small, p, q) = s;
                AT(small, q, p) = s;
            }
        eigh_t eig = jacobi_eigh(&small, 1e-14 * (fsq > 1.0 ? fsq : 1.0));
        for (size_t i = 0; i < k; ++i) est[i] = sqrt(eig.values[i] > 0.0 ? eig.values[i] : 0.0);
        double change = 0.0;
        for (size_t i = 0; i < k; ++i) {
            const double c = fabs(est[i] - prev[i]);
            if (c > change) change = c;
        }
        const double scale = est[0] > 1.0 ? est[0] : 1.0;
        double head = 0.0;
        for (size_t i = 0; i < k; ++i) head += est[i] * est[i];
        const int values_done = sweep > 0 && change <= 1e-10 * scale;
        const int energy_done = sweep >= 30 && fabs(head - prev_energy) <= 1e-9 * (head > 1.0 ? head : 1.0);
        if (values_done || energy_done) {
            memcpy(sigma_out, est, k * sizeof(double));
            *tail_out = fsq - head > 0.0 ? fsq - head : 0.0;
            *sweeps_out = sweep + 1;
            LEAVE();
        }
        memcpy(prev, est, k * sizeof(double));
        prev_energy = head;
        y = orthonormalize(&next);
    }
    THROW_NUMERICAL("exact_tail: no convergence within 1000 sweeps");
}

/* bench.cpp:139-169: |A - A V_k V_k^T|_F^2 / tail (V_k from svd_top of the sketch);
 * *has_value = 0 for the reference's nullopt cases. */
int or_proj_err(const or_csr* a, const double* sketch, size_t ell, size_t k, double tail_sq, double* out,
                int* has_value) {
    ENTER();
    *has_value = 0;
    *out = 0.0;
    if (k < 1 || k > ell) THROW_INVALID("proj_err: k out of range");
    if (tail_sq < 1e-12 * csr_frob_sq(a)) { /* rank <= k input */
        LEAVE();
    }
    mat b = {ell, a->d, (double*)sketch};
    svd_t svd = svd_top(&b, k);
    if (svd.singular[0] == 0.0 || svd.singular[k - 1] < 1e-10 * svd.singular[0]) {
        LEAVE();
    }
    double num = 0.0;
    double* proj = (double*)az(k * sizeof(double));
    for (size_t i = 0; i < a->m; ++i) {
        for (size_t t = 0; t < k; ++t) proj[t] = 0.0;
        double row_sq = 0.0;
        for (int64_t p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
            const double v = a->vals[p];
            row_sq += v * v;
            const uint32_t j = a->cols[p];
            for (size_t t = 0; t < k; ++t) proj[t] += AT(svd.right, j, t) * v;
        }
        double proj_sq = 0.0;
        for (size_t t = 0; t < k; ++t) proj_sq += proj[t] * proj[t];
        num += row_sq - proj_sq;
    }
    *out = (num > 0.0 ? num : 0.0) / tail_sq;
    *has_value = 1;
    LEAVE();
}

/* bench.cpp:171-183: |A^T A - B^T B|_2 / |A|_F^2 */
int or_cov_err(const or_csr* a, const double* sketch, size_t ell, or_rng* rng, size_t iterations, double* out) {
    ENTER();
    const double fsq = csr_frob_sq(a);
    if (fsq == 0.0) {
        *out = 0.0;
        LEAVE();
    }
    mat b = {ell, a->d, (double*)sketch};
    diff_ctx c;
    c.a = a;
    c.b = &b;
    c.scale = 1.0;
    c.tm = (double*)az(a->m * sizeof(double));
    c.tl = (double*)az(ell * sizeof(double));
    c.t2 = (double*)az(a->d * sizeof(double));
    *out = spectral_norm_sym(diff_op, &c, a->d, iterations, rng) / fsq;
    LEAVE();
}

/* ------------------------------------------------------------------------- */
/* FdSketcher (core/src/sketch.cpp:47-78): dense Frequent Directions baseline. */
/* Whole-stream run over n dense rows (n x d row-major).                       */
/* ------------------------------------------------------------------------- */

int or_fd_sketch(const double* rows, size_t n, size_t d, size_t ell, double* out /* ell x d */,
                 size_t* shrink_count) {
    ENTER();
    if (ell < 1 || ell > d) THROW_INVALID("FdSketcher: requires 1 <= ell <= d"); /* sketch.cpp:48-49 */
    mat work = mat_new(2 * ell, d);
    size_t fill = 0, shrinks = 0;
    for (size_t i = 0; i < n; ++i) { /* append (sketch.cpp:52-63) */
        memcpy(work.data + fill * d, rows + i * d, d * sizeof(double));
        fill += 1;
        if (fill == 2 * ell) {
            mat shrunk = dense_shrink(&work, ell);
            memset(work.data, 0, 2 * ell * d * sizeof(double));
            memcpy(work.data, shrunk.data, ell * d * sizeof(double));
            fill = ell;
            shrinks += 1;
        }
    }
    if (fill > ell) { /* finalize (sketch.cpp:65-78) */
        mat live = {fill, d, work.data};
        mat shrunk = dense_shrink(&live, ell);
        memset(work.data, 0, 2 * ell * d * sizeof(double));
        memcpy(work.data, shrunk.data, ell * d * sizeof(double));
        fill = ell;
        shrinks += 1;
    }
    memcpy(out, work.data, ell * d * sizeof(double));
    *shrink_count = shrinks;
    LEAVE();
}

/* ------------------------------------------------------------------------- */
/* SfdSketcher (core/src/sketch.cpp:9-45)                                      */
/* ------------------------------------------------------------------------- */

struct or_sketcher {
    or_sketch_cfg cfg;
    double* b; /* ell x d */
    /* SparseBuffer (sparse.hpp:19-57) */
    int64_t* row_ptr;
    uint32_t* cols;
    double* vals;
    size_t rows, nnz, cap_rows, cap_nnz;
    double frob;
    or_verifier ver;
    or_rng rng;
    size_t flushes, attempts;
};

/* sketch.cpp:9-12 */
static void validate_cfg(const or_sketch_cfg* c) {
    if (c->ell < 1 || c->ell > c->d) THROW_INVALID("SketchConfig: requires 1 <= ell <= d");
    if (c->delta <= 0.0 || c->delta >= 1.0) THROW_INVALID("SketchConfig: delta must be in (0,1)");
}

int or_sketcher_new(const or_sketch_cfg* cfg, or_sketcher** out) {
    ENTER();
    validate_cfg(cfg);
    or_sketcher* s = (or_sketcher*)calloc(1, sizeof(or_sketcher));
    s->cfg = *cfg;
    s->b = (double*)calloc(cfg->ell * cfg->d, sizeof(double));
    s->cap_rows = 16;
    s->cap_nnz = 64;
    s->row_ptr = (int64_t*)calloc(s->cap_rows + 1, sizeof(int64_t));
    s->cols = (uint32_t*)malloc(s->cap_nnz * sizeof(uint32_t));
    s->vals = (double*)malloc(s->cap_nnz * sizeof(double));
    s->ver.i = 0;
    s->ver.delta = cfg->delta;
    s->ver.c_verify = 2.0;
    s->ver.delta_spent = 0.0;
    mt_seed(&s->rng, cfg->seed);
    s->rng.has_spare = 0;
    s->rng.normals = 0;
    s->rng.words = 0;
    *out = s;
    LEAVE();
}

void or_sketcher_free(or_sketcher* s) {
    if (!s) return;
    free(s->b);
    free(s->row_ptr);
    free(s->cols);
    free(s->vals);
    free(s);
}

/* sketch.cpp:25-32 */
static void sk_flush(or_sketcher* s) {
    or_csr a = {s->row_ptr, s->cols, s->vals, s->rows, s->cfg.d};
    double dh;
    size_t att;
    mat bp = boosted_sparse_shrink(&a, s->cfg.ell, &s->ver, &s->cfg.power, &s->rng, &dh, &att);
    mat bm = {s->cfg.ell, s->cfg.d, s->b};
    mat st = vstack(&bm, &bp);
    mat nb = dense_shrink(&st, s->cfg.ell);
    memcpy(s->b, nb.data, s->cfg.ell * s->cfg.d * sizeof(double));
    s->rows = 0;
    s->nnz = 0;
    s->frob = 0.0;
    s->flushes += 1;
    s->attempts += att;
}

int or_sketcher_append_csr(or_sketcher* s, const int64_t* row_ptr, const uint32_t* cols,
                           const double* vals, size_t nrows, size_t* rows_done) {
    ENTER();
    if (rows_done) *rows_done = 0;
    for (size_t r = 0; r < nrows; ++r) {
        const int64_t b0 = row_ptr[r], b1 = row_ptr[r + 1];
        if (b1 < b0) THROW_INVALID("append_row: index/value length mismatch");
        const size_t len = (size_t)(b1 - b0);
        /* sparse.cpp:8-20: validate before committing */
        for (size_t k = 0; k < len; ++k) {
            if (cols[b0 + k] >= s->cfg.d) THROW_INVALID("append_row: column index out of range");
            if (k > 0 && cols[b0 + k] <= cols[b0 + k - 1])
                THROW_INVALID("append_row: indices must be strictly increasing");
            if (!isfinite(vals[b0 + k])) THROW_INVALID("append_row: non-finite value");
        }
        if (s->rows + 1 > s->cap_rows) {
            s->cap_rows *= 2;
            s->row_ptr = (int64_t*)realloc(s->row_ptr, (s->cap_rows + 1) * sizeof(int64_t));
        }
        if (s->nnz + len > s->cap_nnz) {
            while (s->nnz + len > s->cap_nnz) s->cap_nnz *= 2;
            s->cols = (uint32_t*)realloc(s->cols, s->cap_nnz * sizeof(uint32_t));
            s->vals = (double*)realloc(s->vals, s->cap_nnz * sizeof(double));
        }
        memcpy(s->cols + s->nnz, cols + b0, len * sizeof(uint32_t));
        memcpy(s->vals + s->nnz, vals + b0, len * sizeof(double));
        s->nnz += len;
        s->rows += 1;
        s->row_ptr[s->rows] = (int64_t)s->nnz;
        for (size_t k = 0; k < len; ++k) s->frob += vals[b0 + k] * vals[b0 + k];
        /* sketch.cpp:20-23 trigger */
        if (s->nnz >= s->cfg.ell * s->cfg.d || s->rows == s->cfg.d) sk_flush(s);
        if (rows_done) *rows_done = r + 1;
    }
    LEAVE();
}

/* sketch.cpp:34-45 */
int or_sketcher_finalize(or_sketcher* s, double* out) {
    ENTER();
    if (s->rows > 0) {
        if (s->rows >= s->cfg.ell) {
            sk_flush(s);
        } else {
            if (s->nnz > s->cfg.ell * s->cfg.d) THROW_INVALID("densify: nnz cap exceeded");
            mat tail = mat_new(s->rows, s->cfg.d);
            for (size_t i = 0; i < s->rows; ++i)
                for (int64_t k = s->row_ptr[i]; k < s->row_ptr[i + 1]; ++k) AT(tail, i, s->cols[k]) = s->vals[k];
            mat bm = {s->cfg.ell, s->cfg.d, s->b};
            mat st = vstack(&bm, &tail);
            mat nb = dense_shrink(&st, s->cfg.ell);
            memcpy(s->b, nb.data, s->cfg.ell * s->cfg.d * sizeof(double));
            s->rows = 0;
            s->nnz = 0;
            s->frob = 0.0;
        }
    }
    if (out) memcpy(out, s->b, s->cfg.ell * s->cfg.d * sizeof(double));
    LEAVE();
}

void or_sketcher_get_sketch(const or_sketcher* s, double* out) {
    memcpy(out, s->b, s->cfg.ell * s->cfg.d * sizeof(double));
}

void or_sketcher_stats(const or_sketcher* s, size_t* flushes, size_t* attempts, size_t* verifier_i,
                       double* delta_spent, size_t* buf_rows, size_t* buf_nnz, double* buf_frob_sq,
                       uint64_t* normals_drawn) {
    if (flushes) *flushes = s->flushes;
    if (attempts) *attempts = s->attempts;
    if (verifier_i) *verifier_i = s->ver.i;
    if (delta_spent) *delta_spent = s->ver.delta_spent;
    if (buf_rows) *buf_rows = s->rows;
    if (buf_nnz) *buf_nnz = s->nnz;
    if (buf_frob_sq) *buf_frob_sq = s->frob;
    if (normals_drawn) *normals_drawn = s->rng.normals;
}

void or_sketcher_buffer_dense(const or_sketcher* s, double* out) {
    memset(out, 0, s->rows * s->cfg.d * sizeof(double));
    for (size_t i = 0; i < s->rows; ++i)
        for (int64_t k = s->row_ptr[i]; k < s->row_ptr[i + 1]; ++k) out[i * s->cfg.d + s->cols[k]] = s->vals[k];
}
