// ref_shim.cpp -- C-ABI over the UNMODIFIED reference library, for pinning the oracle.
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into oracle/_ref/libsfdref.so
// together with the reference's own core/src/*.cpp compiled where they lie under
// /root/reference/proj (nothing is copied into this repo). The entry points mirror
// oracle/sfd_oracle.h with a `ref_` prefix so tests can run both side by side.
// Exceptions map to the same status codes: 1 invalid_argument, 2 numerical_error.

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

#include "sfd/bench.hpp"
#include "sfd/common.hpp"
#include "sfd/la_core.hpp"
#include "sfd/randsvd.hpp"
#include "sfd/shrink.hpp"
#include "sfd/sketch.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sfd::numerical_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

sfd::SparseBuffer to_buffer(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m,
                            size_t d) {
    sfd::SparseBuffer buf(d);
    for (size_t i = 0; i < m; ++i) {
        sfd::SparseRow r;
        r.indices.assign(cols + row_ptr[i], cols + row_ptr[i + 1]);
        r.values.assign(vals + row_ptr[i], vals + row_ptr[i + 1]);
        buf.append_row(r);
    }
    return buf;
}

sfd::PowerConfig power(double eps, double qc, long long qo) {
    sfd::PowerConfig p;
    p.epsilon = eps;
    p.q_constant = qc;
    if (qo >= 0) p.q_override = static_cast<size_t>(qo);
    return p;
}

void put(const sfd::DenseMatrix& m, double* out) { std::memcpy(out, m.data.data(), m.data.size() * sizeof(double)); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_rng_new(uint64_t seed) { return new sfd::Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<sfd::Rng*>(r); }
uint64_t ref_rng_next_u64(void* r) { return static_cast<sfd::Rng*>(r)->next_u64(); }
double ref_rng_uniform(void* r) { return static_cast<sfd::Rng*>(r)->uniform(); }
double ref_rng_normal(void* r) { return static_cast<sfd::Rng*>(r)->normal(); }
uint64_t ref_rng_uniform_below(void* r, uint64_t n) { return static_cast<sfd::Rng*>(r)->uniform_below(n); }

int ref_dense_shrink(const double* a, size_t rows, size_t cols, size_t ell, double* out) {
    return guarded([&] {
        sfd::DenseMatrix m(rows, cols);
        std::memcpy(m.data.data(), a, rows * cols * sizeof(double));
        put(sfd::dense_shrink(m, ell), out);
    });
}

int ref_orthonormalize(const double* in, size_t n, size_t k, double* out) {
    return guarded([&] {
        sfd::DenseMatrix m(n, k);
        std::memcpy(m.data.data(), in, n * k * sizeof(double));
        put(sfd::orthonormalize(m), out);
    });
}

int ref_jacobi_eigh(const double* sym, size_t n, double off_tol, double* values, double* vectors) {
    return guarded([&] {
        sfd::DenseMatrix m(n, n);
        std::memcpy(m.data.data(), sym, n * n * sizeof(double));
        sfd::EighResult e = sfd::jacobi_eigh(m, off_tol);
        std::memcpy(values, e.values.data(), n * sizeof(double));
        put(e.vectors, vectors);
    });
}

int ref_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                      size_t ell, double eps, double qc, long long qo, void* rng, double* out) {
    return guarded([&] {
        sfd::SparseBuffer buf = to_buffer(row_ptr, cols, vals, m, d);
        put(sfd::sparse_shrink(buf, ell, power(eps, qc, qo), *static_cast<sfd::Rng*>(rng)), out);
    });
}

int ref_simultaneous_iteration(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m,
                               size_t d, size_t k, double eps, double qc, long long qo, void* rng,
                               double* out) {
    return guarded([&] {
        sfd::SparseBuffer buf = to_buffer(row_ptr, cols, vals, m, d);
        put(sfd::simultaneous_iteration(buf, k, power(eps, qc, qo), *static_cast<sfd::Rng*>(rng)), out);
    });
}

// state: [i, delta, c_verify, delta_spent] in/out
int ref_boosted_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m,
                              size_t d, size_t ell, double* state, double eps, double qc, long long qo,
                              void* rng, double* out, double* delta_hat, size_t* attempts) {
    return guarded([&] {
        sfd::SparseBuffer buf = to_buffer(row_ptr, cols, vals, m, d);
        sfd::VerifierState st;
        st.i = static_cast<size_t>(state[0]);
        st.delta = state[1];
        st.c_verify = state[2];
        st.delta_spent = state[3];
        sfd::ShrinkReport rep = sfd::boosted_sparse_shrink(buf, ell, st, power(eps, qc, qo), *static_cast<sfd::Rng*>(rng));
        state[0] = static_cast<double>(st.i);
        state[3] = st.delta_spent;
        put(rep.b, out);
        *delta_hat = rep.delta_hat;
        *attempts = rep.attempts;
    });
}

int ref_merge(const double* b1, size_t r1, const double* b2, size_t r2, size_t d, size_t ell, double* out) {
    return guarded([&] {
        sfd::DenseMatrix m1(r1, d), m2(r2, d);
        std::memcpy(m1.data.data(), b1, r1 * d * sizeof(double));
        std::memcpy(m2.data.data(), b2, r2 * d * sizeof(double));
        put(sfd::merge(m1, m2, ell), out);
    });
}

// cov_err (bench.cpp:171-183) of a sketch (ell x d) against CSR A, rng advanced in place.
int ref_cov_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                const double* sketch, size_t ell, void* rng, size_t iterations, double* out) {
    return guarded([&] {
        sfd::SparseBuffer a = to_buffer(row_ptr, cols, vals, m, d);
        sfd::DenseMatrix b(ell, d);
        std::memcpy(b.data.data(), sketch, ell * d * sizeof(double));
        *out = sfd::cov_err(a, b, *static_cast<sfd::Rng*>(rng), iterations);
    });
}

// exact_tail (bench.cpp:68-137): tail and the top-k singular values.
int ref_exact_tail(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d, size_t k,
                   void* rng, double* sigma_out, double* tail_out) {
    return guarded([&] {
        sfd::SparseBuffer a = to_buffer(row_ptr, cols, vals, m, d);
        sfd::TailResult r = sfd::exact_tail(a, k, *static_cast<sfd::Rng*>(rng));
        *tail_out = r.tail_sq;
        for (size_t i = 0; i < r.sigma.size(); ++i) sigma_out[i] = r.sigma[i];
    });
}

// proj_err (bench.cpp:139-169); *has_value = 0 for nullopt.
int ref_proj_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                 const double* sketch, size_t ell, size_t k, double tail_sq, double* out, int* has_value) {
    return guarded([&] {
        sfd::SparseBuffer a = to_buffer(row_ptr, cols, vals, m, d);
        sfd::DenseMatrix b(ell, d);
        std::memcpy(b.data.data(), sketch, ell * d * sizeof(double));
        sfd::TailResult t;
        t.tail_sq = tail_sq;
        auto r = sfd::proj_err(a, b, k, t);
        *has_value = r ? 1 : 0;
        *out = r ? *r : 0.0;
    });
}

// Whole-stream FdSketcher run (sketch.cpp:47-78) over n dense rows.
int ref_fd_sketch(const double* rows, size_t n, size_t d, size_t ell, double* out, size_t* shrink_count) {
    return guarded([&] {
        sfd::FdSketcher f(ell, d);
        std::vector<double> r(d);
        for (size_t i = 0; i < n; ++i) {
            std::memcpy(r.data(), rows + i * d, d * sizeof(double));
            f.append(r);
        }
        put(f.finalize(), out);
        *shrink_count = f.shrink_count();
    });
}

// Whole-stream SfdSketcher run: append every row, finalize. stats = [flushes, attempts, verifier_i,
// delta_spent].
int ref_sketch(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d,
               size_t ell, double delta, double eps, double qc, long long qo, uint64_t seed, double* out,
               double* stats) {
    return guarded([&] {
        sfd::SketchConfig cfg;
        cfg.ell = ell;
        cfg.d = d;
        cfg.delta = delta;
        cfg.power = power(eps, qc, qo);
        cfg.seed = seed;
        sfd::SfdSketcher s(cfg);
        sfd::SparseRow r;
        for (size_t i = 0; i < n; ++i) {
            r.indices.assign(cols + row_ptr[i], cols + row_ptr[i + 1]);
            r.values.assign(vals + row_ptr[i], vals + row_ptr[i + 1]);
            s.append(r);
        }
        put(s.finalize(), out);
        stats[0] = static_cast<double>(s.flush_count());
        stats[1] = static_cast<double>(s.attempt_total());
        stats[2] = static_cast<double>(s.verifier().i);
        stats[3] = s.verifier().delta_spent;
    });
}

// One power sweep of simultaneous_iteration (randsvd.cpp:39-48: for every column, rmatvec then
// matvec; the finiteness check; orthonormalize) over the reference's own SparseBuffer and
// orthonormalize, from a given Y (m x k). *seconds = wall time of the sweep alone. Used by
// bench.py's reference arm, which extrapolates a flush as (q + 1) sweeps.
int ref_power_sweep(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d, size_t k,
                    const double* y_in, double* y_out, double* seconds) {
    return guarded([&] {
        sfd::SparseBuffer a = to_buffer(row_ptr, cols, vals, m, d);
        sfd::DenseMatrix y(m, k);
        std::memcpy(y.data.data(), y_in, m * k * sizeof(double));
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<double> ycol(m);
        sfd::DenseMatrix next(m, k);
        for (size_t j = 0; j < k; ++j) {
            for (size_t i = 0; i < m; ++i) ycol[i] = y(i, j);
            std::vector<double> w = a.rmatvec(ycol);
            std::vector<double> yc = a.matvec(w);
            for (size_t i = 0; i < m; ++i) next(i, j) = yc[i];
        }
        if (!sfd::all_finite(next)) throw sfd::numerical_error("simultaneous_iteration: non-finite intermediate");
        y = sfd::orthonormalize(next);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        put(y, y_out);
    });
}

// A live SfdSketcher (sketch.hpp:22-49) driven row by row, so tests can read the reference's
// state after an append that throws (sketch.cpp:20-32: the exception leaves B, the counters
// and the buffer as they were at the failing flush).
void* ref_sketcher_new(size_t ell, size_t d, double delta, uint64_t seed) {
    sfd::SketchConfig cfg;
    cfg.ell = ell;
    cfg.d = d;
    cfg.delta = delta;
    cfg.seed = seed;
    try {
        return new sfd::SfdSketcher(cfg);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_sketcher_free(void* h) { delete static_cast<sfd::SfdSketcher*>(h); }
int ref_sketcher_append(void* h, const uint32_t* cols, const double* vals, size_t len) {
    return guarded([&] {
        sfd::SparseRow r;
        r.indices.assign(cols, cols + len);
        r.values.assign(vals, vals + len);
        static_cast<sfd::SfdSketcher*>(h)->append(r);
    });
}
void ref_sketcher_sketch(void* h, double* out) { put(static_cast<sfd::SfdSketcher*>(h)->sketch(), out); }
// [flushes, attempts, verifier_i, delta_spent, buffer_rows, buffer_nnz, buffer_frob_sq]
void ref_sketcher_stats(void* h, double* st) {
    auto* s = static_cast<sfd::SfdSketcher*>(h);
    st[0] = static_cast<double>(s->flush_count());
    st[1] = static_cast<double>(s->attempt_total());
    st[2] = static_cast<double>(s->verifier().i);
    st[3] = s->verifier().delta_spent;
    st[4] = static_cast<double>(s->buffer().rows());
    st[5] = static_cast<double>(s->buffer().nnz());
    st[6] = s->buffer().frob_sq();
}

}  // extern "C"
