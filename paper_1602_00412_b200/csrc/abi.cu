// abi.cu -- SfdSketcher on the device and the extern "C" boundary (include/sfdg.h).
//
// Sketcher mirrors sfd::SfdSketcher (core/include/sfd/sketch.hpp:22-49,
// core/src/sketch.cpp:9-45): rows are validated and committed one at a time with the
// exact trigger `nnz >= ell*d || rows == d` evaluated after each row; the running
// ||A'||_F^2 is accumulated on the host in row order (bit-identical to sparse.cpp:22);
// the flush runs the device engine (engine.cu). Batches are cut at the exact trigger rows
// and each segment is copied to the device buffer in one transfer.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/sfdg.h"
#include "engine.cuh"

namespace sfdg {

namespace {

thread_local std::string g_last_error;

struct SketchCfg {
    size_t ell = 0, d = 0;
    double delta = 0.1;
    PowerCfg power;
    uint64_t seed = 0;
};

PowerCfg to_power(const sfdg_power_config* p) {
    PowerCfg c;
    if (p) {
        c.epsilon = p->epsilon;
        c.q_constant = p->q_constant;
        c.q_override = p->q_override;
    }
    return c;
}

void validate_cfg(const SketchCfg& c) {  // sketch.cpp:9-12
    if (c.ell < 1 || c.ell > c.d) throw invalid_argument("SketchConfig: requires 1 <= ell <= d");
    if (c.delta <= 0.0 || c.delta >= 1.0) throw invalid_argument("SketchConfig: delta must be in (0,1)");
    if (c.d >= (size_t)INT32_MAX) throw invalid_argument("SketchConfig: d must be < 2^31");
}

// sparse.cpp:8-20: first failing check in element order decides the message.
void validate_row(const uint32_t* cols, const double* vals, int64_t len, size_t d) {
    for (int64_t k = 0; k < len; ++k) {
        if (cols[k] >= d) throw invalid_argument("append_row: column index out of range");
        if (k > 0 && cols[k] <= cols[k - 1]) throw invalid_argument("append_row: indices must be strictly increasing");
        if (!std::isfinite(vals[k])) throw invalid_argument("append_row: non-finite value");
    }
}

void validate_csr(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d) {
    for (size_t i = 0; i < m; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) throw invalid_argument("append_row: index/value length mismatch");
        validate_row(cols + row_ptr[i], vals + row_ptr[i], row_ptr[i + 1] - row_ptr[i], d);
    }
}

double csr_frob(const int64_t* row_ptr, const double* vals, size_t m) {
    double f = 0.0;
    for (int64_t k = row_ptr[0]; k < row_ptr[m]; ++k) f += vals[k] * vals[k];
    return f;
}

}  // namespace

class Sketcher {
  public:
    Sketcher(const SketchCfg& c, int device) : cfg(c) {
        validate_cfg(cfg);
        nnz_trigger = (int64_t)(cfg.ell * cfg.d);
        eng = std::make_unique<Engine>(device, (int)cfg.d, (int)cfg.ell, cfg.seed, (uint64_t)nnz_trigger + cfg.d,
                                       (int)cfg.d);
        ver.delta = cfg.delta;
        buf_rp.assign(1, 0);
    }

    void append_host(const int64_t* rp, const uint32_t* cols, const double* vals, size_t nrows, size_t* done) {
        eng->set_device();
        if (done) *done = 0;
        size_t r = 0;
        while (r < nrows) {
            const size_t take = segment(rp, r, nrows);
            // validate before committing (sparse.cpp:8-20); rows before a bad row stay in
            size_t good = 0;
            std::string err;
            for (; good < take; ++good) {
                const size_t i = r + good;
                try {
                    if (rp[i + 1] < rp[i]) throw invalid_argument("append_row: index/value length mismatch");
                    validate_row(cols + rp[i], vals + rp[i], rp[i + 1] - rp[i], cfg.d);
                } catch (const invalid_argument& e) {
                    err = e.what();
                    break;
                }
            }
            if (good > 0) commit_host(rp, cols, vals, r, good);
            if (good < take) {
                if (done) *done = r + good;
                throw invalid_argument(err);
            }
            r += take;
            if (done) *done = r;
            maybe_flush();
        }
    }

    void append_device(const int64_t* h_rp, const uint32_t* d_cols, const double* d_vals, size_t nrows, size_t* done) {
        eng->set_device();
        if (done) *done = 0;
        if (nrows == 0) return;
        for (size_t i = 0; i < nrows; ++i)
            if (h_rp[i + 1] < h_rp[i]) throw invalid_argument("append_row: index/value length mismatch");
        int64_t* d_rp = eng->scr.take<int64_t>((int64_t)nrows + 1);
        CK(cudaMemcpyAsync(d_rp, h_rp, (nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, eng->st));
        int kind = 0;
        const int64_t bad = validate_rows_device(d_rp, (int64_t)nrows, d_cols, d_vals, (uint32_t)cfg.d, &kind,
                                                 eng->scr, eng->st);
        eng->scr.reset();
        const size_t limit = bad < 0 ? nrows : (size_t)bad;
        size_t r = 0;
        while (r < limit) {
            const size_t take = segment(h_rp, r, limit);
            commit_device(h_rp, d_cols, d_vals, r, take);
            r += take;
            if (done) *done = r;
            maybe_flush();
        }
        if (bad >= 0)
            throw invalid_argument((kind & ERR_BAD_INDEX) ? "append_row: column index out of range or not increasing"
                                                          : "append_row: non-finite value");
    }

    void finalize(double* out) {  // sketch.cpp:34-45
        eng->set_device();
        eng->sync();
        eng->check_errors();
        if (buf_rows() > 0) {
            if (buf_rows() >= cfg.ell) {
                flush();
            } else {
                upload_row_ptr();
                const int m = (int)buf_rows();
                eng->densify_into_stack(eng->lp);
                eng->scr.reset();
                eng->dense_shrink_stack(eng->Mt[eng->cur], 2 * eng->lp, (int)cfg.ell, eng->lp, m,
                                        eng->Mt[eng->cur ^ 1], 2 * eng->lp);
                eng->check_errors();
                eng->cur ^= 1;
                clear_buffer();
            }
        }
        if (out) get_sketch(out);
    }

    void get_sketch(double* out) {
        eng->set_device();
        eng->sync();
        eng->check_errors();
        eng->scr.reset();
        eng->sketch_to_host(out);
    }

    void get_sketch_device(double* d_out, size_t ld) {
        eng->set_device();
        eng->sync();
        eng->check_errors();
        copy2d(eng->Mt[eng->cur], (int)cfg.d, (int)cfg.ell, 2 * eng->lp, d_out, (int)ld, eng->st);
        eng->sync();
    }

    void stats(sfdg_stats* s) {
        eng->set_device();
        eng->sync();
        s->flush_count = flushes;
        s->attempt_total = attempts;
        s->verifier = {ver.i, ver.delta, ver.c_verify, ver.delta_spent};
        s->buffer_rows = buf_rows();
        s->buffer_nnz = (size_t)buf_nnz;
        s->buffer_frob_sq = buf_frob;
        s->rng.seed = cfg.seed;
        s->rng.words = eng->pos.words;
        s->rng.has_spare = eng->pos.has_spare ? 1 : 0;
        s->rng.spare = eng->pos.has_spare ? eng->rng.spare_value(eng->st) : 0.0;
    }

    void get_buffer(int64_t* rp, uint32_t* cols, double* vals) {
        eng->set_device();
        if (rp) std::memcpy(rp, buf_rp.data(), buf_rp.size() * sizeof(int64_t));
        if (buf_nnz > 0) {
            if (cols) CK(cudaMemcpyAsync(cols, eng->a.col, buf_nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost, eng->st));
            if (vals) CK(cudaMemcpyAsync(vals, eng->a.val, buf_nnz * sizeof(double), cudaMemcpyDeviceToHost, eng->st));
        }
        eng->sync();
    }

    void synchronize() {
        eng->set_device();
        eng->sync();
    }

    // Back to a freshly constructed sketcher with `seed`, reusing every allocation.
    void reset(uint64_t seed) {
        eng->set_device();
        eng->sync();
        cfg.seed = seed;
        eng->rng.restart(seed);
        eng->pos = RngPos{};
        for (int i = 0; i < 2; ++i)
            CK(cudaMemsetAsync(eng->Mt[i], 0, (size_t)cfg.d * 2 * eng->lp * sizeof(double), eng->st));
        eng->cur = 0;
        CK(cudaMemsetAsync(eng->d_err, 0, sizeof(int), eng->st));
        eng->sync();
        ver = Verifier{};
        ver.delta = cfg.delta;
        clear_buffer();
        flushes = attempts = 0;
    }

  private:
    size_t buf_rows() const { return buf_rp.size() - 1; }

    // rows [r, r+take) such that the trigger can fire only after the last one
    size_t segment(const int64_t* rp, size_t r, size_t nrows) const {
        size_t take = std::min(nrows - r, cfg.d - buf_rows());
        const int64_t need = nnz_trigger - buf_nnz;  // > 0 while the buffer is below the trigger
        // first j in [r, r+take) with rp[j+1] - rp[r] >= need
        size_t lo = r, hi = r + take;
        while (lo < hi) {
            const size_t mid = (lo + hi) / 2;
            if (rp[mid + 1] - rp[r] >= need) hi = mid;
            else lo = mid + 1;
        }
        if (lo < r + take) take = lo - r + 1;
        return take;
    }

    void commit_host(const int64_t* rp, const uint32_t* cols, const double* vals, size_t r, size_t n) {
        const int64_t b = rp[r], e = rp[r + n];
        if (e > b) {
            CK(cudaMemcpyAsync(eng->a.col + buf_nnz, cols + b, (e - b) * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               eng->st));
            CK(cudaMemcpyAsync(eng->a.val + buf_nnz, vals + b, (e - b) * sizeof(double), cudaMemcpyHostToDevice,
                               eng->st));
        }
        for (int64_t k = b; k < e; ++k) buf_frob += vals[k] * vals[k];  // sparse.cpp:22, row order
        for (size_t i = 1; i <= n; ++i) buf_rp.push_back(buf_nnz + (rp[r + i] - b));
        buf_nnz += e - b;
    }

    void commit_device(const int64_t* rp, const uint32_t* d_cols, const double* d_vals, size_t r, size_t n) {
        const int64_t b = rp[r], e = rp[r + n];
        if (e > b) {
            CK(cudaMemcpyAsync(eng->a.col + buf_nnz, d_cols + b, (e - b) * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                               eng->st));
            CK(cudaMemcpyAsync(eng->a.val + buf_nnz, d_vals + b, (e - b) * sizeof(double), cudaMemcpyDeviceToDevice,
                               eng->st));
            eng->scr.reset();
            sumsq(eng->a.val + buf_nnz, e - b, 1, 1, eng->d_scal + 3, nullptr, 0, eng->scr, eng->st);
            buf_frob += eng->read_scalar(eng->d_scal + 3);
        }
        for (size_t i = 1; i <= n; ++i) buf_rp.push_back(buf_nnz + (rp[r + i] - b));
        buf_nnz += e - b;
    }

    void maybe_flush() {  // sketch.cpp:22
        if (buf_nnz >= nnz_trigger || buf_rows() == cfg.d) flush();
    }

    void upload_row_ptr() {
        const int m = (int)buf_rows();
        eng->a.set_shape(m, (int)cfg.d, buf_nnz);
        h_rp32.resize(m + 1);
        for (int i = 0; i <= m; ++i) h_rp32[i] = (int)buf_rp[i];
        CK(cudaMemcpyAsync(eng->a.row_ptr, h_rp32.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice, eng->st));
    }

    void flush() {  // sketch.cpp:25-32
        eng->scr.reset();
        upload_row_ptr();
        eng->prepare();
        // B'_f goes into the right half of Mt[cur]: first wait for the shrink that last read it
        CK(cudaStreamWaitEvent(eng->st, eng->ev_read_done[eng->cur], 0));
        double delta_hat = 0.0;
        const size_t att = eng->boosted(ver, cfg.power, buf_frob, &delta_hat);
        // B = dense_shrink([B; B']) on the shrink stream: it overlaps the next flush's power
        // iteration. Errors it raises (Jacobi non-convergence) surface at the next sync point.
        CK(cudaEventRecord(eng->ev_bprime, eng->st));
        CK(cudaStreamWaitEvent(eng->st2, eng->ev_bprime, 0));
        eng->scr2.reset();
        eng->dense_shrink_stack(eng->Mt[eng->cur], 2 * eng->lp, (int)cfg.ell, eng->lp, (int)cfg.ell,
                                eng->Mt[eng->cur ^ 1], 2 * eng->lp, /*side=*/true);
        CK(cudaEventRecord(eng->ev_read_done[eng->cur], eng->st2));
        eng->cur ^= 1;
        clear_buffer();
        flushes += 1;
        attempts += att;
    }

    void clear_buffer() {
        buf_rp.assign(1, 0);
        buf_nnz = 0;
        buf_frob = 0.0;
    }

    SketchCfg cfg;
    std::unique_ptr<Engine> eng;
    Verifier ver;
    std::vector<int64_t> buf_rp;
    std::vector<int> h_rp32;
    int64_t buf_nnz = 0;
    int64_t nnz_trigger = 0;
    double buf_frob = 0.0;
    size_t flushes = 0, attempts = 0;
};

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return SFDG_OK;
    } catch (const invalid_argument& e) {
        g_last_error = e.what();
        return SFDG_INVALID_ARGUMENT;
    } catch (const numerical_error& e) {
        g_last_error = e.what();
        return SFDG_NUMERICAL_ERROR;
    } catch (const cuda_error& e) {
        g_last_error = e.what();
        return SFDG_CUDA_ERROR;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return SFDG_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SFDG_CUDA_ERROR;
    }
}

void require_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw cuda_error("sfdg: no CUDA device available (this library has no CPU path)");
    }
    if (device < 0 || device >= n) throw invalid_argument("sfdg: device index out of range");
}

void rng_in(Engine& e, const sfdg_rng_state* r) {
    e.pos.words = r->words;
    e.pos.has_spare = r->has_spare != 0;
    if (e.pos.has_spare) e.rng.set_spare(r->spare, e.st);
}

void rng_out(Engine& e, sfdg_rng_state* r) {
    r->words = e.pos.words;
    r->has_spare = e.pos.has_spare ? 1 : 0;
    r->spare = e.pos.has_spare ? e.rng.spare_value(e.st) : 0.0;
}

// B'^T (d x lp, ldb) on device -> B' (ell x d) on host
void bt_to_host(Engine& e, const double* bt, int ldb, double* out) {
    double* tmp = e.scr.take<double>((int64_t)e.ell * e.d);
    transpose(bt, e.d, e.ell, ldb, tmp, e.d, e.st);
    CK(cudaMemcpyAsync(out, tmp, (size_t)e.ell * e.d * sizeof(double), cudaMemcpyDeviceToHost, e.st));
    e.sync();
}

// dense_shrink of a host matrix (rows x cols) on the device
void dense_shrink_host(const double* a, size_t rows, size_t cols, size_t ell, double* out, int device) {
    if (ell < 1 || ell > rows) throw invalid_argument("dense_shrink: ell out of range");
    for (size_t i = 0; i < rows * cols; ++i)
        if (!std::isfinite(a[i])) throw invalid_argument("dense_shrink: non-finite input");
    if (rows > cols && ell > cols) throw invalid_argument("dense_shrink: ell exceeds column count");
    if (ell > (size_t)kMaxEll) throw invalid_argument("sfdg: ell must be in [1, 256] for this build");
    Engine e(device, (int)cols, (int)ell, 0, 1, 1);
    double* A = e.scr.take<double>((int64_t)rows * cols);
    double* Xt = e.scr.take<double>((int64_t)cols * rows);
    double* bt = e.scr.take<double>((int64_t)cols * e.lp);
    CK(cudaMemcpyAsync(A, a, rows * cols * sizeof(double), cudaMemcpyHostToDevice, e.st));
    transpose(A, (int)rows, (int)cols, (int)cols, Xt, (int)rows, e.st);
    e.dense_shrink_stack(Xt, (int)rows, (int)rows, (int)rows, 0, bt, e.lp);
    e.check_errors();
    bt_to_host(e, bt, e.lp, out);
}

}  // namespace

}  // namespace sfdg

using namespace sfdg;

struct sfdg_sketcher {
    std::unique_ptr<Sketcher> impl;
};

static Sketcher* impl_of(sfdg_sketcher* h) {
    if (!h || !h->impl) throw invalid_argument("null sketcher handle");
    return h->impl.get();
}

extern "C" {

const char* sfdg_last_error(void) { return g_last_error.c_str(); }
const char* sfdg_version(void) { return "sfdg 0.1.0 (sm_100a, FP64)"; }
uint64_t sfdg_launch_count(void) { return g_launches.load(); }

int sfdg_device_count(int* count) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (count) *count = n;
    return SFDG_OK;
}

int sfdg_sketcher_create(const sfdg_sketch_config* cfg, int device, sfdg_sketcher** out) {
    return guard([&] {
        if (!cfg || !out) throw invalid_argument("sfdg_sketcher_create: null argument");
        SketchCfg c;
        c.ell = cfg->ell;
        c.d = cfg->d;
        c.delta = cfg->delta;
        c.power = to_power(&cfg->power);
        c.seed = cfg->seed;
        validate_cfg(c);
        require_device(device);
        auto h = std::make_unique<sfdg_sketcher>();
        h->impl = std::make_unique<Sketcher>(c, device);
        *out = h.release();
    });
}

int sfdg_sketcher_destroy(sfdg_sketcher* h) {
    return guard([&] { delete h; });
}

int sfdg_sketcher_append_csr(sfdg_sketcher* h, const int64_t* row_ptr, const uint32_t* cols, const double* vals,
                             size_t nrows, size_t* rows_done) {
    return guard([&] {
        if (!h) throw invalid_argument("null sketcher");
        h->impl->append_host(row_ptr, cols, vals, nrows, rows_done);
    });
}

int sfdg_sketcher_append_csr_device(sfdg_sketcher* h, const int64_t* h_row_ptr, const uint32_t* d_cols,
                                    const double* d_vals, size_t nrows, size_t* rows_done) {
    return guard([&] {
        if (!h) throw invalid_argument("null sketcher");
        h->impl->append_device(h_row_ptr, d_cols, d_vals, nrows, rows_done);
    });
}

int sfdg_sketcher_finalize(sfdg_sketcher* h, double* out) {
    return guard([&] { impl_of(h)->finalize(out); });
}

int sfdg_sketcher_get_sketch(sfdg_sketcher* h, double* out) {
    return guard([&] { impl_of(h)->get_sketch(out); });
}

int sfdg_sketcher_get_sketch_device(sfdg_sketcher* h, double* d_out, size_t ld) {
    return guard([&] { impl_of(h)->get_sketch_device(d_out, ld); });
}

int sfdg_sketcher_stats(sfdg_sketcher* h, sfdg_stats* out) {
    return guard([&] { impl_of(h)->stats(out); });
}

int sfdg_sketcher_get_buffer(sfdg_sketcher* h, int64_t* row_ptr, uint32_t* cols, double* vals) {
    return guard([&] { impl_of(h)->get_buffer(row_ptr, cols, vals); });
}

int sfdg_sketcher_reset(sfdg_sketcher* h, uint64_t seed) {
    return guard([&] { impl_of(h)->reset(seed); });
}

int sfdg_sketcher_synchronize(sfdg_sketcher* h) {
    return guard([&] { impl_of(h)->synchronize(); });
}

int sfdg_merge(const double* b1, size_t rows1, const double* b2, size_t rows2, size_t d, size_t ell, double* out,
               int device) {
    return guard([&] {
        require_device(device);
        std::vector<double> st((rows1 + rows2) * d);  // vstack (dense_matrix.cpp:20-28)
        std::memcpy(st.data(), b1, rows1 * d * sizeof(double));
        std::memcpy(st.data() + rows1 * d, b2, rows2 * d * sizeof(double));
        dense_shrink_host(st.data(), rows1 + rows2, d, ell, out, device);
    });
}

int sfdg_merge_device(const double* d_b1t, const double* d_b2t, size_t ell, size_t d, size_t ld, double* d_outt,
                      int device, void* stream) {
    return guard([&] {
        require_device(device);
        CK(cudaSetDevice(device));
        if (stream) CK(cudaStreamSynchronize((cudaStream_t)stream));
        else CK(cudaDeviceSynchronize());
        Engine e(device, (int)d, (int)ell, 0, 1, 1);
        const int lp = e.lp;
        double* X = e.Mt[0];
        copy2d(d_b1t, (int)d, (int)ell, (int)ld, X, 2 * lp, e.st);
        copy2d(d_b2t, (int)d, (int)ell, (int)ld, X + lp, 2 * lp, e.st);
        e.dense_shrink_stack(X, 2 * lp, (int)ell, lp, (int)ell, e.Mt[1], 2 * lp);
        copy2d(e.Mt[1], (int)d, (int)ell, 2 * lp, d_outt, (int)ld, e.st);
        e.check_errors();
    });
}

int sfdg_dense_shrink(const double* a, size_t rows, size_t cols, size_t ell, double* out, int device) {
    return guard([&] {
        require_device(device);
        dense_shrink_host(a, rows, cols, ell, out, device);
    });
}

int sfdg_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d, size_t ell,
                       const sfdg_power_config* power, sfdg_rng_state* rng, double* out, int device) {
    return guard([&] {
        if (ell < 1 || ell > m) throw invalid_argument("sparse_shrink: ell out of range");
        if (ell > d) throw invalid_argument("sparse_shrink: ell exceeds column count");
        validate_csr(row_ptr, cols, vals, m, d);
        require_device(device);
        Engine e(device, (int)d, (int)ell, rng->seed, (uint64_t)(row_ptr[m] - row_ptr[0]), (int)m);
        rng_in(e, rng);
        e.load_csr(row_ptr, cols, vals, (int)m, row_ptr[m] - row_ptr[0]);
        e.prepare();
        double* bt = e.Mt[0] + e.lp;
        e.sparse_shrink(to_power(power), bt, 2 * e.lp);
        e.check_errors();
        bt_to_host(e, bt, 2 * e.lp, out);
        rng_out(e, rng);
    });
}

int sfdg_boosted_sparse_shrink(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                               size_t ell, sfdg_verifier_state* verifier, const sfdg_power_config* power,
                               sfdg_rng_state* rng, double* out, double* delta_hat, size_t* attempts, int device) {
    return guard([&] {
        if (ell < 1 || ell > m) throw invalid_argument("boosted_sparse_shrink: ell out of range");
        if (ell > d) throw invalid_argument("sparse_shrink: ell exceeds column count");
        validate_csr(row_ptr, cols, vals, m, d);
        require_device(device);
        Engine e(device, (int)d, (int)ell, rng->seed, (uint64_t)(row_ptr[m] - row_ptr[0]), (int)m);
        rng_in(e, rng);
        e.load_csr(row_ptr, cols, vals, (int)m, row_ptr[m] - row_ptr[0]);
        e.prepare();
        Verifier v;
        v.i = verifier->i;
        v.delta = verifier->delta;
        v.c_verify = verifier->c_verify;
        v.delta_spent = verifier->delta_spent;
        double dh = 0.0;
        const size_t att = e.boosted(v, to_power(power), csr_frob(row_ptr, vals, m), &dh);
        e.check_errors();
        bt_to_host(e, e.Mt[e.cur] + e.lp, 2 * e.lp, out);
        verifier->i = v.i;
        verifier->delta_spent = v.delta_spent;
        if (delta_hat) *delta_hat = dh;
        if (attempts) *attempts = att;
        rng_out(e, rng);
    });
}

int sfdg_simultaneous_iteration(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d,
                                size_t k, const sfdg_power_config* power, sfdg_rng_state* rng, double* z_out,
                                int device) {
    return guard([&] {
        if (k < 1 || k > std::min(m, d)) throw invalid_argument("simultaneous_iteration: k out of range");
        validate_csr(row_ptr, cols, vals, m, d);
        require_device(device);
        Engine e(device, (int)d, (int)k, rng->seed, (uint64_t)(row_ptr[m] - row_ptr[0]), (int)m);
        rng_in(e, rng);
        e.load_csr(row_ptr, cols, vals, (int)m, row_ptr[m] - row_ptr[0]);
        e.prepare();
        e.simultaneous_iteration((int)k, to_power(power));
        e.check_errors();
        double* tmp = e.scr.take<double>((int64_t)m * k);
        copy2d(e.Y, (int)m, (int)k, e.lp, tmp, (int)k, e.st);
        CK(cudaMemcpyAsync(z_out, tmp, m * k * sizeof(double), cudaMemcpyDeviceToHost, e.st));
        e.sync();
        rng_out(e, rng);
    });
}

int sfdg_power_iteration_count(size_t m, const sfdg_power_config* power, size_t* q) {
    return guard([&] { *q = power_iteration_count(m, to_power(power)); });
}

int sfdg_gaussian_matrix(sfdg_rng_state* rng, size_t rows, size_t cols, double* out, int device) {
    return guard([&] {
        if (rows < 1 || cols < 1) throw invalid_argument("gaussian_matrix: empty shape");
        require_device(device);
        CK(cudaSetDevice(device));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        RngStream rs;
        rs.init(rng->seed, 2 * rows * cols + 64, device);
        RngPos pos{rng->words, rng->has_spare != 0};
        if (pos.has_spare) rs.set_spare(rng->spare, st);
        double* dout = nullptr;
        int* derr = nullptr;
        CK(cudaMalloc(&dout, rows * cols * sizeof(double)));
        CK(cudaMalloc(&derr, sizeof(int)));
        CK(cudaMemsetAsync(derr, 0, sizeof(int), st));
        rs.normals(pos, rows * cols, cols, cols, dout, derr, st);
        int herr = 0;
        CK(cudaMemcpyAsync(out, dout, rows * cols * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        rng->words = pos.words;
        rng->has_spare = pos.has_spare ? 1 : 0;
        rng->spare = pos.has_spare ? rs.spare_value(st) : 0.0;
        cudaFree(dout);
        cudaFree(derr);
        cudaStreamDestroy(st);
        if (herr) throw numerical_error("rng: Box-Muller u1 == 0 redraw (probability 2^-53) is not reproduced on device");
    });
}

int sfdg_eigh(const double* sym, size_t n, double off_tol, double* values, double* vectors, int device) {
    return guard([&] {
        if (n < 1 || n > 1024) throw invalid_argument("eigh: n must be in [1, 1024]");
        require_device(device);
        Engine e(device, 8, 1, 0, 1, 1);
        double* K = e.scr.take<double>((int64_t)n * n);
        double* ev = e.scr.take<double>(n);
        double* V = e.scr.take<double>((int64_t)n * n);
        CK(cudaMemcpyAsync(K, sym, n * n * sizeof(double), cudaMemcpyHostToDevice, e.st));
        eigh(K, (int)n, (int)n, off_tol, nullptr, ev, V, (int)n, e.d_err, e.scr, e.st);
        CK(cudaMemcpyAsync(values, ev, n * sizeof(double), cudaMemcpyDeviceToHost, e.st));
        CK(cudaMemcpyAsync(vectors, V, n * n * sizeof(double), cudaMemcpyDeviceToHost, e.st));
        e.check_errors();
    });
}

int sfdg_orthonormalize(const double* in, size_t n, size_t k, double* out, int device) {
    return guard([&] {
        if (n < k) throw invalid_argument("orthonormalize: needs n >= k");
        if (k < 1 || k > (size_t)kMaxEll) throw invalid_argument("orthonormalize: k must be in [1, 256]");
        require_device(device);
        Engine e(device, 8, (int)k, 0, 1, (int)n);
        CK(cudaMemsetAsync(e.Y, 0, n * e.lp * sizeof(double), e.st));
        double* tmp = e.scr.take<double>((int64_t)n * k);
        CK(cudaMemcpyAsync(tmp, in, n * k * sizeof(double), cudaMemcpyHostToDevice, e.st));
        copy2d(tmp, (int)n, (int)k, (int)k, e.Y, e.lp, e.st);
        e.orthonormalize(e.Y, (int)n, ERR_NONFINITE_ITER);
        copy2d(e.Y, (int)n, (int)k, e.lp, tmp, (int)k, e.st);
        CK(cudaMemcpyAsync(out, tmp, n * k * sizeof(double), cudaMemcpyDeviceToHost, e.st));
        e.check_errors();
    });
}

int sfdg_csr_products(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t m, size_t d, size_t k,
                      const double* x, double* y, const double* z, double* w, int device) {
    return guard([&] {
        validate_csr(row_ptr, cols, vals, m, d);
        require_device(device);
        const int kk = (int)round_up(std::max<size_t>(k, 1), 2);
        Engine e(device, (int)d, 1, 0, (uint64_t)(row_ptr[m] - row_ptr[0]), (int)m);
        e.load_csr(row_ptr, cols, vals, (int)m, row_ptr[m] - row_ptr[0]);
        e.prepare();
        double* xin = e.scr.take<double>((int64_t)std::max(m, d) * kk);
        double* yout = e.scr.take<double>((int64_t)std::max(m, d) * kk);
        double* tmp = e.scr.take<double>((int64_t)std::max(m, d) * k);
        if (x && y) {
            CK(cudaMemsetAsync(xin, 0, d * kk * sizeof(double), e.st));
            CK(cudaMemcpyAsync(tmp, x, d * k * sizeof(double), cudaMemcpyHostToDevice, e.st));
            copy2d(tmp, (int)d, (int)k, (int)k, xin, kk, e.st);
            spmm(e.a.row_ptr, (const int*)e.a.col, e.a.val, (int)m, e.plan_r, e.a.nnz, xin, kk, kk, yout, kk, e.scr,
                 e.st);
            copy2d(yout, (int)m, (int)k, kk, tmp, (int)k, e.st);
            CK(cudaMemcpyAsync(y, tmp, m * k * sizeof(double), cudaMemcpyDeviceToHost, e.st));
            e.sync();
        }
        if (z && w) {
            CK(cudaMemsetAsync(xin, 0, m * kk * sizeof(double), e.st));
            CK(cudaMemcpyAsync(tmp, z, m * k * sizeof(double), cudaMemcpyHostToDevice, e.st));
            copy2d(tmp, (int)m, (int)k, (int)k, xin, kk, e.st);
            spmm(e.a.col_ptr, e.a.row_idx, e.a.cval, (int)d, e.plan_c, e.a.nnz, xin, kk, kk, yout, kk, e.scr, e.st);
            copy2d(yout, (int)d, (int)k, kk, tmp, (int)k, e.st);
            CK(cudaMemcpyAsync(w, tmp, d * k * sizeof(double), cudaMemcpyDeviceToHost, e.st));
            e.sync();
        }
        e.check_errors();
    });
}

}  // extern "C"
