// sfd_compat.cpp -- the reference's sketch / shrink / randsvd / bench entry points implemented
// over the sfdg C ABI, so the reference's own unit tests (tests/test_sketch.cpp,
// test_shrink.cpp, test_randsvd.cpp, test_bench.cpp) run against the device build unchanged.
// Test infrastructure: built by oracle/Makefile (target refsuite) into oracle/_ref/refsuite,
// together with the reference's dense_matrix / sparse / la_core sources, which supply the
// value types and the tests' own oracles. Every computation the tests check runs in
// libsfdg.so on the GPU.
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../tools/synthetic_rows.hpp"
#include "sfd/bench.hpp"
#include "sfd/common.hpp"
#include "sfd/rng.hpp"
#include "sfd/sketch.hpp"
#include "sfdg.h"

namespace sfd {

namespace {

void check(int rc) {
    if (rc == SFDG_OK) return;
    const std::string msg = sfdg_last_error();
    if (rc == SFDG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == SFDG_NUMERICAL_ERROR) throw numerical_error(msg);
    throw std::runtime_error(msg);
}

sfdg_power_config power_c(const PowerConfig& p) {
    return {p.epsilon, p.q_constant, p.q_override ? static_cast<int64_t>(*p.q_override) : int64_t(-1)};
}

// SparseBuffer (size_t offsets) -> int64 CSR for the ABI; a 1-element dummy keeps pointers valid.
struct Csr {
    std::vector<int64_t> rp;
    const uint32_t* cols;
    const double* vals;
    size_t m, d;
    uint32_t no_col = 0;
    double no_val = 0.0;
    explicit Csr(const SparseBuffer& a) : m(a.rows()), d(a.cols()) {
        rp.assign(a.row_offsets().begin(), a.row_offsets().end());
        cols = a.nnz() ? a.col_indices().data() : &no_col;
        vals = a.nnz() ? a.values().data() : &no_val;
    }
};

const int kDevice = 0;

}  // namespace

// ---- Rng (rng.cpp:9-34) ------------------------------------------------------------
std::uint64_t Rng::uniform_below(std::uint64_t n) {
    if (n == 0) throw std::invalid_argument("uniform_below: n must be positive");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t v;
    do v = next_u64();
    while (v >= limit);
    return v % n;
}

double Rng::normal() {
    if (has_spare_) {
        has_spare_ = false;
        return spare_;
    }
    double u1;
    do u1 = uniform();
    while (u1 <= 0.0);
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(theta);
    has_spare_ = true;
    return r * std::cos(theta);
}

void Rng::set_device_state(const sfdg_rng_state& s) {
    if (s.seed != seed_ || s.words < words_) throw std::logic_error("Rng: device state from another stream");
    engine_.discard(s.words - words_);
    words_ = s.words;
    has_spare_ = s.has_spare != 0;
    spare_ = s.spare;
}

// ---- randsvd -------------------------------------------------------------------------
std::size_t power_iteration_count(std::size_t m, const PowerConfig& cfg) {
    const sfdg_power_config p = power_c(cfg);
    size_t q = 0;
    check(sfdg_power_iteration_count(m, &p, &q));
    return q;
}

DenseMatrix simultaneous_iteration(const SparseBuffer& a, std::size_t k, const PowerConfig& cfg, Rng& rng) {
    const Csr c(a);
    const sfdg_power_config p = power_c(cfg);
    sfdg_rng_state st = rng.device_state();
    DenseMatrix z(c.m, k);
    check(sfdg_simultaneous_iteration(c.rp.data(), c.cols, c.vals, c.m, c.d, k, &p, &st, z.data.data(), kDevice));
    rng.set_device_state(st);
    return z;
}

// ---- shrink --------------------------------------------------------------------------
DenseMatrix dense_shrink(const DenseMatrix& a, std::size_t ell) {
    DenseMatrix out(ell, a.cols);
    check(sfdg_dense_shrink(a.data.data(), a.rows, a.cols, ell, out.data.data(), kDevice));
    return out;
}

DenseMatrix sparse_shrink(const SparseBuffer& a, std::size_t ell, const PowerConfig& cfg, Rng& rng) {
    const Csr c(a);
    const sfdg_power_config p = power_c(cfg);
    sfdg_rng_state st = rng.device_state();
    DenseMatrix out(ell, c.d);
    check(sfdg_sparse_shrink(c.rp.data(), c.cols, c.vals, c.m, c.d, ell, &p, &st, out.data.data(), kDevice));
    rng.set_device_state(st);
    return out;
}

// The caller's std::function operator runs on the host through sfdg_verify_spectral's
// callback; the draw of x and the step bookkeeping are the library's.
bool verify_spectral(const SymOp& apply, std::size_t d, VerifierState& state, Rng& rng) {
    struct Ctx {
        const SymOp* op;
        std::vector<double> x;
    } ctx{&apply, std::vector<double>(d)};
    auto cb = [](const double* x, double* y, size_t n, void* user) -> int {
        Ctx* c = static_cast<Ctx*>(user);
        c->x.assign(x, x + n);
        const std::vector<double> out = (*c->op)(c->x);
        if (out.size() != n) return 1;
        std::copy(out.begin(), out.end(), y);
        return 0;
    };
    sfdg_verifier_state vs{state.i, state.delta, state.c_verify, state.delta_spent};
    sfdg_rng_state st = rng.device_state();
    int accepted = 0;
    check(sfdg_verify_spectral(cb, &ctx, 0, d, &vs, &st, &accepted, kDevice));
    rng.set_device_state(st);
    state.i = vs.i;
    state.delta_spent = vs.delta_spent;
    return accepted != 0;
}

ShrinkReport boosted_sparse_shrink(const SparseBuffer& a, std::size_t ell, VerifierState& state,
                                   const PowerConfig& cfg, Rng& rng) {
    const Csr c(a);
    const sfdg_power_config p = power_c(cfg);
    sfdg_rng_state st = rng.device_state();
    sfdg_verifier_state v{state.i, state.delta, state.c_verify, state.delta_spent};
    ShrinkReport rep;
    rep.b = DenseMatrix(ell, c.d);
    check(sfdg_boosted_sparse_shrink(c.rp.data(), c.cols, c.vals, c.m, c.d, ell, &v, &p, &st, rep.b.data.data(),
                                     &rep.delta_hat, &rep.attempts, kDevice));
    rng.set_device_state(st);
    state.i = v.i;
    state.delta = v.delta;
    state.c_verify = v.c_verify;
    state.delta_spent = v.delta_spent;
    return rep;
}

// ---- sketch --------------------------------------------------------------------------
void SketchConfig::validate() const {
    // the library validates at construction (sketch.cpp:9-12): build and drop a handle
    sfdg_sketch_config c{ell, d, delta, power_c(power), seed};
    sfdg_sketcher* h = nullptr;
    check(sfdg_sketcher_create(&c, kDevice, &h));
    sfdg_sketcher_destroy(h);
}

SfdSketcher::SfdSketcher(const SketchConfig& cfg) : cfg_(cfg), view_b_(cfg.ell, cfg.d), view_buf_(cfg.d) {
    sfdg_sketch_config c{cfg.ell, cfg.d, cfg.delta, power_c(cfg.power), cfg.seed};
    check(sfdg_sketcher_create(&c, kDevice, &h_));
}

SfdSketcher::~SfdSketcher() {
    if (h_) sfdg_sketcher_destroy(h_);
}

void SfdSketcher::append(const SparseRow& row) {
    if (row.indices.size() != row.values.size()) throw std::invalid_argument("append_row: index/value length mismatch");
    static const uint32_t kNoCol = 0;
    static const double kNoVal = 0.0;
    const int64_t rp[2] = {0, static_cast<int64_t>(row.indices.size())};
    check(sfdg_sketcher_append_csr(h_, rp, row.indices.empty() ? &kNoCol : row.indices.data(),
                                   row.values.empty() ? &kNoVal : row.values.data(), 1, nullptr));
}

DenseMatrix SfdSketcher::finalize() {
    DenseMatrix b(cfg_.ell, cfg_.d);
    check(sfdg_sketcher_finalize(h_, b.data.data()));
    return b;
}

const DenseMatrix& SfdSketcher::sketch() const {
    view_b_ = DenseMatrix(cfg_.ell, cfg_.d);
    check(sfdg_sketcher_get_sketch(h_, view_b_.data.data()));
    return view_b_;
}

const SparseBuffer& SfdSketcher::buffer() const {
    sfdg_stats s{};
    check(sfdg_sketcher_stats(h_, &s));
    std::vector<int64_t> rp(s.buffer_rows + 1);
    std::vector<uint32_t> cols(s.buffer_nnz ? s.buffer_nnz : 1);
    std::vector<double> vals(s.buffer_nnz ? s.buffer_nnz : 1);
    check(sfdg_sketcher_get_buffer(h_, rp.data(), cols.data(), vals.data()));
    view_buf_ = SparseBuffer(cfg_.d);
    for (size_t i = 0; i < s.buffer_rows; ++i) {
        SparseRow r;
        r.indices.assign(cols.begin() + rp[i], cols.begin() + rp[i + 1]);
        r.values.assign(vals.begin() + rp[i], vals.begin() + rp[i + 1]);
        view_buf_.append_row(r);
    }
    return view_buf_;
}

const VerifierState& SfdSketcher::verifier() const {
    sfdg_stats s{};
    check(sfdg_sketcher_stats(h_, &s));
    view_ver_ = {s.verifier.i, s.verifier.delta, s.verifier.c_verify, s.verifier.delta_spent};
    return view_ver_;
}

std::size_t SfdSketcher::flush_count() const {
    sfdg_stats s{};
    check(sfdg_sketcher_stats(h_, &s));
    return s.flush_count;
}

std::size_t SfdSketcher::attempt_total() const {
    sfdg_stats s{};
    check(sfdg_sketcher_stats(h_, &s));
    return s.attempt_total;
}

FdSketcher::FdSketcher(std::size_t ell, std::size_t d) : ell_(ell), d_(d) {
    check(sfdg_fd_create(ell, d, kDevice, &h_));
}

FdSketcher::~FdSketcher() {
    if (h_) sfdg_fd_destroy(h_);
}

void FdSketcher::append(const std::vector<double>& row) {
    if (row.size() != d_) throw std::invalid_argument("FdSketcher::append: row width mismatch");
    check(sfdg_fd_append(h_, row.data(), 1));
}

DenseMatrix FdSketcher::finalize() {
    DenseMatrix b(ell_, d_);
    check(sfdg_fd_finalize(h_, b.data.data()));
    return b;
}

std::size_t FdSketcher::shrink_count() const {
    size_t c = 0;
    check(sfdg_fd_shrink_count(h_, &c));
    return c;
}

DenseMatrix merge(const DenseMatrix& b1, const DenseMatrix& b2, std::size_t ell) {
    if (b1.cols != b2.cols) throw std::invalid_argument("vstack: column mismatch");
    DenseMatrix out(ell, b1.cols);
    check(sfdg_merge(b1.data.data(), b1.rows, b2.data.data(), b2.rows, b1.cols, ell, out.data.data(), kDevice));
    return out;
}

// ---- bench ---------------------------------------------------------------------------
std::size_t SyntheticSpec::head_cols() const {
    return std::min(static_cast<std::size_t>(std::ceil(1.5 * static_cast<double>(z))), d);
}

void SyntheticSpec::validate() const {
    sfdg_tools::SyntheticRows probe(0, d, z, p_head, seed);  // throws the reference's messages
}

SyntheticStream::SyntheticStream(const SyntheticSpec& spec)
    : rows_(std::make_unique<sfdg_tools::SyntheticRows>(spec.n, spec.d, spec.z, spec.p_head, spec.seed)) {}

SyntheticStream::~SyntheticStream() = default;

bool SyntheticStream::has_next() const { return rows_->more(); }

SparseRow SyntheticStream::next() {
    if (!rows_->more()) throw std::logic_error("SyntheticStream: stream exhausted");
    std::vector<std::pair<uint32_t, double>> row;
    rows_->next(row);
    SparseRow r;
    for (const auto& [c, v] : row) {
        r.indices.push_back(c);
        r.values.push_back(v);
    }
    return r;
}

TailResult exact_tail(const SparseBuffer& a, std::size_t k, Rng& rng) {
    const Csr c(a);
    sfdg_rng_state st = rng.device_state();
    TailResult t;
    std::vector<double> sig(k ? k : 1);
    check(sfdg_exact_tail(c.rp.data(), c.cols, c.vals, c.m, c.d, k, &st, sig.data(), &t.tail_sq, nullptr, kDevice));
    rng.set_device_state(st);
    t.sigma.assign(sig.begin(), sig.begin() + static_cast<long>(k));
    return t;
}

std::optional<double> proj_err(const SparseBuffer& a, const DenseMatrix& sketch, std::size_t k, const TailResult& tail) {
    const Csr c(a);
    double v = 0.0;
    int has = 0;
    check(sfdg_proj_err(c.rp.data(), c.cols, c.vals, c.m, c.d, sketch.data.data(), sketch.rows, k, tail.tail_sq, &v,
                        &has, kDevice));
    if (!has) return std::nullopt;
    return v;
}

double cov_err(const SparseBuffer& a, const DenseMatrix& sketch, Rng& rng, std::size_t iterations) {
    if (sketch.cols != a.cols()) throw std::invalid_argument("cov_err: dimension mismatch");
    const Csr c(a);
    sfdg_rng_state st = rng.device_state();
    double v = 0.0;
    check(sfdg_cov_err(c.rp.data(), c.cols, c.vals, c.m, c.d, sketch.data.data(), sketch.rows, iterations, &st, &v,
                       kDevice));
    rng.set_device_state(st);
    return v;
}

MetricsRow timed_run(const std::string& algo, const SparseBuffer& a, const SketchConfig& cfg, std::size_t k,
                     std::size_t z, const TailResult* tail_cache) {
    MetricsRow row;
    row.algo = algo;
    row.n = a.rows();
    row.d = a.cols();
    row.ell = cfg.ell;
    row.z = z;
    row.k = k;
    row.seed = cfg.seed;
    const Csr c(a);
    DenseMatrix sketch;
    const auto t0 = std::chrono::steady_clock::now();
    if (algo == "fd") {
        FdSketcher fd(cfg.ell, cfg.d);
        std::vector<double> dense(cfg.d, 0.0);
        for (std::size_t i = 0; i < c.m; ++i) {
            std::fill(dense.begin(), dense.end(), 0.0);
            for (int64_t p = c.rp[i]; p < c.rp[i + 1]; ++p) dense[c.cols[p]] = c.vals[p];
            fd.append(dense);
        }
        sketch = fd.finalize();
    } else if (algo == "sfd") {
        SfdSketcher s(cfg);
        for (std::size_t i = 0; i < c.m; ++i) {
            SparseRow r;
            r.indices.assign(c.cols + c.rp[i], c.cols + c.rp[i + 1]);
            r.values.assign(c.vals + c.rp[i], c.vals + c.rp[i + 1]);
            s.append(r);
        }
        sketch = s.finalize();
    } else {
        throw std::invalid_argument("timed_run: unknown algorithm tag '" + algo + "'");
    }
    row.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    Rng metrics_rng(cfg.seed ^ 0x9e3779b97f4a7c15ULL);
    const TailResult tail = tail_cache ? *tail_cache : exact_tail(a, k, metrics_rng);
    if (k >= 1) row.proj_err = proj_err(a, sketch, k, tail);
    row.cov_err = cov_err(a, sketch, metrics_rng);
    return row;
}

}  // namespace sfd
