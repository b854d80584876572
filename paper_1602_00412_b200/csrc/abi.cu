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
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/sfdg.h"
#include "engine.cuh"
#include "io.cuh"

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

// One host thread per lane: a lane's phase (a few hundred launches) is enqueued off the
// coordinating thread, so the coordinator keeps reacting to the other lanes. Tasks run one
// at a time; busy() is true from post() until the task returned.
class Worker {
  public:
    explicit Worker(int device) : dev(device), th([this] { loop(); }) {}
    ~Worker() {
        {
            std::lock_guard<std::mutex> g(mu);
            stop = true;
        }
        cv.notify_one();
        th.join();
    }
    void post(std::function<void()> f) {
        busy_.store(true, std::memory_order_release);
        {
            std::lock_guard<std::mutex> g(mu);
            task = std::move(f);
            has = true;
        }
        cv.notify_one();
    }
    bool busy() const { return busy_.load(std::memory_order_acquire); }
    void wait() const {
        while (busy()) std::this_thread::yield();
    }
    std::exception_ptr take_error() {
        std::lock_guard<std::mutex> g(mu);
        std::exception_ptr e = err;
        err = nullptr;
        return e;
    }

  private:
    void loop() {
        cudaSetDevice(dev);
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return has || stop; });
                if (!has) return;
                f = std::move(task);
                has = false;
            }
            try {
                f();
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                err = std::current_exception();
            }
            busy_.store(false, std::memory_order_release);
        }
    }
    int dev;
    std::mutex mu;
    std::condition_variable cv;
    std::function<void()> task;
    bool has = false, stop = false;
    std::atomic<bool> busy_{false};
    std::exception_ptr err;
    std::thread th;  // last: starts after the members above exist
};

// Position in the reference's state sequence at a flush boundary: the Rng stream and the
// verifier (sketch.cpp:25-32 threads both through every flush).
struct FlushState {
    RngPos pos;
    Verifier ver;
};

bool same_state(const FlushState& a, const FlushState& b) {
    return a.pos.words == b.pos.words && a.pos.has_spare == b.pos.has_spare && a.ver.i == b.ver.i &&
           a.ver.delta_spent == b.ver.delta_spent;
}

// Flush pipeline.
//
// Flushes are independent SparseShrink problems except for (1) the Rng / verifier state
// they inherit and (2) the dense_shrink chain B_f = dense_shrink([B_{f-1}; B'_f]). So the
// sketcher keeps up to 4 flushes in flight, each on its own lane (engine, stream,
// buffers): a flush starts from the state its predecessor is predicted to end in (one
// attempt that verifies), and is re-run from the true state if the prediction was wrong
// (a retry or an exact-recovery flush upstream). Flushes commit strictly in order; a commit
// queues the dense shrink on the chain stream. Results do not depend on the lane count or
// on timing: every flush is computed from its true start state, and the adaptive
// orthonormalisation interval of flush f depends only on flush f - kLag, which has always
// committed when f starts.
class Sketcher {
  public:
    Sketcher(const SketchCfg& c, int device) : cfg(c) {
        validate_cfg(cfg);
        nnz_trigger = (int64_t)(cfg.ell * cfg.d);
        CK(cudaSetDevice(device));
        const int lanes_n = lane_count();
        const uint64_t per_flush = (uint64_t)cfg.d * cfg.ell + cfg.d + 16;  // raw words drawn per attempt
        rng.init(cfg.seed, std::max<uint64_t>((uint64_t)(lanes_n + 3) * per_flush, 1 << 20), device);
        chain = std::make_unique<Engine>(device, (int)cfg.d, (int)cfg.ell, cfg.seed, 1, 1, &rng, true,
                                         std::getenv("SFDG_CHAIN_PRIORITY") != nullptr &&
                                             std::atoi(std::getenv("SFDG_CHAIN_PRIORITY")) != 0);
        lanes.resize(lanes_n);
        for (auto& L : lanes) {
            L.eng = std::make_unique<Engine>(device, (int)cfg.d, (int)cfg.ell, cfg.seed, (uint64_t)nnz_trigger + cfg.d,
                                             (int)cfg.d, &rng, false);
            CK(cudaEventCreateWithFlags(&L.ev, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&L.ev_bp_free, cudaEventDisableTiming));
            if (use_workers()) L.worker = std::make_unique<Worker>(device);
        }
        CK(cudaEventCreateWithFlags(&ev_verify, cudaEventDisableTiming));
        CK(cudaEventRecord(ev_verify, chain->st));
        if (const char* t = std::getenv("SFDG_TRACE")) {
            trace_path = t;
            CK(cudaEventCreate(&tr_epoch));
            CK(cudaEventRecord(tr_epoch, chain->st));
            CK(cudaStreamSynchronize(chain->st));
            tr_host0 = host_us();
            for (auto& L : lanes) {
                CK(cudaEventCreate(&L.tr0));
                CK(cudaEventCreate(&L.tr1));
            }
        }
        hist.assign(kLag, Hist{});
        committed.ver.delta = cfg.delta;
        fill = 0;
        lanes[0].phase = Lane::Filling;
        lanes[0].clear_rows();
    }

    ~Sketcher() {
        try {
            for (auto& L : lanes)
                if (L.worker) L.worker->wait();
            sync_all();
            if (!trace_path.empty()) dump_trace();
        } catch (...) {
        }
        for (auto& L : lanes) {
            if (L.ev) cudaEventDestroy(L.ev);
            if (L.ev_bp_free) cudaEventDestroy(L.ev_bp_free);
        }
        if (ev_verify) cudaEventDestroy(ev_verify);
    }

    // sync_errors (the public append): the call returns only when every flush it triggered
    // has committed, so a numerical error surfaces here, reported at its trigger row with the
    // reference's state (sketch.cpp:20-32: B and the counters of the last good flush, the
    // failing flush's rows still buffered, rows after the trigger not appended). Without it
    // (the file reader, which overlaps parsing with the device) flushes may still run on return.
    void append_host(const int64_t* rp, const uint32_t* cols, const double* vals, size_t nrows, size_t* done,
                     bool sync_errors = true) {
        chain->set_device();
        if (done) *done = 0;
        // segment() binary-searches row_ptr for the trigger row, which needs it monotone: rows
        // past a decreasing offset are never segmented (the per-row check below rejects it)
        for (size_t i = 0; i < nrows; ++i)
            if (rp[i + 1] < rp[i]) {
                nrows = i + 1;
                break;
            }
        failed_row = -1;
        try {
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
                    finish_copies();
                    if (sync_errors) settle();  // a flush before the bad row fails first (row order)
                    if (done) *done = r + good;
                    throw invalid_argument(err);
                }
                r += take;
                if (done) *done = r;
                trigger_row = (int64_t)r - 1;  // the trigger can only fire at a segment's last row
                maybe_flush();
            }
            finish_copies();  // the caller may reuse its (possibly pinned) buffers on return
            if (sync_errors) settle();
            else pump();
        } catch (const numerical_error&) {
            finish_copies();
            if (done && failed_row >= 0) *done = (size_t)failed_row + 1;
            throw;
        }
    }

    void append_device(const int64_t* h_rp, const uint32_t* d_cols, const double* d_vals, size_t nrows, size_t* done) {
        chain->set_device();
        if (done) *done = 0;
        if (nrows == 0) return;
        size_t bad_rp = nrows;  // first row with a decreasing offset: rows before it are committed
        for (size_t i = 0; i < nrows; ++i)
            if (h_rp[i + 1] < h_rp[i]) {
                bad_rp = i;
                break;
            }
        if (bad_rp < nrows) {
            if (bad_rp > 0) append_device(h_rp, d_cols, d_vals, bad_rp, done);
            if (done) *done = bad_rp;
            throw invalid_argument("append_row: index/value length mismatch");
        }
        Engine& E = *lanes[fill].eng;  // idle apart from row copies
        E.scr.reset();
        int64_t* d_rp = E.scr.take<int64_t>((int64_t)nrows + 1);
        CK(cudaMemcpyAsync(d_rp, h_rp, (nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, E.st));
        int kind = 0;
        const int64_t bad = validate_rows_device(d_rp, (int64_t)nrows, d_cols, d_vals, (uint32_t)cfg.d, &kind, E.scr,
                                                 E.st);
        E.scr.reset();
        const size_t limit = bad < 0 ? nrows : (size_t)bad;
        failed_row = -1;
        try {
            size_t r = 0;
            while (r < limit) {
                const size_t take = segment(h_rp, r, limit);
                commit_device(h_rp, d_cols, d_vals, r, take);
                r += take;
                if (done) *done = r;
                trigger_row = (int64_t)r - 1;
                maybe_flush();
            }
            finish_copies();
            settle();
        } catch (const numerical_error&) {
            finish_copies();
            if (done && failed_row >= 0) *done = (size_t)failed_row + 1;
            throw;
        }
        if (bad >= 0)
            throw invalid_argument((kind & ERR_BAD_INDEX) ? "append_row: column index out of range or not increasing"
                                                          : "append_row: non-finite value");
    }

    void finalize(double* out) {  // sketch.cpp:34-45
        chain->set_device();
        drain();
        Lane& F = lanes[fill];
        if (F.rows() > 0) {
            if (F.rows() >= cfg.ell) {
                trigger_row = -1;
                flush();
                drain();
            } else {
                upload_row_ptr(F);
                CK(cudaStreamSynchronize(F.eng->st));
                const int m = (int)F.rows();
                Engine& C = *chain;
                C.scr.reset();
                C.densify_into_stack(F.eng->a, C.lp);
                C.dense_shrink_stack(C.Mt[C.cur], 2 * C.lp, (int)cfg.ell, C.lp, m, C.Mt[C.cur ^ 1], 2 * C.lp);
                C.check_errors();
                C.cur ^= 1;
                F.clear_rows();
            }
        }
        if (out) get_sketch(out);
    }

    void get_sketch(double* out) {
        chain->set_device();
        drain();
        chain->sync();
        chain->check_errors();
        chain->scr.reset();
        chain->sketch_to_host(out);
    }

    void get_sketch_device(double* d_out, size_t ld) {
        chain->set_device();
        drain();
        chain->sync();
        chain->check_errors();
        copy2d(chain->Mt[chain->cur], (int)cfg.d, (int)cfg.ell, 2 * chain->lp, d_out, (int)ld, chain->st);
        chain->sync();
    }

    void stats(sfdg_stats* s) {
        chain->set_device();
        drain();
        chain->sync();
        const Lane& F = lanes[fill];
        s->flush_count = flushes;
        s->attempt_total = attempts;
        s->verifier = {committed.ver.i, committed.ver.delta, committed.ver.c_verify, committed.ver.delta_spent};
        s->buffer_rows = F.rows();
        s->buffer_nnz = (size_t)F.nnz;
        s->buffer_frob_sq = F.frob;
        s->rng.seed = cfg.seed;
        s->rng.words = committed.pos.words;
        s->rng.has_spare = committed.pos.has_spare ? 1 : 0;
        s->rng.spare = committed.pos.has_spare ? rng.spare_value(committed.pos, chain->st) : 0.0;
    }

    void get_buffer(int64_t* rp, uint32_t* cols, double* vals) {
        chain->set_device();
        Lane& F = lanes[fill];
        CK(cudaStreamSynchronize(F.eng->st));
        if (rp) std::memcpy(rp, F.rp.data(), F.rp.size() * sizeof(int64_t));
        if (F.nnz > 0) {
            if (cols) CK(cudaMemcpyAsync(cols, F.eng->a.col, F.nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost, F.eng->st));
            if (vals) CK(cudaMemcpyAsync(vals, F.eng->a.val, F.nnz * sizeof(double), cudaMemcpyDeviceToHost, F.eng->st));
        }
        CK(cudaStreamSynchronize(F.eng->st));
    }

    void synchronize() {
        chain->set_device();
        drain();
        chain->sync();
    }

    // Back to a freshly constructed sketcher with `seed`, reusing every allocation.
    void reset(uint64_t seed) {
        chain->set_device();
        abort_inflight();
        cfg.seed = seed;
        rng.restart(seed);
        for (int i = 0; i < 2; ++i)
            CK(cudaMemsetAsync(chain->Mt[i], 0, (size_t)cfg.d * 2 * chain->lp * sizeof(double), chain->st));
        chain->cur = 0;
        CK(cudaMemsetAsync(chain->d_err, 0, sizeof(int), chain->st));
        chain->sync();
        for (auto& L : lanes) {
            CK(cudaMemsetAsync(L.eng->d_err, 0, sizeof(int), L.eng->st));
            CK(cudaStreamSynchronize(L.eng->st));
            L.phase = Lane::Idle;
            L.clear_rows();
        }
        committed = FlushState{};
        committed.ver.delta = cfg.delta;
        hist.assign(kLag, Hist{});
        next_id = 0;
        fill = 0;
        lanes[0].phase = Lane::Filling;
        flushes = attempts = 0;
    }

    // this <- merge(this, other) with other's B^T (d x ell, leading dimension ld) already on
    // this sketcher's device (the torchrun shard tree receives it over NCCL). No allocation:
    // the chain's own [B^T | B'^T] pair holds the stack.
    void merge_device(const double* d_bt, size_t ld) {
        chain->set_device();
        drain();
        Engine& C = *chain;
        const int lp = C.lp;
        copy2d(d_bt, (int)cfg.d, (int)cfg.ell, (int)ld, C.Mt[C.cur] + lp, 2 * lp, C.st);
        if (lp > (int)cfg.ell) fill2d(C.Mt[C.cur] + lp + cfg.ell, (int)cfg.d, lp - (int)cfg.ell, 2 * lp, 0.0, C.st);
        C.scr.reset();
        C.dense_shrink_stack(C.Mt[C.cur], 2 * lp, (int)cfg.ell, lp, (int)cfg.ell, C.Mt[C.cur ^ 1], 2 * lp);
        C.check_errors();
        C.cur ^= 1;
    }

    // Shard tree (sfdg_sharded_sketch): B^T lives in the left half of chain Mt[cur].
    Engine& chain_engine() { return *chain; }
    // this <- merge(this, other) = dense_shrink([B_this; B_other]) (sketch.cpp:80-83);
    // `other` may live on another device (peer copy).
    void merge_from(Sketcher& other) {
        drain();
        other.drain();
        other.chain->sync();
        Engine& C = *chain;
        Engine& O = *other.chain;
        C.set_device();
        const int lp = C.lp;
        const size_t bytes = (size_t)cfg.d * 2 * lp * sizeof(double);
        C.scr.reset();
        double* tmp = C.scr.take<double>((int64_t)cfg.d * 2 * lp);
        if (O.device == C.device) CK(cudaMemcpyAsync(tmp, O.Mt[O.cur], bytes, cudaMemcpyDeviceToDevice, C.st));
        else CK(cudaMemcpyPeerAsync(tmp, C.device, O.Mt[O.cur], O.device, bytes, C.st));
        copy2d(tmp, (int)cfg.d, lp, 2 * lp, C.Mt[C.cur] + lp, 2 * lp, C.st);
        C.dense_shrink_stack(C.Mt[C.cur], 2 * lp, (int)cfg.ell, lp, (int)cfg.ell, C.Mt[C.cur ^ 1], 2 * lp);
        C.check_errors();
        C.cur ^= 1;
    }

  private:
    struct Lane {
        std::unique_ptr<Engine> eng;
        enum Phase { Idle, Filling, Preparing, Shrinking, Verifying, Done } phase = Idle;
        std::vector<int64_t> rp{0};
        std::vector<int> rp32;
        int64_t nnz = 0;
        double frob = 0.0;
        uint64_t id = 0;
        FlushState start, cur;
        int interval = 1, interval_base = 1, interval_used = 1;
        bool checked = false, checked_base = false;  // Engine::exact_check for the attempt / flush start
        bool uncertain_seen = false;                 // a checked attempt met uncertain drops
        bool probe = false;  // no kappa history: the attempt measures its own (Engine::probe)
        RngPos pos0;
        size_t attempt = 0;
        double delta_hat = 0.0, kappa_last = 0.0;
        int last_since = 1;
        cudaEvent_t ev = nullptr;          // completion of the queued phase
        cudaEvent_t ev_bp_free = nullptr;  // the chain finished reading Bp
        std::unique_ptr<Worker> worker;            // null: enqueue on the calling thread
        cudaEvent_t tr0 = nullptr, tr1 = nullptr;  // SFDG_TRACE: timed bounds of the queued phase
        double tr_enq = 0.0, tr_enq_end = 0.0;
        bool bp_pending = false;
        int64_t trigger_row = -1;      // row of the append call whose trigger started this flush
        std::exception_ptr failure;    // numerical error of this flush, raised when it is the head
        size_t rows() const { return rp.size() - 1; }
        void clear_rows() {
            rp.assign(1, 0);
            nnz = 0;
            frob = 0.0;
        }
    };
    // The orthonormalisation interval of flush f comes from flush f - kLag (>= the lane
    // count, so committed when f starts): the same schedule for every lane count.
    static constexpr uint64_t kLag = 8;
    // Flushes without history start at a moderate interval; a conditioning blow-up
    // (kappa > kKappaUnsafe) replays that attempt with the every-sweep schedule.
    static constexpr int kFirstInterval = 4;
    static constexpr int kDefaultLanes = 4;
    struct Hist {
        double kappa_last = 0.0;
        int last_since = 1;
        bool valid = false;
        bool checked = false;  // the flush needed exact drop decisions: start checked
    };

    // Flushes in flight: 4, or fewer when 4 lanes' working sets (CSR + CSC of ell*d nnz,
    // Y/Yt of d x lp, W/B' of d x lp, a share of the Rng ring) would exceed 20% of the HBM;
    // 2 when an ell-wide panel (d x lp doubles) is larger than the L2: those SpMMs gather from
    // HBM and extra lanes only contend for it (c5 shard: 2 lanes 6.70 s, 3 lanes 6.89 s, 4 lanes
    // 6.94 s; c3, 6 flushes: 1098 / 1105 / 1146 ms; c4, panels in L2: 3, 4, 6 lanes equal).
    // SFDG_LANES overrides (1 = one flush at a time); the results are the same either way.
    int lane_count() const {
        if (const char* e = std::getenv("SFDG_LANES")) return std::max(1, std::min((int)kLag, std::atoi(e)));
        const double lp = (double)round_up(cfg.ell, 8);
        const double per_lane = 24.0 * ((double)cfg.ell * cfg.d + cfg.d) + 32.0 * cfg.d * lp + 8.0 * cfg.d * (cfg.ell + 1);
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const int fit = (int)std::floor(0.2 * (double)total_b / std::max(per_lane, 1.0));
        int dev = 0, l2 = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
        const int cap = 8.0 * cfg.d * lp > (double)l2 ? 2 : kDefaultLanes;
        return std::max(1, std::min(cap, fit));
    }

    size_t buf_rows() const { return lanes[fill].rows(); }

    // rows [r, r+take) such that the trigger can fire only after the last one
    size_t segment(const int64_t* rp, size_t r, size_t nrows) const {
        const Lane& F = lanes[fill];
        size_t take = std::min(nrows - r, cfg.d - F.rows());
        const int64_t need = nnz_trigger - F.nnz;  // > 0 while the buffer is below the trigger
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
        Lane& F = lanes[fill];
        Engine& e = *F.eng;
        const int64_t b = rp[r], end = rp[r + n];
        if (end > b) {
            CK(cudaMemcpyAsync(e.a.col + F.nnz, cols + b, (end - b) * sizeof(uint32_t), cudaMemcpyHostToDevice, e.st));
            CK(cudaMemcpyAsync(e.a.val + F.nnz, vals + b, (end - b) * sizeof(double), cudaMemcpyHostToDevice, e.st));
        }
        for (int64_t k = b; k < end; ++k) F.frob += vals[k] * vals[k];  // sparse.cpp:22, row order
        for (size_t i = 1; i <= n; ++i) F.rp.push_back(F.nnz + (rp[r + i] - b));
        F.nnz += end - b;
        copies_on.push_back(fill);
    }

    void commit_device(const int64_t* rp, const uint32_t* d_cols, const double* d_vals, size_t r, size_t n) {
        Lane& F = lanes[fill];
        Engine& e = *F.eng;
        const int64_t b = rp[r], end = rp[r + n];
        if (end > b) {
            CK(cudaMemcpyAsync(e.a.col + F.nnz, d_cols + b, (end - b) * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                               e.st));
            CK(cudaMemcpyAsync(e.a.val + F.nnz, d_vals + b, (end - b) * sizeof(double), cudaMemcpyDeviceToDevice, e.st));
            e.scr.reset();
            sumsq(e.a.val + F.nnz, end - b, 1, 1, e.d_scal + 3, nullptr, 0, e.scr, e.st);
            F.frob += e.read_scalar(e.d_scal + 3);
        }
        for (size_t i = 1; i <= n; ++i) F.rp.push_back(F.nnz + (rp[r + i] - b));
        F.nnz += end - b;
    }

    // The host->device row copies of this call are on the streams in copies_on.
    void finish_copies() {
        for (int i : copies_on) CK(cudaStreamSynchronize(lanes[i].eng->st));
        copies_on.clear();
    }

    void maybe_flush() {  // sketch.cpp:22
        const Lane& F = lanes[fill];
        if (F.nnz >= nnz_trigger || F.rows() == cfg.d) flush();
    }

    void upload_row_ptr(Lane& L) {
        const int m = (int)L.rows();
        L.eng->a.set_shape(m, (int)cfg.d, L.nnz);
        L.rp32.resize(m + 1);
        for (int i = 0; i <= m; ++i) L.rp32[i] = (int)L.rp[i];
        CK(cudaMemcpyAsync(L.eng->a.row_ptr, L.rp32.data(), (m + 1) * sizeof(int), cudaMemcpyHostToDevice, L.eng->st));
    }

    // sketch.cpp:25-32: the filling lane's buffer becomes a flush in flight.
    void flush() {
        Lane& L = lanes[fill];
        L.id = next_id++;
        L.trigger_row = trigger_row;
        L.failure = nullptr;
        L.phase = Lane::Preparing;
        run(L, [this, &L] {
            L.eng->scr.reset();
            trace_begin(L);
            upload_row_ptr(L);
            L.eng->prepare_async();
            trace_end(L);
            CK(cudaEventRecord(L.ev, L.eng->st));
        });
        inflight.push_back(fill);
        // the next filling lane: an idle one, committing older flushes until one frees up
        for (;;) {
            int idle = -1;
            for (int i = 0; i < (int)lanes.size(); ++i)
                if (lanes[i].phase == Lane::Idle) {
                    idle = i;
                    break;
                }
            if (idle >= 0) {
                fill = idle;
                break;
            }
            step(true);
        }
        Lane& F = lanes[fill];
        F.clear_rows();
        F.phase = Lane::Filling;
        // no wait here: rows go to the lane's CSR buffer, while the chain may still be reading
        // its previous B' (a separate buffer; the next attempt waits on ev_bp_free)
    }

    FlushState predicted_end(const Lane& P) const {
        if (P.phase == Lane::Done) return P.cur;
        FlushState s = P.start;
        s.pos = rng_advance(rng_advance(s.pos, (uint64_t)cfg.d * cfg.ell), (uint64_t)cfg.d);
        s.ver.i += 1;
        const double di = static_cast<double>(s.ver.i);
        s.ver.delta_spent += s.ver.delta / (2.0 * di * di);
        return s;
    }

    void start_flush(Lane& L, const FlushState& st) {
        L.start = st;
        L.cur = st;
        L.failure = nullptr;
        L.attempt = 0;
        L.interval = L.interval_base;
        L.checked = L.checked_base;
        L.uncertain_seen = false;
        CK(cudaMemsetAsync(L.eng->d_err, 0, sizeof(int), L.eng->st));
        enqueue_attempt(L);
    }

    void enqueue_attempt(Lane& L) {
        if (++L.attempt > kRetryCap) throw numerical_error("boosted_sparse_shrink: retry cap exceeded");
        L.pos0 = L.cur.pos;
        if (L.checked) L.interval = 1;
        L.interval_used = L.eng->adaptive ? L.interval : 1;
        const bool wait_bp = L.bp_pending;  // the chain's dense shrink of this lane's previous B'
        L.bp_pending = false;
        L.phase = Lane::Shrinking;
        run(L, [this, &L, wait_bp] {
            Engine& e = *L.eng;
            e.orth_interval = L.interval_used;
            e.exact_check = L.checked;
            e.probe = L.probe && L.interval_used > 1;
            e.pos = L.cur.pos;
            e.scr.reset();
            if (wait_bp) CK(cudaStreamWaitEvent(e.st, L.ev_bp_free, 0));
            trace_begin(L);
            e.attempt_enqueue(cfg.power, e.Bp, e.lp);
            trace_end(L);
            L.cur.pos = e.pos;
            CK(cudaEventRecord(L.ev, e.st));
        });
    }

    // Enqueue a phase on the lane's worker thread (or inline without workers).
    void run(Lane& L, std::function<void()> f) {
        if (L.worker) L.worker->post(std::move(f));
        else f();
    }

    // Off by default: measured no gain on c2 (212.5 vs 211.1 ms per stream) -- the device,
    // not the enqueueing thread, is the bottleneck with 4 lanes. SFDG_WORKERS=1 enables.
    static bool use_workers() {
        const char* e = std::getenv("SFDG_WORKERS");
        return e && std::atoi(e) != 0;
    }

    // Advance one lane whose queued phase has completed. A numerical error (retry cap,
    // non-finite intermediate) is held on the lane: it is the reference's error only if the
    // lane reaches the head of the queue with its start state confirmed (step()).
    void advance(Lane& L, size_t idx_in_flight) {
        try {
            advance_phase(L, idx_in_flight);
        } catch (const numerical_error&) {
            L.failure = std::current_exception();
            L.phase = Lane::Done;
        }
    }

    void advance_phase(Lane& L, size_t idx_in_flight) {
        Engine& e = *L.eng;
        switch (L.phase) {
            case Lane::Preparing: {
                e.prepare_finish();
                const uint64_t lag = kLag;
                const Hist& h = hist[L.id % lag];
                L.interval_base =
                    (L.id >= lag && h.valid) ? next_orth_interval(h.kappa_last, h.last_since) : kFirstInterval;
                L.checked_base = L.id >= lag && h.valid && h.checked;
                L.probe = !(L.id >= lag && h.valid);
                const FlushState st = idx_in_flight == 0 ? committed : predicted_end(lanes[inflight[idx_in_flight - 1]]);
                start_flush(L, st);
                break;
            }
            case Lane::Shrinking: {
                const double b_fsq = e.h_scal[1];
                const double kappa_last = e.h_scal[16 + 3], kappa_max = e.h_scal[16 + 5];
                const int err = e.h_err[0];
                const double uncertain = e.h_scal[16 + 7] + e.h_scal[24 + 7];
                const int used = e.adaptive ? e.orth_interval : 1;  // a probe may have changed it
                if (!L.checked && (uncertain > 0.0 || (used > 1 && (kappa_max > kKappaUnsafe ||
                                                                                 (err & ERR_NONFINITE_ITER))))) {
                    // redo from the same draws with the every-sweep schedule and exact drop
                    // decisions (as Engine::boosted)
                    CK(cudaMemsetAsync(e.d_err, 0, sizeof(int), e.st));
                    L.cur.pos = L.pos0;
                    L.interval = 1;
                    L.probe = false;
                    L.checked = uncertain > 0.0;  // exact drop decisions only where CholeskyQR cannot vouch
                    --L.attempt;
                    enqueue_attempt(L);
                    break;
                }
                if (L.checked && uncertain > 0.0) L.uncertain_seen = true;
                raise_device_flags(err);
                L.kappa_last = kappa_last;
                L.last_since = e.last_since;
                const double drop = L.frob - b_fsq;  // shrink.cpp:112-113
                const double delta_hat = drop / (kAlpha * static_cast<double>(cfg.ell));
                if (drop <= 1e-12 * L.frob) {  // exact recovery (shrink.cpp:115-118)
                    L.delta_hat = 0.0;
                    L.phase = Lane::Done;
                    break;
                }
                L.delta_hat = delta_hat;
                L.phase = Lane::Verifying;
                run(L, [this, &L, delta_hat] {
                    Engine& e = *L.eng;
                    e.pos = L.cur.pos;
                    trace_begin(L);
                    {
                        std::lock_guard<std::mutex> g(verify_mu);  // keeps the ev_verify chain in order
                        // cluster verifiers run concurrently; grid ones are chained (co-residency)
                        e.verify_enqueue(L.cur.ver, delta_hat, e.Bp, e.lp,
                                         serial_verify && e.verify_cluster == 0 && !e.verify_as_graph()
                                             ? ev_verify
                                             : nullptr);
                    }
                    trace_end(L);
                    L.cur.pos = e.pos;
                    CK(cudaEventRecord(L.ev, e.st));
                });
                break;
            }
            case Lane::Verifying: {
                if (e.verify_result()) L.phase = Lane::Done;
                else enqueue_attempt(L);
                break;
            }
            default:
                break;
        }
    }

    void commit(Lane& L) {
        committed = L.cur;
        if (e_adaptive(L)) hist[L.id % kLag] = Hist{L.kappa_last, L.last_since, true, L.uncertain_seen};
        flushes += 1;
        attempts += L.attempt;
        Engine& C = *chain;
        const int lp = C.lp;
        // B = dense_shrink([B; B']) on the chain stream (the lane's work is complete: its
        // event was observed); errors surface at the next chain sync.
        C.scr.reset();
        cudaEvent_t c0 = nullptr, c1 = nullptr;
        if (!trace_path.empty()) {
            CK(cudaEventCreate(&c0));
            CK(cudaEventCreate(&c1));
            CK(cudaEventRecord(c0, C.st));
        }
        copy2d(L.eng->Bp, (int)cfg.d, lp, lp, C.Mt[C.cur] + lp, 2 * lp, C.st);
        CK(cudaEventRecord(L.ev_bp_free, C.st));
        L.bp_pending = true;
        C.dense_shrink_stack(C.Mt[C.cur], 2 * lp, (int)cfg.ell, lp, (int)cfg.ell, C.Mt[C.cur ^ 1], 2 * lp);
        if (c1) {
            CK(cudaEventRecord(c1, C.st));
            tr_chain.push_back({L.id, c0, c1, host_us()});
        }
        C.cur ^= 1;
        L.phase = Lane::Idle;
        L.clear_rows();
    }

    static bool e_adaptive(const Lane& L) { return L.eng->adaptive; }

    // One round of progress; blocking = wait for the oldest pending phase if nothing moved.
    void step(bool blocking) {
        bool moved = false, head_failed = false;
        try {
            for (size_t k = 0; k < inflight.size(); ++k) {
                Lane& L = lanes[inflight[k]];
                if (L.phase == Lane::Done) continue;
                if (L.worker) {
                    if (L.worker->busy()) continue;  // its phase is still being enqueued
                    if (std::exception_ptr ep = L.worker->take_error()) std::rethrow_exception(ep);
                }
                const cudaError_t q = cudaEventQuery(L.ev);
                if (q == cudaErrorNotReady) continue;
                CK(q);
                trace_observe(L, inflight[k]);
                advance(L, k);
                moved = true;
            }
            while (!inflight.empty()) {
                Lane& L = lanes[inflight.front()];
                if (L.phase != Lane::Done) break;
                if (!same_state(L.start, committed)) {  // mispredicted start: recompute from the truth
                    start_flush(L, committed);
                    moved = true;
                    break;
                }
                if (L.failure) {
                    head_failed = true;
                    break;
                }
                commit(L);
                inflight.pop_front();
                moved = true;
            }
        } catch (...) {
            abort_inflight();
            throw;
        }
        if (head_failed) fail_head();
        // Nothing moved: the caller spins. Polling every lane (rather than blocking on one
        // event) lets whichever lane finishes first get its next phase queued at once.
        if (!moved && blocking) std::this_thread::yield();
    }

    void pump() { step(false); }

    // ---- SFDG_TRACE=<path>: per-phase device intervals and host reaction times (JSON lines)
    static double host_us() {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    void trace_begin(Lane& L) {
        if (trace_path.empty()) return;
        CK(cudaEventRecord(L.tr0, L.eng->st));
        L.tr_enq = host_us();
    }
    void trace_end(Lane& L) {
        if (trace_path.empty()) return;
        CK(cudaEventRecord(L.tr1, L.eng->st));
        L.tr_enq_end = host_us();
    }
    void trace_observe(Lane& L, int lane_idx) {
        if (trace_path.empty()) return;
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, tr_epoch, L.tr0));
        CK(cudaEventElapsedTime(&b, tr_epoch, L.tr1));
        static const char* names[] = {"idle", "filling", "prepare", "shrink", "verify", "done"};
        char buf[384];
        snprintf(buf, sizeof buf,
                 "{\"lane\": %d, \"flush\": %llu, \"phase\": \"%s\", \"gpu_start_us\": %.1f, \"gpu_end_us\": %.1f, "
                 "\"host_enqueue_us\": %.1f, \"host_enqueue_end_us\": %.1f, \"host_observe_us\": %.1f}",
                 lane_idx, (unsigned long long)L.id, names[L.phase], 1e3 * a, 1e3 * b, L.tr_enq - tr_host0,
                 L.tr_enq_end - tr_host0, host_us() - tr_host0);
        tr_lines.push_back(buf);
    }
    void dump_trace() {
        FILE* f = fopen(trace_path.c_str(), "a");
        if (!f) return;
        for (auto& l : tr_lines) fprintf(f, "%s\n", l.c_str());
        for (auto& c : tr_chain) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, tr_epoch, c.e0);
            cudaEventElapsedTime(&b, tr_epoch, c.e1);
            fprintf(f,
                    "{\"lane\": -1, \"flush\": %llu, \"phase\": \"dense_shrink\", \"gpu_start_us\": %.1f, "
                    "\"gpu_end_us\": %.1f, \"host_enqueue_us\": %.1f}\n",
                    (unsigned long long)c.id, 1e3 * a, 1e3 * b, c.host - tr_host0);
            cudaEventDestroy(c.e0);
            cudaEventDestroy(c.e1);
        }
        fclose(f);
        tr_lines.clear();
        tr_chain.clear();
    }

    void drain() {
        while (!inflight.empty()) step(true);
    }

    // End of a public append: every flush it triggered has committed and the chain's dense
    // shrinks have run (their device errors, which cannot be rolled back, are raised here).
    void settle() {
        drain();
        chain->check_errors();
    }

    // The head flush failed for real (sketch.cpp:25-32 throws out of append): the sketcher
    // takes the reference's post-exception state -- B and the counters of the last committed
    // flush, the Rng / verifier advanced by the failed attempts, the failing flush's rows
    // back in the buffer, every later row dropped (never appended in the reference) -- and
    // the error is rethrown with its trigger row in failed_row.
    void fail_head() {
        const int h = inflight.front();
        Lane& L = lanes[h];
        std::exception_ptr ep = L.failure;
        for (auto& K : lanes)
            if (K.worker) {
                K.worker->wait();
                K.worker->take_error();
            }
        for (auto& K : lanes) CK(cudaStreamSynchronize(K.eng->st));
        chain->sync();
        committed = L.cur;
        for (int i : inflight)
            if (i != h) {
                lanes[i].phase = Lane::Idle;
                lanes[i].clear_rows();
            }
        inflight.clear();
        if (fill != h) {
            lanes[fill].phase = Lane::Idle;
            lanes[fill].clear_rows();
        }
        for (auto& K : lanes) CK(cudaMemsetAsync(K.eng->d_err, 0, sizeof(int), K.eng->st));
        fill = h;
        L.phase = Lane::Filling;  // keeps rp / nnz / frob and its device CSR
        L.failure = nullptr;
        failed_row = L.trigger_row;
        copies_on.clear();
        std::rethrow_exception(ep);
    }

    void sync_all() {
        for (auto& L : lanes)
            if (L.worker) L.worker->wait();
        for (auto& L : lanes) CK(cudaStreamSynchronize(L.eng->st));
        chain->sync();
    }

    // Drop every in-flight flush (after an error, or on reset); committed state stays.
    void abort_inflight() {
        for (auto& L : lanes)
            if (L.worker) {
                L.worker->wait();
                L.worker->take_error();
            }
        for (auto& L : lanes) cudaStreamSynchronize(L.eng->st);
        chain->sync();
        for (int i : inflight) {
            lanes[i].phase = Lane::Idle;
            lanes[i].clear_rows();
            CK(cudaMemsetAsync(lanes[i].eng->d_err, 0, sizeof(int), lanes[i].eng->st));
        }
        inflight.clear();
        if (lanes[fill].phase != Lane::Filling) {
            lanes[fill].phase = Lane::Filling;
            lanes[fill].clear_rows();
        }
    }

    SketchCfg cfg;
    RngStream rng;
    std::unique_ptr<Engine> chain;  // B (= Mt[cur] left half), the dense-shrink stream
    std::vector<Lane> lanes;
    std::deque<int> inflight;  // lane indices in flush order
    std::vector<int> copies_on;
    std::vector<Hist> hist;
    std::string trace_path;
    cudaEvent_t tr_epoch = nullptr;
    double tr_host0 = 0.0;
    std::vector<std::string> tr_lines;
    struct ChainTrace {
        uint64_t id;
        cudaEvent_t e0, e1;
        double host;
    };
    std::vector<ChainTrace> tr_chain;
    cudaEvent_t ev_verify = nullptr;
    std::mutex verify_mu;
    bool serial_verify = !(std::getenv("SFDG_VERIFY_SERIAL") && std::atoi(std::getenv("SFDG_VERIFY_SERIAL")) == 0);
    FlushState committed;
    int64_t trigger_row = -1;  // call-relative row whose trigger the next flush() records
    int64_t failed_row = -1;   // trigger row of the flush whose numerical error was raised
    int fill = 0;
    uint64_t next_id = 0;
    int64_t nnz_trigger = 0;
    size_t flushes = 0, attempts = 0;
};

// FdSketcher (core/include/sfd/sketch.hpp:53-67, core/src/sketch.cpp:47-78): dense
// Frequent Directions, the paper's baseline. The 2ell x d work buffer is the engine's
// [B^T | B'^T] pair (d x 2lp): rows 0..ell-1 are columns of the left half, rows
// ell..2ell-1 of the right half, so a full buffer is exactly the dense_shrink stack the
// sketcher uses. Appends are batched: rows are copied to the device and transposed (or,
// for sparse input, scattered) into their columns; a shrink runs whenever the buffer fills.
class FdSketch {
  public:
    FdSketch(size_t ell_, size_t d_, int device) : ell(ell_), d(d_) {
        if (ell < 1 || ell > d) throw invalid_argument("FdSketcher: requires 1 <= ell <= d");  // sketch.cpp:48-49
        if (ell > (size_t)kMaxEll) throw invalid_argument("sfdg: ell must be in [1, 512] for this build");
        if (d >= (size_t)INT32_MAX) throw invalid_argument("FdSketcher: d must be < 2^31");
        e = std::make_unique<Engine>(device, (int)d, (int)ell, 0, 1, 1);
    }

    // n dense rows, row-major (append, sketch.cpp:52-63)
    void append_dense(const double* rows, size_t n) {
        e->set_device();
        size_t r = 0;
        while (r < n) {
            const size_t take = chunk(n - r);
            for (size_t i = r; i < r + take; ++i)
                for (size_t j = 0; j < d; ++j)
                    if (!std::isfinite(rows[i * d + j])) bad = true;
            e->scr.reset();
            double* tmp = e->scr.take<double>((int64_t)take * d);
            CK(cudaMemcpyAsync(tmp, rows + r * d, take * d * sizeof(double), cudaMemcpyHostToDevice, e->st));
            transpose(tmp, (int)take, (int)d, (int)d, e->Mt[e->cur] + col_of(fill), 2 * e->lp, e->st);
            advance(take);
            r += take;
        }
        CK(cudaStreamSynchronize(e->st));
    }

    // n sparse rows (CSR, row_ptr absolute into cols/vals), densified on the device
    void append_csr(const int64_t* rp, const uint32_t* cols, const double* vals, size_t n) {
        e->set_device();
        validate_csr(rp, cols, vals, n, d);
        size_t r = 0;
        while (r < n) {
            const size_t take = chunk(n - r);
            e->ensure_rows((int)take);
            e->load_csr(rp + r, cols, vals, (int)take, rp[r + take] - rp[r]);
            e->scr.reset();
            e->scatter_rows_t(e->Mt[e->cur], 2 * e->lp, col_of(fill));
            advance(take);
            r += take;
        }
        CK(cudaStreamSynchronize(e->st));
    }

    void finalize(double* out) {  // sketch.cpp:65-78
        e->set_device();
        if (fill > ell) shrink(fill - ell);
        e->sync();
        e->check_errors();
        e->scr.reset();
        e->sketch_to_host(out);
    }

    size_t shrink_count() const { return shrinks; }

  private:
    // rows appended in one transfer: up to the next shrink, never across the ell boundary
    size_t chunk(size_t left) const {
        size_t take = std::min(left, 2 * ell - fill);
        if (fill < ell) take = std::min(take, ell - fill);
        return take;
    }
    int col_of(size_t row) const { return row < ell ? (int)row : e->lp + (int)(row - ell); }
    void advance(size_t take) {
        fill += take;
        if (fill == 2 * ell) shrink(ell);
    }
    void shrink(size_t n2) {
        if (bad) throw invalid_argument("dense_shrink: non-finite input");  // shrink.cpp:32
        e->scr.reset();
        e->dense_shrink_stack(e->Mt[e->cur], 2 * e->lp, (int)ell, e->lp, (int)n2, e->Mt[e->cur ^ 1], 2 * e->lp);
        e->cur ^= 1;
        fill = ell;
        shrinks += 1;
    }

    size_t ell, d;
    std::unique_ptr<Engine> e;
    size_t fill = 0, shrinks = 0;
    bool bad = false;
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
    if (e.pos.has_spare) e.rng->set_spare(e.pos, r->spare, e.st);
}

void rng_out(Engine& e, sfdg_rng_state* r) {
    r->words = e.pos.words;
    r->has_spare = e.pos.has_spare ? 1 : 0;
    r->spare = e.pos.has_spare ? e.rng->spare_value(e.pos, e.st) : 0.0;
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
    if (ell > (size_t)kMaxEll) throw invalid_argument("sfdg: ell must be in [1, 512] for this build");
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

struct sfdg_fd_sketcher {
    std::unique_ptr<FdSketch> impl;
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

int sfdg_sketcher_merge_device(sfdg_sketcher* h, const double* d_other_bt, size_t ld) {
    return guard([&] {
        if (!d_other_bt) throw invalid_argument("sfdg_sketcher_merge_device: null argument");
        impl_of(h)->merge_device(d_other_bt, ld);
    });
}

int sfdg_sketcher_reset(sfdg_sketcher* h, uint64_t seed) {
    return guard([&] { impl_of(h)->reset(seed); });
}

int sfdg_sketcher_synchronize(sfdg_sketcher* h) {
    return guard([&] { impl_of(h)->synchronize(); });
}

int sfdg_fd_create(size_t ell, size_t d, int device, sfdg_fd_sketcher** out) {
    return guard([&] {
        if (!out) throw invalid_argument("sfdg_fd_create: null argument");
        if (ell < 1 || ell > d) throw invalid_argument("FdSketcher: requires 1 <= ell <= d");
        require_device(device);
        auto h = std::make_unique<sfdg_fd_sketcher>();
        h->impl = std::make_unique<FdSketch>(ell, d, device);
        *out = h.release();
    });
}

int sfdg_fd_destroy(sfdg_fd_sketcher* h) {
    return guard([&] { delete h; });
}

int sfdg_fd_append(sfdg_fd_sketcher* h, const double* rows, size_t nrows) {
    return guard([&] {
        if (!h || !h->impl) throw invalid_argument("null FD sketcher");
        h->impl->append_dense(rows, nrows);
    });
}

int sfdg_fd_append_csr(sfdg_fd_sketcher* h, const int64_t* row_ptr, const uint32_t* cols, const double* vals,
                       size_t nrows) {
    return guard([&] {
        if (!h || !h->impl) throw invalid_argument("null FD sketcher");
        h->impl->append_csr(row_ptr, cols, vals, nrows);
    });
}

int sfdg_fd_finalize(sfdg_fd_sketcher* h, double* out) {
    return guard([&] {
        if (!h || !h->impl) throw invalid_argument("null FD sketcher");
        h->impl->finalize(out);
    });
}

int sfdg_fd_shrink_count(sfdg_fd_sketcher* h, size_t* count) {
    return guard([&] {
        if (!h || !h->impl || !count) throw invalid_argument("null FD sketcher");
        *count = h->impl->shrink_count();
    });
}

int sfdg_sketch_file(const char* path, size_t plain_cols, const sfdg_sketch_config* cfg, int device, double* out,
                     sfdg_stats* stats, size_t* d_out) {
    return guard([&] {
        if (!path || !cfg) throw invalid_argument("sfdg_sketch_file: null argument");
        require_device(device);
        CK(cudaSetDevice(device));
        SketchCfg c;
        c.ell = cfg->ell;
        c.d = cfg->d;
        c.delta = cfg->delta;
        c.power = to_power(&cfg->power);
        c.seed = cfg->seed;
        std::unique_ptr<Sketcher> sk;
        size_t d = 0;
        auto make = [&] {
            if (sk) return;
            if (c.d == 0) c.d = d;  // tools/sfd_main.cpp:65-69: cfg.d = stream->cols()
            if (c.d != d) throw invalid_argument("sfdg_sketch_file: config d does not match the file's columns");
            validate_cfg(c);
            sk = std::make_unique<Sketcher>(c, device);
        };
        try {
            read_row_stream(path, plain_cols, 0, &d, [&](const int64_t* rp, const uint32_t* cs, const double* vs,
                                                         size_t nrows) {
                make();
                sk->append_host(rp, cs, vs, nrows, nullptr, false);
            });
        } catch (...) {
            if (d_out) *d_out = d;
            throw;
        }
        make();
        sk->finalize(out);
        if (stats) sk->stats(stats);
        if (d_out) *d_out = d;
    });
}

int sfdg_read_row_stream(const char* path, size_t plain_cols, size_t* nrows, size_t* d, size_t* nnz,
                         int64_t* row_ptr, uint32_t* cols, double* vals) {
    return guard([&] {
        if (!path || !nrows || !d || !nnz) throw invalid_argument("sfdg_read_row_stream: null argument");
        std::vector<int64_t> rp{0};
        std::vector<uint32_t> cs;
        std::vector<double> vs;
        size_t dd = 0;
        read_row_stream(path, plain_cols, 0, &dd, [&](const int64_t* r, const uint32_t* c, const double* v,
                                                      size_t n) {
            const int64_t base = rp.back();
            for (size_t i = 1; i <= n; ++i) rp.push_back(base + (r[i] - r[0]));
            cs.insert(cs.end(), c + r[0], c + r[n]);
            vs.insert(vs.end(), v + r[0], v + r[n]);
        });
        *nrows = rp.size() - 1;
        *d = dd;
        *nnz = cs.size();
        if (row_ptr) std::memcpy(row_ptr, rp.data(), rp.size() * sizeof(int64_t));
        if (cols) std::memcpy(cols, cs.data(), cs.size() * sizeof(uint32_t));
        if (vals) std::memcpy(vals, vs.data(), vs.size() * sizeof(double));
    });
}

int sfdg_sharded_sketch(const sfdg_sketch_config* cfg, const int64_t* row_ptr, const uint32_t* cols,
                        const double* vals, size_t nrows, int shards, const int* devices, int ndev, double* out,
                        sfdg_stats* shard_stats) {
    return guard([&] {
        if (!cfg || !row_ptr || !devices) throw invalid_argument("sharded_sketch: null argument");
        if (shards < 1) throw invalid_argument("sharded_sketch: shards must be >= 1");
        if (ndev < 1) throw invalid_argument("sharded_sketch: needs at least one device");
        SketchCfg c;
        c.ell = cfg->ell;
        c.d = cfg->d;
        c.delta = cfg->delta;
        c.power = to_power(&cfg->power);
        c.seed = cfg->seed;
        validate_cfg(c);
        for (int i = 0; i < ndev; ++i) require_device(devices[i]);
        const size_t per = (nrows + shards - 1) / shards;
        std::vector<std::unique_ptr<Sketcher>> sk(shards);
        std::vector<std::string> errs(shards);
        std::vector<int> codes(shards, SFDG_OK);
        std::vector<std::thread> th;
        for (int g = 0; g < shards; ++g)
            th.emplace_back([&, g] {
                codes[g] = guard([&] {
                    const int dev = devices[g % ndev];
                    CK(cudaSetDevice(dev));
                    SketchCfg cg = c;
                    cg.seed = c.seed + (uint64_t)g;  // per-shard seed
                    sk[g] = std::make_unique<Sketcher>(cg, dev);
                    const size_t r0 = std::min(nrows, g * per), r1 = std::min(nrows, (g + 1) * per);
                    if (r1 > r0) sk[g]->append_host(row_ptr + r0, cols, vals, r1 - r0, nullptr);
                    sk[g]->finalize(nullptr);
                });
                if (codes[g] != SFDG_OK) errs[g] = g_last_error;
            });
        for (auto& t : th) t.join();
        for (int g = 0; g < shards; ++g)
            if (codes[g] != SFDG_OK) {
                g_last_error = errs[g];
                if (codes[g] == SFDG_INVALID_ARGUMENT) throw invalid_argument(errs[g]);
                if (codes[g] == SFDG_NUMERICAL_ERROR) throw numerical_error(errs[g]);
                throw cuda_error(errs[g]);
            }
        if (shard_stats)
            for (int g = 0; g < shards; ++g) sk[g]->stats(&shard_stats[g]);
        for (int step = 1; step < shards; step *= 2)  // shards.py tree order, lower rank first
            for (int r = 0; r + step < shards; r += 2 * step) sk[r]->merge_from(*sk[r + step]);
        sk[0]->get_sketch(out);
    });
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
        e.exact_check = true;  // the reference's orthonormalize decisions on every pass
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
        e.exact_check = true;
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

int sfdg_cov_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d, const double* b,
                 size_t ell, size_t iterations, sfdg_rng_state* rng, double* out, int device) {
    return guard([&] {
        if (!row_ptr || !b || !rng || !out) throw invalid_argument("cov_err: null argument");
        if (ell < 1) throw invalid_argument("cov_err: sketch rows must be positive");
        if (d < 1 || d >= (size_t)INT32_MAX) throw invalid_argument("cov_err: dimension mismatch");
        validate_csr(row_ptr, cols, vals, n, d);
        require_device(device);
        const int64_t nnz = row_ptr[n] - row_ptr[0];
        // the power step only needs the stream's CSR / CSC and 2-wide panels: any sketch height
        Engine e(device, (int)d, 1, rng->seed, (uint64_t)std::max<int64_t>(nnz, 1), 1);
        rng_in(e, rng);
        e.load_csr(row_ptr, cols, vals, (int)n, nnz, /*panels=*/false);
        e.prepare();
        *out = device_cov_err(e, b, (int)ell, iterations, csr_frob(row_ptr, vals, n));
        rng_out(e, rng);
    });
}

int sfdg_exact_tail(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d, size_t k,
                    sfdg_rng_state* rng, double* sigma_out, double* tail_out, size_t* sweeps_out, int device) {
    return guard([&] {
        if (!row_ptr || !rng || !tail_out) throw invalid_argument("exact_tail: null argument");
        validate_csr(row_ptr, cols, vals, n, d);
        const double fsq = csr_frob(row_ptr, vals, n);
        size_t sweeps = 0;
        if (k == 0) {  // bench.cpp:70-73
            *tail_out = fsq;
            if (sweeps_out) *sweeps_out = 0;
            return;
        }
        if (k > std::min(n, d)) throw invalid_argument("exact_tail: k exceeds matrix rank bound");
        const size_t block = std::min(k + 10, std::min(n, d));
        if (block > (size_t)kMaxEll) throw invalid_argument("exact_tail: k + 10 must be <= 512 for this build");
        require_device(device);
        const int64_t nnz = row_ptr[n] - row_ptr[0];
        Engine e(device, (int)d, (int)block, rng->seed, (uint64_t)std::max<int64_t>(nnz, 1), (int)n);
        rng_in(e, rng);
        e.load_csr(row_ptr, cols, vals, (int)n, nnz);
        e.prepare();
        std::vector<double> sig(k);
        device_exact_tail(e, (int)k, fsq, sig.data(), tail_out, &sweeps);
        if (sigma_out) std::memcpy(sigma_out, sig.data(), k * sizeof(double));
        if (sweeps_out) *sweeps_out = sweeps;
        rng_out(e, rng);
    });
}

int sfdg_proj_err(const int64_t* row_ptr, const uint32_t* cols, const double* vals, size_t n, size_t d, const double* b,
                  size_t ell, size_t k, double tail_sq, double* out, int* has_value, int device) {
    return guard([&] {
        if (!row_ptr || !b || !out || !has_value) throw invalid_argument("proj_err: null argument");
        if (k < 1 || k > ell) throw invalid_argument("proj_err: k out of range");
        if (ell > (size_t)kMaxEll) throw invalid_argument("proj_err: sketch rows must be in [1, 512]");
        if (ell > d) throw invalid_argument("svd_top: expects m <= d");
        validate_csr(row_ptr, cols, vals, n, d);
        require_device(device);
        const int64_t nnz = row_ptr[n] - row_ptr[0];
        Engine e(device, (int)d, (int)ell, 0, (uint64_t)std::max<int64_t>(nnz, 1), 1);
        e.load_csr(row_ptr, cols, vals, (int)n, nnz, /*panels=*/false);
        e.prepare();
        *has_value = device_proj_err(e, b, (int)ell, (int)k, csr_frob(row_ptr, vals, n), tail_sq, out) ? 1 : 0;
        if (!*has_value) *out = 0.0;
    });
}

int sfdg_power_iteration_count(size_t m, const sfdg_power_config* power, size_t* q) {
    return guard([&] { *q = power_iteration_count(m, to_power(power)); });
}

int sfdg_verify_spectral(sfdg_symop_fn op, void* user, int op_on_device, size_t d, sfdg_verifier_state* state,
                         sfdg_rng_state* rng, int* accepted, int device) {
    return guard([&] {
        if (!op || !state || !rng || !accepted) throw invalid_argument("verify_spectral: null argument");
        if (d < 1) throw invalid_argument("unit_sphere_vector: d must be positive");  // la_core.cpp:175
        require_device(device);
        CK(cudaSetDevice(device));
        // shrink.cpp:76-82 (host arithmetic identical to the reference)
        state->i += 1;
        const double di = static_cast<double>(state->i);
        const double delta_i = state->delta / (2.0 * di * di);
        state->delta_spent += delta_i;
        const size_t steps =
            static_cast<size_t>(std::ceil(state->c_verify * std::log2(static_cast<double>(d) / delta_i)));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct Res {
            cudaStream_t st;
            std::vector<void*> mem;
            ~Res() {
                cudaStreamSynchronize(st);
                for (void* p : mem) cudaFree(p);
                cudaStreamDestroy(st);
            }
        } res{st, {}};
        auto dalloc = [&](size_t n) {
            void* p = nullptr;
            CK(cudaMalloc(&p, n * sizeof(double)));
            res.mem.push_back(p);
            return static_cast<double*>(p);
        };
        double* dx = dalloc(d);
        double* dy = dalloc(d);
        double* dscal = dalloc(2);
        int* derr = reinterpret_cast<int*>(dalloc(1));
        CK(cudaMemsetAsync(derr, 0, sizeof(int), st));
        RngStream rs;
        RngPos pos{rng->words, rng->has_spare != 0};
        rs.init(rng->seed, 4 * d + 64, device);
        if (pos.has_spare) rs.set_spare(pos, rng->spare, st);
        Scratch scr;
        std::vector<double> x(d), y(d);
        // x = unit_sphere_vector(d, rng): d normals in draw order, redrawn while all zero
        for (;;) {
            rs.normals(pos, d, 1, 1, dx, derr, st);
            double nrm_sq = 0.0;
            if (op_on_device) {
                sumsq(dx, (int64_t)d, 1, 1, dscal, nullptr, 0, scr, st);
                CK(cudaMemcpyAsync(&nrm_sq, dscal, sizeof(double), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (nrm_sq > 0.0) {
                    scale_vector(dx, (int64_t)d, 1.0 / std::sqrt(nrm_sq), st);
                    break;
                }
            } else {
                CK(cudaMemcpyAsync(x.data(), dx, d * sizeof(double), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (size_t i = 0; i < d; ++i) nrm_sq += x[i] * x[i];
                if (nrm_sq > 0.0) {
                    const double inv = 1.0 / std::sqrt(nrm_sq);
                    for (double& v : x) v *= inv;
                    break;
                }
            }
        }
        int herr = 0;
        CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        rng->words = pos.words;
        rng->has_spare = pos.has_spare ? 1 : 0;
        rng->spare = pos.has_spare ? rs.spare_value(pos, st) : 0.0;
        if (herr) throw numerical_error("rng: Box-Muller u1 == 0 redraw (probability 2^-53) is not reproduced on device");
        // shrink.cpp:85-101
        double log_mag = 0.0;
        for (size_t t = 0; t < steps; ++t) {
            double nrm_sq = 0.0;
            if (op_on_device) {
                CK(cudaStreamSynchronize(st));
                if (op(dx, dy, d, user) != 0) throw invalid_argument("verify_spectral: operator callback failed");
                CK(cudaDeviceSynchronize());  // the operator's own work, on any stream
                sumsq(dy, (int64_t)d, 1, 1, dscal, derr, ERR_NONFINITE_VERIFY, scr, st);
                CK(cudaMemcpyAsync(&nrm_sq, dscal, sizeof(double), cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                scr.reset();
                if (herr) throw numerical_error("verify_spectral: non-finite operator output");
            } else {
                if (op(x.data(), y.data(), d, user) != 0) throw invalid_argument("verify_spectral: operator callback failed");
                for (double v : y) {
                    if (!std::isfinite(v)) throw numerical_error("verify_spectral: non-finite operator output");
                    nrm_sq += v * v;
                }
            }
            if (nrm_sq == 0.0) {  // iterate annihilated, norm estimate 0
                *accepted = 1;
                return;
            }
            const double nrm = std::sqrt(nrm_sq);
            log_mag += std::log(nrm);
            if (log_mag > 0.0 && nrm >= 1.0) {
                *accepted = 0;
                return;
            }
            if (op_on_device) {
                copy2d(dy, (int)d, 1, 1, dx, 1, st);
                scale_vector(dx, (int64_t)d, 1.0 / nrm, st);
            } else {
                for (size_t i = 0; i < d; ++i) x[i] = y[i] / nrm;
            }
        }
        *accepted = log_mag <= 0.0 ? 1 : 0;
    });
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
        if (pos.has_spare) rs.set_spare(pos, rng->spare, st);
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
        rng->spare = pos.has_spare ? rs.spare_value(pos, st) : 0.0;
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
        if (k < 1 || k > (size_t)kMaxEll) throw invalid_argument("orthonormalize: k must be in [1, 512]");
        require_device(device);
        Engine e(device, 8, (int)k, 0, 1, (int)n);
        CK(cudaMemsetAsync(e.Y, 0, n * e.lp * sizeof(double), e.st));
        double* tmp = e.scr.take<double>((int64_t)n * k);
        CK(cudaMemcpyAsync(tmp, in, n * k * sizeof(double), cudaMemcpyHostToDevice, e.st));
        copy2d(tmp, (int)n, (int)k, (int)k, e.Y, e.lp, e.st);
        e.exact_check = true;
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
