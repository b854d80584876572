// engine.cuh -- device implementation of the SFD flush (see engine.cu).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "sparse.cuh"
#include "verify.cuh"

namespace sfdg {

constexpr double kAlpha = 6.0 / 41.0;  // core/include/sfd/common.hpp:10
constexpr size_t kRetryCap = 64;       // core/src/shrink.cpp:12
constexpr int kMaxEll = 512;           // 2*ell <= 1024: the eigensolver and CholeskyQR limits
constexpr double kKappaTarget = 1e5;   // cond(Y) allowed to build up between CholeskyQR2 passes
constexpr double kKappaUnsafe = 1e7;   // above this CholeskyQR2 may lose orthogonality: redo
constexpr int kMaxInterval = 8;

struct PowerCfg {  // randsvd.hpp:10-14
    double epsilon = 0.25;
    double q_constant = 1.0;
    int64_t q_override = -1;
};

struct Verifier {  // shrink.hpp:11-16
    size_t i = 0;
    double delta = 0.1;
    double c_verify = 2.0;
    double delta_spent = 0.0;
};

size_t power_iteration_count(size_t m, const PowerCfg& cfg);  // randsvd.cpp:10-16

// Adaptive CholeskyQR2 schedule: sweeps between passes so that cond(Y) grows by at most
// kKappaTarget, from the condition number seen after the last pass-1 factorisation.
int next_orth_interval(double kappa_last, int last_since);

// Throws the reference's error class for a set of device error flags (0 = no-op).
void raise_device_flags(int flags);

// Per-device working set for one sketch stream (or one standalone call).
class Engine {
  public:
    // shared_rng: draw from a sketcher-wide generator (flush pipeline lanes) instead of an
    // own one. stack: allocate Mt[2] (= [B^T | B'^T] pairs); lanes only need Bp (d x lp).
    // high_priority: streams at the device's greatest priority (the sketcher's dense-shrink
    // chain, a serial dependency that the lanes' kernels must not starve).
    Engine(int device, int d, int ell, uint64_t seed, uint64_t nnz_cap, int m_cap, RngStream* shared_rng = nullptr,
           bool stack = true, bool high_priority = false);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    int device, d, ell, lp;
    cudaStream_t st = nullptr;
    Scratch scr;
    // dense_shrink of flush f runs on st2 while flush f+1's power iteration runs on st:
    // ev_read_done[i] = the shrink that reads Mt[i] finished; ev_bprime = B' of this flush ready
    cudaStream_t st2 = nullptr;
    Scratch scr2;
    cudaEvent_t ev_read_done[2] = {nullptr, nullptr};
    cudaEvent_t ev_bprime = nullptr;
    std::unique_ptr<RngStream> own_rng;
    RngStream* rng = nullptr;
    RngPos pos;
    DevCsr a;
    SegPlan plan_r, plan_c;
    int m_cap = 0;

    double *Y = nullptr, *Yt = nullptr, *W = nullptr;  // m_cap x lp, m_cap x lp, d x lp
    double* Mt[2] = {nullptr, nullptr};                 // d x 2lp : [B^T | B'^T]
    double* Bp = nullptr;                               // d x lp : this lane's B'^T (no stack)
    int cur = 0;
    double* tinvb = nullptr;  // R^-1 of the current CholeskyQR pass (trsm_apply's inverse + GEMM path)
    double *gram = nullptr, *rinv = nullptr, *rfac = nullptr, *dinv8 = nullptr, *kc = nullptr, *evals = nullptr, *evecs = nullptr, *S = nullptr;
    double *x0 = nullptr, *ybuf = nullptr, *u = nullptr, *tpart = nullptr, *tvec = nullptr, *vpart = nullptr;
    double* vout = nullptr;
    double* xtmp = nullptr;  // m_cap: exact_orth's residual column
    int* d_udrop = nullptr;  // 512: CholeskyQR's uncertain drops
    unsigned* bar = nullptr;
    int* d_err = nullptr;
    double* d_scal = nullptr;  // device scalars
    double* h_scal = nullptr;  // pinned mirror
    int* h_err = nullptr;
    int verify_blocks = 0;
    int* varrive = nullptr;  // arrival counters of the kernel-sequence verifier's long-row pieces
    int64_t varrive_cap = 0;
    int* vcarrive = nullptr;  // ... and of its long-column pieces
    double* vw = nullptr;     // w = A'^T u (d)
    int64_t vcarrive_cap = 0;
    int verify_cluster = 0;  // > 0: the verifier is one cluster of this many CTAs (no grid barrier)
    int vg_blocks = 0;       // column blocks of the kernel-sequence verifier
    // SFDG_VERIFY_MODE=graph: the kernel-sequence verifier (concurrent across flushes). Off by
    // default: on c2 its three dependent kernels per step queue behind the other lanes' work
    // (2.5 ms per verification, 188 ms per stream) where the cooperative kernel holds its 32
    // SMs (1.5 ms, 166 ms per stream, serialised).
    bool use_vgraph = false;
    void* vstate = nullptr;  // the kernel-sequence verifier's device state
    cudaStream_t vst = nullptr;  // its high-priority stream (joined to st by events)
    cudaEvent_t ev_v0 = nullptr, ev_v1 = nullptr;
    // true when this flush's verification runs as the kernel sequence (concurrent-safe);
    // the persistent kernels (skewed columns, or opted in) must be serialised by the caller
    bool verify_as_graph() const { return use_vgraph; }
    // adaptive orthonormalisation schedule (simultaneous_iteration)
    bool adaptive = true;   // SFDG_ORTH_EVERY_SWEEP=1 forces the reference schedule
    int orth_interval = 1;  // sweeps per CholeskyQR2
    int last_since = 1;     // sweeps folded into the last pass-1 factorisation
    // Every pass-1 factorisation followed by exact_orth (chol.cu): CholeskyQR's uncertain
    // column drops re-decided by the reference's rule. Set for attempts replayed after an
    // uncertain drop (with orth_interval = 1, the reference's schedule).
    bool exact_check = false;
    // No kappa history (a stream's first flushes): simultaneous_iteration measures the growth
    // over its first sweep (one host read-back) and picks the interval from it.
    bool probe = false;

    void set_device() const;
    void ensure_rows(int m);
    // Host CSR -> device A' (standalone entry points); panels = false skips the m-row Y panels
    // (metrics over a whole stream only need the CSR/CSC).
    void load_csr(const int64_t* row_ptr, const uint32_t* cols, const double* vals, int m, int64_t nnz,
                  bool panels = true);
    // CSC + long-row plans for the current A'. prepare_async queues the build and the
    // read-back of the long-row counts; prepare_finish consumes them once the stream got there.
    void prepare();
    void prepare_async();
    void prepare_finish();
    int* h_counts = nullptr;  // pinned [4]
    // Per-flush hot columns of the CSR SpMM (sparse.cuh HotSet): chosen on the host from the
    // CSC column counts (h_colptr, copied by prepare_async) in prepare_finish. Opt-in
    // (SFDG_HOT=1): measured slower on c3-c5 (tools/spmm_bench, profiles/r02_spmm_hot.txt) --
    // the L1 already serves the hot rows (21 % hit rate of the plain gather), and the 200 KB of
    // staged rows shrink it for everything else.
    bool hot_enabled = false;
    HotSet hot;
    int* h_colptr = nullptr;  // pinned d + 1
    int* d_hot_cols = nullptr;
    int* d_slot = nullptr;    // d
    int* d_idx2 = nullptr;    // relabelled CSR column indices
    int64_t idx2_cap = 0;
    double hot_share = 0.0;   // share of this flush's nonzeros in the hot columns
    void choose_hot();
    // la_core.cpp:130-165 contract on Y (m x lp, first k columns meaningful): CholeskyQR2.
    void orthonormalize(double* Yp, int m, int err_bit);
    // Single CholeskyQR pass on Y (between sweeps of the adaptive schedule; swaps Y/Yt).
    void orthonormalize_light(int m, int err_bit);
    // `interval` sweeps + the light orthonormalisation that closes them, as one CUDA graph
    // (captured on first use per shape and buffer set, replayed after: ~20 launches -> 1).
    void sweep_block(int interval, int m);
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t kernels = 0;
    };
    std::map<std::vector<uintptr_t>, GraphEntry> graphs;
    std::map<std::array<uintptr_t, 42>, GraphEntry> vgraphs;  // kernel-sequence verifier graphs
    bool use_graphs = true;  // SFDG_GRAPHS=0 disables
    // randsvd.cpp:18-51: Z (m x lp) left in Y.
    void simultaneous_iteration(int k, const PowerCfg& cfg);
    // shrink.cpp:63-73 (+ la_core.cpp:82-128): B'^T (d x lp) into bpt (ld).
    void sparse_shrink(const PowerCfg& cfg, double* bpt, int ldb);
    // shrink.cpp:75-102 on diff_op (shrink.cpp:121-126); host syncs for the verdict.
    bool verify(Verifier& v, double delta_hat, const double* bpt, int ldb);
    // Asynchronous halves: queue the verification (optionally ordered after the event
    // `serial`, re-recorded after it: verify is a persistent grid-barrier kernel, and two of
    // them must never share the GPU) and read its verdict once the stream is past it.
    void verify_enqueue(Verifier& v, double delta_hat, const double* bpt, int ldb, cudaEvent_t serial);
    bool verify_result() const;
    // One sparse_shrink attempt + ||B'||_F^2 + schedule statistics, read back into h_scal
    // (b_fsq at [1], pass-1 stats at [16..23]) and h_err[0] without a host sync.
    void attempt_enqueue(const PowerCfg& cfg, double* bpt, int ldb);
    // shrink.cpp:104-131; B'^T lands in Mt[cur] right half. Returns attempts.
    size_t boosted(Verifier& v, const PowerCfg& cfg, double a_fsq, double* delta_hat_out);
    // dense_shrink (shrink.cpp:30-61) of the row stack whose transpose is Xt (d x kcols, ldx),
    // rows = columns [0, n1) and [off, off + n2) of Xt; writes B^T (d x lp, ldo).
    // side = true: on the shrink stream st2 with its own scratch (overlaps the next flush).
    void dense_shrink_stack(const double* Xt, int ldx, int n1, int off, int n2, double* bt_out, int ldo,
                            bool side = false);
    // Zero the B'^T half of Mt[cur] and scatter the buffer rows of A' into columns
    // [off, off + m) of Mt[cur] (densify, sparse.cpp:71-78, already transposed).
    void densify_into_stack(int off);
    // Same from another engine's buffer (the sketcher's filling lane).
    void densify_into_stack(const DevCsr& src, int off);
    // Rows of this engine's CSR buffer into columns [col0, col0 + m) of dst (d x ld), those
    // columns zeroed first (FdSketcher appends of sparse rows).
    void scatter_rows_t(double* dst, int ld, int col0);
    // Copies the current B (ell x d row-major) to host.
    void sketch_to_host(double* out);
    double read_scalar(const double* dptr);
    void check_errors();  // syncs; throws the reference's error class for any device flag
    void sync();
};

// cov_err (bench.cpp:171-183) of B (ell x d, host row-major) against the A held by e
// (load_csr + prepare done); draws unit_sphere_vector(d) at e.pos (metrics.cu).
double device_cov_err(Engine& e, const double* b_host, int ell, size_t iterations, double a_fsq);
// proj_err (bench.cpp:139-169); false = the reference's nullopt (metrics.cu).
bool device_proj_err(Engine& e, const double* b_host, int ell, int k, double a_fsq, double tail_sq, double* out);
// exact_tail (bench.cpp:68-137) with block = e.ell = min(k + 10, m, d) (metrics.cu).
void device_exact_tail(Engine& e, int k, double a_fsq, double* sigma_out, double* tail_out, size_t* sweeps_out);

}  // namespace sfdg
