// common.cuh -- shared host/device helpers for the sfdg library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

namespace sfdg {

// Error classes mirroring the reference (core/include/sfd/common.hpp:14-17); the
// C-ABI maps them to SFDG_INVALID_ARGUMENT / SFDG_NUMERICAL_ERROR / SFDG_CUDA_ERROR.
struct invalid_argument : std::invalid_argument {
    explicit invalid_argument(const std::string& w) : std::invalid_argument(w) {}
};
struct numerical_error : std::runtime_error {
    explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};
struct cuda_error : std::runtime_error {
    explicit cuda_error(const std::string& w) : std::runtime_error(w) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
                 file, line, what);
        throw cuda_error(buf);
    }
}
#define CK(x) ::sfdg::cuda_check((x), #x, __FILE__, __LINE__)

#ifdef __CUDACC__
// Thread-block cluster helpers (sm_90+): rank in the cluster, a full cluster barrier with
// release/acquire semantics for shared::cluster accesses, and the DSMEM address of `p` in
// the CTA of cluster rank `rank`.
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class T>
__device__ __forceinline__ T* cluster_map(T* p, unsigned rank) {
    unsigned long long out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
    return reinterpret_cast<T*>(out);
}
// Programmatic dependent launch (PDL): every kernel starts with pdl_entry(), which waits
// until the previous kernel of the stream has completed and its writes are visible
// (griddepcontrol.wait). With the PDL launch attribute the next kernel is launched as this
// grid's blocks exit instead of after the grid's completion is processed, hiding part of the
// launch latency between the short dependent kernels of a flush (c2: 167 -> 162 ms per
// stream). An early griddepcontrol.launch_dependents at kernel entry was measured slower
// (193 ms): the dependents' waiting blocks hold SM slots the other lanes need. Without the
// attribute the wait is a no-op.
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

// Every kernel launch goes through LAUNCH so the process-wide launch counter
// (sfdg_launch_count) is exact and launch errors surface immediately. Kernels are launched
// with the PDL attribute (see pdl_entry) unless SFDG_PDL=0.
extern std::atomic<uint64_t> g_launches;
bool pdl_enabled();
template <class... KArgs, class... Args>
inline void launch_kernel(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}
// Same launch with an L2 access-policy window: [base, base + bytes) persisting in L2, the
// kernel's other accesses streaming (SpMM panels far larger than L2: the hot columns' rows).
template <class... KArgs, class... Args>
inline void launch_kernel_l2win(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                const void* base, size_t bytes, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    at[na].val.accessPolicyWindow.num_bytes = bytes;
    at[na].val.accessPolicyWindow.hitRatio = 1.0f;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}
#define LAUNCH(kernel, grid, block, smem, stream, ...)                                                \
    do {                                                                                              \
        ::sfdg::launch_kernel(kernel, dim3(grid), dim3(block), (size_t)(smem), (stream), __VA_ARGS__); \
        ::sfdg::g_launches.fetch_add(1, std::memory_order_relaxed);                                   \
    } while (0)

// Times everything a launcher enqueues on `st` between construction and destruction
// under the kernel class `cls` when profiling is on (prof.cu); a no-op otherwise.
extern std::atomic<bool> g_prof_on;
class ProfScope {
  public:
    ProfScope(const char* cls, cudaStream_t st);
    ~ProfScope();
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

    // Algorithmic work of this launch (SURVEY 8(d) formulas), reported by sfdg_profile_end.
    void work(double flops, double bytes) {
        flops_ = flops;
        bytes_ = bytes;
    }

  private:
    const char* cls_ = nullptr;
    double flops_ = 0.0, bytes_ = 0.0;
    cudaStream_t st_;
    cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

// Opt a kernel into the largest dynamic shared memory the device allows next to its
// static shared memory (227 KB per CTA on sm_100a).
template <class F>
inline void allow_max_dynamic_smem(F* func) {
    cudaFuncAttributes attr;
    CK(cudaFuncGetAttributes(&attr, (const void*)func));
    int dev = 0, optin = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CK(cudaFuncSetAttribute((const void*)func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            optin - (int)attr.sharedSizeBytes));
}

// True the first time `key` (a kernel's address) is seen on the calling thread's current
// device; thread-safe. Function attributes such as the dynamic shared memory opt-in are per
// device, so a process driving several GPUs (sfdg_sharded_sketch) must set them on each.
bool first_on_device(const void* key);

inline size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }
inline unsigned ceil_div(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Device error flags (one int array per context); bits set by kernels, read by host.
enum : int {
    ERR_NONFINITE_ITER = 1,     // simultaneous_iteration non-finite intermediate (randsvd.cpp:46-47)
    ERR_NONFINITE_PROJ = 2,     // sparse_shrink non-finite projection (shrink.cpp:70)
    ERR_NONFINITE_VERIFY = 4,   // verify_spectral non-finite operator output (shrink.cpp:90)
    ERR_JACOBI_NOCONV = 8,      // jacobi_eigh 100 sweeps (la_core.cpp:34-35)
    ERR_RNG_U1_ZERO = 16,       // Box-Muller u1 == 0 rejection (rng.cpp:27-29), p = 2^-53
    ERR_BAD_INDEX = 32,         // device-input validation: index out of range / not increasing
    ERR_BAD_VALUE = 64,         // device-input validation: non-finite value
    ERR_NONFINITE_INPUT = 128,  // dense_shrink non-finite input (shrink.cpp:32)
};

}  // namespace sfdg
