// metrics.cu -- device evaluation metrics cov_err and exact_tail.
//
// Reference: cov_err (core/src/bench.cpp:171-183) = spectral_norm_sym (la_core.cpp:191-211)
// of x -> A^T(A x) - B^T(B x), divided by |A|_F^2. On the CPU it is 1000 power steps over
// the whole stream A -- infeasible at c3-c5 -- here one step is two gather SpMVs over the
// stream's CSR/CSC (the flush SpMM kernels with a 2-wide panel), two passes over B^T and
// fixed-order reductions, captured once as a CUDA graph and replayed `iterations` times.
// The start vector is unit_sphere_vector(d, rng) from the same draw stream as the CPU.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "engine.cuh"
#include "sparse.cuh"

namespace sfdg {

namespace {

constexpr int kMBlocks = 2 * kSMs;

// part[b][j] = sum_{c in block b's rows} bt[c][j] * x[c * 2]   (t = B x, split over rows of B^T)
__global__ void bt_x_partial_kernel(const double* __restrict__ bt, int ldb, int d, int L, const double* __restrict__ x2,
                                    double* __restrict__ part) {
    pdl_entry();
    const int per = (d + gridDim.x - 1) / gridDim.x;
    const int c0 = blockIdx.x * per, c1 = min(d, c0 + per);
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        double s = 0.0;
        for (int c = c0; c < c1; ++c) s = fma(bt[(size_t)c * ldb + j], x2[2 * (size_t)c], s);
        part[(size_t)blockIdx.x * L + j] = s;
    }
}

__global__ void bt_x_reduce_kernel(const double* __restrict__ part, int nb, int L, double* __restrict__ t) {
    pdl_entry();
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[(size_t)b * L + j];  // fixed order
        t[j] = s;
    }
}

// z[c] = (A^T A x)[c] - (B^T t)[c]  (z2 column 0 holds A^T u); per-block partials of x.z, z.z
__global__ void diff_dots_kernel(const double* __restrict__ bt, int ldb, int d, int L, const double* __restrict__ t,
                                 double* __restrict__ z2, const double* __restrict__ x2, double* __restrict__ part) {
    pdl_entry();
    __shared__ double sd[32], sn[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double pd = 0.0, pn = 0.0;
    for (int c = blockIdx.x * nw + w; c < d; c += gridDim.x * nw) {
        double s = 0.0;
        for (int j = lane; j < L; j += 32) s = fma(bt[(size_t)c * ldb + j], t[j], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double z = z2[2 * (size_t)c] - s;
        if (lane == 0) z2[2 * (size_t)c] = z;
        pd = fma(x2[2 * (size_t)c], z, pd);
        pn = fma(z, z, pn);
    }
    if (lane == 0) {
        sd[w] = pd;
        sn[w] = pn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < nw; ++i) {
            a += sd[i];
            b += sn[i];
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

// sc: [0] rayleigh, [1] |y|^2 of this step, [2] annihilated (sticky), [3] non-finite (sticky)
__global__ void step_scalars_kernel(const double* __restrict__ part, int nb, double* __restrict__ sc) {
    pdl_entry();
    if (threadIdx.x != 0) return;
    double dot = 0.0, nrm = 0.0;
    for (int b = 0; b < nb; ++b) {
        dot += part[2 * b];
        nrm += part[2 * b + 1];
    }
    if (sc[2] != 0.0 || sc[3] != 0.0) return;  // the reference has returned already
    if (!isfinite(dot) || !isfinite(nrm)) {
        sc[3] = 1.0;
        return;
    }
    sc[0] = dot;  // la_core.cpp:205
    sc[1] = nrm;
    if (nrm == 0.0) sc[2] = 1.0;  // la_core.cpp:206
}

// x = z / |z| (column 0 of the 2-wide panels), frozen once the reference would have stopped
__global__ void normalize_kernel(const double* __restrict__ z2, double* __restrict__ x2, int d,
                                 const double* __restrict__ sc) {
    pdl_entry();
    if (sc[2] != 0.0 || sc[3] != 0.0) return;
    const double inv = 1.0 / sqrt(sc[1]);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x)
        x2[2 * (size_t)c] = z2[2 * (size_t)c] * inv;
}

// |x0|^2 partials of the raw normals, then x = x0 / |x0| (unit_sphere_vector, la_core.cpp:174-189)
__global__ void sumsq2_partial_kernel(const double* __restrict__ x2, int d, double* __restrict__ part) {
    pdl_entry();
    __shared__ double sh[32];
    double s = 0.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x)
        s = fma(x2[2 * (size_t)c], x2[2 * (size_t)c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += sh[i];
        part[blockIdx.x] = a;
    }
}

__global__ void unit_scale_kernel(double* __restrict__ x2, int d, const double* __restrict__ part, int nb,
                                  int* __restrict__ err) {
    pdl_entry();
    __shared__ double inv;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[b];
        if (!(s > 0.0)) atomicOr(err, ERR_RNG_U1_ZERO);  // an all-zero draw would be redrawn
        inv = 1.0 / sqrt(s);
    }
    __syncthreads();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x) x2[2 * (size_t)c] *= inv;
}

}  // namespace

// cov_err of B (ell x d, host row-major) against the CSR A (host); pos advanced by the d
// draws of unit_sphere_vector. Engine e holds A (load_csr + prepare done by the caller).
double device_cov_err(Engine& e, const double* b_host, int ell, size_t iterations, double a_fsq) {
    if (iterations < 1) throw invalid_argument("spectral_norm_sym: iterations must be >= 1");
    if (a_fsq == 0.0) return 0.0;  // bench.cpp:176
    const int d = e.d, m = e.a.m;
    const int lp = (int)round_up((size_t)ell, 8);  // the sketch's own width: any ell (the engine's is 2-wide)
    cudaStream_t st = e.st;
    Scratch& scr = e.scr;
    // B^T (d x lp) on the device
    double* bhost_dev = scr.take<double>((int64_t)ell * d);
    double* bt = scr.take<double>((int64_t)d * lp);
    CK(cudaMemcpyAsync(bhost_dev, b_host, (size_t)ell * d * sizeof(double), cudaMemcpyHostToDevice, st));
    fill2d(bt, d, lp, lp, 0.0, st);
    transpose(bhost_dev, ell, d, d, bt, lp, st);
    double* x2 = scr.take<double>(2 * (int64_t)d);
    double* u2 = scr.take<double>(2 * (int64_t)std::max(m, 1));
    double* z2 = scr.take<double>(2 * (int64_t)d);
    double* t = scr.take<double>(lp);
    double* tpart = scr.take<double>((int64_t)kMBlocks * lp);
    double* dpart = scr.take<double>(2 * (int64_t)kMBlocks);
    double* sc = scr.take<double>(4);
    CK(cudaMemsetAsync(x2, 0, 2 * (size_t)d * sizeof(double), st));
    CK(cudaMemsetAsync(u2, 0, 2 * (size_t)std::max(m, 1) * sizeof(double), st));
    CK(cudaMemsetAsync(z2, 0, 2 * (size_t)d * sizeof(double), st));
    CK(cudaMemsetAsync(sc, 0, 4 * sizeof(double), st));
    // x = unit_sphere_vector(d, rng): d normals into column 0 of the 2-wide panel
    e.rng->normals(e.pos, (uint64_t)d, 1, 2, x2, e.d_err, st);
    LAUNCH(sumsq2_partial_kernel, kMBlocks, 256, 0, st, x2, d, dpart);
    LAUNCH(unit_scale_kernel, kMBlocks, 256, 0, st, x2, d, dpart, kMBlocks, e.d_err);
    // one power step, captured as a graph
    Scratch& gscr = e.scr;  // SpMM long-row partials come from the same arena (fixed addresses)
    auto step = [&] {
        spmm(e.a.row_ptr, (const int*)e.a.col, e.a.val, m, e.plan_r, e.a.nnz, x2, 2, 2, u2, 2, gscr, st);
        spmm(e.a.col_ptr, e.a.row_idx, e.a.cval, d, e.plan_c, e.a.nnz, u2, 2, 2, z2, 2, gscr, st);
        LAUNCH(bt_x_partial_kernel, kMBlocks, 256, 0, st, bt, lp, d, ell, x2, tpart);
        LAUNCH(bt_x_reduce_kernel, 1, 256, 0, st, tpart, kMBlocks, ell, t);
        LAUNCH(diff_dots_kernel, kMBlocks, 256, 0, st, bt, lp, d, ell, t, z2, x2, dpart);
        LAUNCH(step_scalars_kernel, 1, 32, 0, st, dpart, kMBlocks, sc);
        LAUNCH(normalize_kernel, kMBlocks, 256, 0, st, z2, x2, d, sc);
    };
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    gscr.headroom((size_t)256 << 20);  // the capture must not allocate
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    step();
    CK(cudaStreamEndCapture(st, &graph));
    CK(cudaGraphInstantiate(&exec, graph, 0));
    for (size_t it = 0; it < iterations; ++it) CK(cudaGraphLaunch(exec, st));
    double h[4];
    CK(cudaMemcpyAsync(h, sc, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGraphExecDestroy(exec));
    CK(cudaGraphDestroy(graph));
    e.check_errors();
    if (h[3] != 0.0) throw numerical_error("spectral_norm_sym: non-finite operator output");
    if (h[2] != 0.0) return 0.0;
    return h[0] / a_fsq;
}

// proj_err (core/src/bench.cpp:139-169): |A - A V_k V_k^T|_F^2 / tail with V_k the top-k
// right singular vectors of the sketch (svd_top, la_core.cpp:82-128: Gram B B^T, eigen,
// v = B^T u / s). Device: Gram + eigh, V_k = B^T S (S = U diag(1/s)) by GEMM, then
// |A V_k|_F^2 by one SpMM over the stream, num = |A|_F^2 - |A V_k|_F^2 (the reference sums the
// same per row). Returns false for the reference's nullopt cases.
bool device_proj_err(Engine& e, const double* b_host, int ell, int k, double a_fsq, double tail_sq, double* out) {
    if (k < 1 || k > ell) throw invalid_argument("proj_err: k out of range");
    if (tail_sq < 1e-12 * a_fsq) return false;  // rank <= k input
    const int d = e.d, m = e.a.m, lp = e.lp;
    const int kp = (k + 1) / 2 * 2;
    cudaStream_t st = e.st;
    e.scr.reset();
    double* bdev = e.scr.take<double>((int64_t)ell * d);
    CK(cudaMemcpyAsync(bdev, b_host, (size_t)ell * d * sizeof(double), cudaMemcpyHostToDevice, st));
    fill2d(e.W, d, lp, lp, 0.0, st);
    transpose(bdev, ell, d, d, e.W, lp, st);  // B^T (d x lp)
    double* fsq = e.d_scal + 6;
    sumsq(e.W, d, lp, lp, fsq, nullptr, 0, e.scr, st);
    gram_tn(e.W, d, lp, lp, e.gram, lp, e.scr, st);  // B B^T
    eigh(e.gram, ell, lp, 0.0, fsq, e.evals, e.evecs, ell, e.d_err, e.scr, st, k);  // tol 1e-12 max(|B|^2, 1)
    std::vector<double> lam(k), U((size_t)ell * ell);
    CK(cudaMemcpyAsync(lam.data(), e.evals, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(U.data(), e.evecs, (size_t)ell * ell * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    e.check_errors();
    std::vector<double> sig(k);
    for (int t = 0; t < k; ++t) sig[t] = std::sqrt(std::max(lam[t], 0.0));
    if (sig[0] == 0.0 || sig[k - 1] < 1e-10 * sig[0]) return false;  // no k-dimensional span
    // S (lp x kp): S[i][t] = U[i][t] / s_t
    std::vector<double> S((size_t)lp * kp, 0.0);
    for (int i = 0; i < ell; ++i)
        for (int t = 0; t < k; ++t) S[(size_t)i * kp + t] = U[(size_t)i * ell + t] / sig[t];
    double* Sd = e.scr.take<double>((int64_t)lp * kp);
    double* V = e.scr.take<double>((int64_t)d * kp);
    double* P = e.scr.take<double>((int64_t)std::max(m, 1) * kp);
    CK(cudaMemcpyAsync(Sd, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    gemm_nn(e.W, d, lp, lp, Sd, kp, kp, V, kp, st);  // V_k = B^T U / s  (d x kp)
    spmm(e.a.row_ptr, (const int*)e.a.col, e.a.val, m, e.plan_r, e.a.nnz, V, kp, kp, P, kp, e.scr, st);  // A V_k
    double* pe = e.d_scal + 7;
    sumsq(P, m, kp, kp, pe, nullptr, 0, e.scr, st);
    const double proj = e.read_scalar(pe);
    *out = std::max(a_fsq - proj, 0.0) / tail_sq;
    return true;
}

// exact_tail (core/src/bench.cpp:68-137): |A - A_k|_F^2 by block power iteration with block
// = k + 10 columns (the engine's ell), <= 1000 sweeps, the reference's convergence tests on
// the top-k Ritz values of W^T W (W = A^T Y). A (whole stream) is held by e (load_csr with
// panels + prepare done); the Gaussian start block is drawn at e.pos.
void device_exact_tail(Engine& e, int k, double a_fsq, double* sigma_out, double* tail_out, size_t* sweeps_out) {
    *sweeps_out = 0;
    if (k == 0) {
        *tail_out = a_fsq;
        return;
    }
    const int m = e.a.m, d = e.d, lp = e.lp, block = e.ell;
    cudaStream_t st = e.st;
    e.exact_check = true;  // the reference's orthonormalize decisions (rank-deficient blocks)
    e.scr.reset();
    e.rng->normals(e.pos, (uint64_t)d * block, (uint64_t)block, (uint64_t)lp, e.W, e.d_err, st);  // la_core.cpp:167
    spmm(e.a.row_ptr, (const int*)e.a.col, e.a.val, m, e.plan_r, e.a.nnz, e.W, lp, lp, e.Y, lp, e.scr, st);
    e.orthonormalize(e.Y, m, ERR_NONFINITE_ITER);
    std::vector<double> prev(k, -1.0), est(k), vals(block);
    double prev_energy = -1.0;
    const double tol = 1e-14 * std::max(a_fsq, 1.0);
    for (size_t sweep = 0; sweep < 1000; ++sweep) {
        e.scr.reset();
        spmm(e.a.col_ptr, e.a.row_idx, e.a.cval, d, e.plan_c, e.a.nnz, e.Y, lp, lp, e.W, lp, e.scr, st);  // W = A^T Y
        spmm(e.a.row_ptr, (const int*)e.a.col, e.a.val, m, e.plan_r, e.a.nnz, e.W, lp, lp, e.Y, lp, e.scr, st);  // next
        gram_tn(e.W, d, lp, lp, e.gram, lp, e.scr, st);  // small = W^T W (block x block leading part)
        eigh(e.gram, block, lp, tol, nullptr, e.evals, e.evecs, block, e.d_err, e.scr, st, k);
        CK(cudaMemcpyAsync(vals.data(), e.evals, k * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double change = 0.0, head = 0.0;
        for (int i = 0; i < k; ++i) {
            est[i] = std::sqrt(std::max(vals[i], 0.0));
            change = std::max(change, std::abs(est[i] - prev[i]));
            head += est[i] * est[i];
        }
        const double scale = std::max(est[0], 1.0);
        const bool values_done = sweep > 0 && change <= 1e-10 * scale;
        const bool energy_done = sweep >= 30 && std::abs(head - prev_energy) <= 1e-9 * std::max(head, 1.0);
        if (values_done || energy_done) {
            for (int i = 0; i < k; ++i) sigma_out[i] = est[i];
            *tail_out = std::max(a_fsq - head, 0.0);
            *sweeps_out = sweep + 1;
            e.check_errors();
            return;
        }
        prev = est;
        prev_energy = head;
        e.orthonormalize(e.Y, m, ERR_NONFINITE_ITER);
    }
    throw numerical_error("exact_tail: no convergence within 1000 sweeps");
}

}  // namespace sfdg
