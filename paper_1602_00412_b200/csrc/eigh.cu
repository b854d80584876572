// eigh.cu -- symmetric eigensolver with the jacobi_eigh contract (la_core.cpp:24-80).
//
// The reference runs cyclic Jacobi (row-by-row pair order) until the off-diagonal
// Frobenius norm falls below an absolute tolerance (<= 100 sweeps), then stable-sorts
// eigenpairs by descending eigenvalue. Here each sweep uses the parallel round-robin
// ("tournament") order: each of the N-1 rounds rotates N/2 disjoint pairs at once.
// Rotation angles use the reference formula (la_core.cpp:40-44); the stopping test is the
// same off-diagonal norm against the same tolerance, checked at the start of every sweep,
// so the returned spectrum has the same accuracy contract. Any order of Jacobi rotations
// converges to the same eigendecomposition up to roundoff and the sign/order of
// degenerate eigenvectors, to which B^T B is invariant.
//
// One cooperative launch, two roles:
//  * CTA 0 (the rotator) keeps the upper triangle packed in shared memory (N <= 232) or
//    L2 (larger N), computes each round's N/2 rotations, applies them as independent 2x2
//    block updates, and publishes (c, s) per pair per round to a log in global memory.
//  * CTAs 1.. (the accumulators) each own 32 rows of V = J_1 J_2 ... and apply rounds
//    as soon as CTA 0 publishes them (progress counter), so the eigenvector accumulation
//    runs concurrently on other SMs instead of after the sweeps.
// A final pass sorts eigenpairs (stable, descending; la_core.cpp:67-78).
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr int kJacThreads = 1024;
constexpr int kMaxSweeps = 100;  // la_core.cpp:31
constexpr int kPackedSmemMax = 232;
constexpr int kRowsPerAcc = kJacThreads / 32;

__device__ __forceinline__ int pidx(int i, int j) {  // packed upper, i <= j
    return j * (j + 1) / 2 + i;
}

__device__ __forceinline__ void pair_of(int r, int k, int N, int& p, int& q) {
    int a, b;
    if (k == 0) {
        a = N - 1;
        b = r;
    } else {
        a = r + k;
        if (a >= N - 1) a -= N - 1;
        b = r - k;
        if (b < 0) b += N - 1;
    }
    p = min(a, b);
    q = max(a, b);
}

__device__ __forceinline__ double& at(double* A, int i, int j) { return i <= j ? A[pidx(i, j)] : A[pidx(j, i)]; }

struct JacArgs {
    const double* K;
    int n, ldk, N;
    double tol_sq;
    const double* d_fsq;
    double* gpacked;
    int use_smem;
    double2* rotlog;
    int* progress;  // [rounds published, done flag]
    double* diag;
    double* V;  // N x N accumulated rotations (row-major)
    int* err;
};

__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(JacArgs a) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int N = a.N, P = N / 2, n = a.n;

    if (blockIdx.x > 0) {
        // ---------------- accumulator CTA: rows of V
        const int row = (blockIdx.x - 1) * kRowsPerAcc + warp;
        double* v = sm + (size_t)warp * N;
        for (int j = lane; j < N; j += 32) v[j] = (j == row) ? 1.0 : 0.0;
        __syncwarp();
        volatile int* prog = a.progress;
        int r = 0;
        for (;;) {
            int avail = prog[0];
            const int done = prog[1];
            if (r >= avail) {
                if (done) {
                    avail = prog[0];
                    if (r >= avail) break;
                } else {
                    __nanosleep(64);
                    continue;
                }
            }
            __threadfence();
            for (; r < avail; ++r) {
                if (row < N) {
                    const int rr = r % (N - 1);
                    const double2* lg = a.rotlog + (size_t)r * P;
                    for (int k = lane; k < P; k += 32) {
                        const double2 cs = __ldcg(lg + k);
                        if (cs.y == 0.0) continue;
                        int p, q;
                        pair_of(rr, k, N, p, q);
                        const double vp = v[p], vq = v[q];
                        v[p] = cs.x * vp - cs.y * vq;
                        v[q] = cs.y * vp + cs.x * vq;
                    }
                }
                __syncwarp();
            }
        }
        if (row < N)
            for (int j = lane; j < N; j += 32) a.V[(size_t)row * N + j] = v[j];
        return;
    }

    // ---------------- rotator CTA
    double* A = a.use_smem ? sm : a.gpacked;
    __shared__ double2 cs[512];
    __shared__ int pp[512], qq[512];
    __shared__ double red[32];
    __shared__ int s_go;
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {  // svd_top / dense_shrink tolerance 1e-12 * max(|a|_F^2, 1) (la_core.cpp:103, shrink.cpp:53)
        const double off_tol = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = off_tol * off_tol;
    }
    for (int e = tid; e < N * N; e += nt) {  // odd n: index n is a zero pad row/column
        const int i = e / N, j = e % N;
        if (i <= j) A[pidx(i, j)] = (i < n && j < n) ? a.K[(size_t)i * a.ldk + j] : 0.0;
    }
    __syncthreads();
    int rounds = 0;
    for (int sweep = 0;; ++sweep) {
        // off-diagonal Frobenius norm^2 of the full symmetric matrix (la_core.cpp:14-20)
        double acc = 0.0;
        for (int j = warp; j < N; j += nw)
            for (int i = lane; i < j; i += 32) {
                const double x = A[pidx(i, j)];
                acc += 2.0 * x * x;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[w];
            int go = (s > tol_sq && n > 1) ? 1 : 0;
            if (go && sweep >= kMaxSweeps) {
                atomicOr(a.err, ERR_JACOBI_NOCONV);
                go = 0;
            }
            s_go = go;
        }
        __syncthreads();
        if (!s_go) break;
        for (int r = 0; r < N - 1; ++r) {
            for (int k = tid; k < P; k += nt) {
                int p, q;
                pair_of(r, k, N, p, q);
                pp[k] = p;
                qq[k] = q;
                double c = 1.0, s = 0.0;
                const double apq = A[pidx(p, q)];
                if (apq != 0.0) {
                    const double theta = (A[pidx(q, q)] - A[pidx(p, p)]) / (2.0 * apq);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                    c = 1.0 / sqrt(t * t + 1.0);
                    s = t * c;
                }
                cs[k] = make_double2(c, s);
                a.rotlog[(size_t)rounds * P + k] = make_double2(c, s);
                __threadfence();  // log visible device-wide before the round is published
            }
            __syncthreads();
            // block rows K in snake order over warps; lanes sweep L >= K
            const int kend = ((P + nw - 1) / nw) * nw;
            for (int qk = warp; qk < kend; qk += nw) {
                const int rnd = qk / nw, pos = qk % nw;
                const int Kb = (rnd & 1) ? rnd * nw + (nw - 1 - pos) : qk;
                if (Kb >= P) continue;
                const double2 rk = cs[Kb];
                const int pK = pp[Kb], qK = qq[Kb];
                for (int Lb = Kb + lane; Lb < P; Lb += 32) {
                    const double2 rl = cs[Lb];
                    if (rk.y == 0.0 && rl.y == 0.0) continue;
                    if (Lb == Kb) {
                        double& app = A[pidx(pK, pK)];
                        double& aqq = A[pidx(qK, qK)];
                        double& apq = A[pidx(pK, qK)];
                        const double c = rk.x, s = rk.y;
                        const double y11 = c * app - s * apq, y12 = s * app + c * apq;
                        const double y21 = c * apq - s * aqq, y22 = s * apq + c * aqq;
                        app = c * y11 - s * y21;
                        apq = c * y12 - s * y22;
                        aqq = s * y12 + c * y22;
                    } else {
                        const int pL = pp[Lb], qL = qq[Lb];
                        double& x11 = at(A, pK, pL);
                        double& x12 = at(A, pK, qL);
                        double& x21 = at(A, qK, pL);
                        double& x22 = at(A, qK, qL);
                        const double cl = rl.x, sl = rl.y, ck = rk.x, sk = rk.y;
                        const double y11 = cl * x11 - sl * x12, y12 = sl * x11 + cl * x12;
                        const double y21 = cl * x21 - sl * x22, y22 = sl * x21 + cl * x22;
                        x11 = ck * y11 - sk * y21;
                        x21 = sk * y11 + ck * y21;
                        x12 = ck * y12 - sk * y22;
                        x22 = sk * y12 + ck * y22;
                    }
                }
            }
            ++rounds;
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicExch(a.progress, rounds);  // publish this round to the accumulators
            }
        }
    }
    for (int i = tid; i < N; i += nt) a.diag[i] = A[pidx(i, i)];
    if (tid == 0) {
        __threadfence();
        atomicExch(a.progress, rounds);
        atomicExch(a.progress + 1, 1);
    }
}

// Stable descending sort of eigenpairs (la_core.cpp:67-78); V (N x N) -> out (n x n).
__global__ void sort_kernel(int n, int N, const double* __restrict__ diag, const double* __restrict__ V,
                            double* __restrict__ values, double* __restrict__ out, int ldo) {
    __shared__ int rank[1024];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double di = diag[i];
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const double dj = diag[j];
            if (dj > di || (dj == di && j < i)) ++r;
        }
        rank[i] = r;
        values[r] = di;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int row = e / n, i = e % n;
        out[(size_t)row * ldo + rank[i]] = V[(size_t)row * N + i];
    }
}

}  // namespace

void eigh(const double* K, int n, int ldk, double off_tol, const double* d_fsq, double* values, double* vectors,
          int ldv, int* d_err, Scratch& scr, cudaStream_t st) {
    if (n <= 0) return;
    if (n > 1024) throw invalid_argument("eigh: n > 1024 unsupported");
    const int N = n + (n & 1);
    const int P = N / 2;
    const bool use_smem = N <= kPackedSmemMax;
    const size_t packed = (size_t)N * (N + 1) / 2;
    JacArgs a{};
    a.K = K;
    a.n = n;
    a.ldk = ldk;
    a.N = N;
    a.tol_sq = off_tol * off_tol;
    a.d_fsq = d_fsq;
    a.gpacked = use_smem ? nullptr : scr.take<double>((int64_t)packed);
    a.use_smem = use_smem ? 1 : 0;
    const int64_t max_rounds = (int64_t)kMaxSweeps * (N - 1) + 1;
    a.rotlog = scr.take<double2>(std::max<int64_t>(1, max_rounds * P));
    a.progress = scr.take<int>(2);
    a.diag = scr.take<double>(N);
    a.V = scr.take<double>((int64_t)N * N);
    a.err = d_err;
    static bool attr = false;
    if (!attr) {
        allow_max_dynamic_smem(jacobi_kernel);
        attr = true;
    }
    const size_t smem = std::max(use_smem ? packed * sizeof(double) : 0, (size_t)kRowsPerAcc * N * sizeof(double));
    const int nacc = (N + kRowsPerAcc - 1) / kRowsPerAcc;
    CK(cudaMemsetAsync(a.progress, 0, 2 * sizeof(int), st));
    {
        ProfScope prof("eigh", st);
        void* params[] = {(void*)&a};
        CK(cudaLaunchCooperativeKernel((const void*)jacobi_kernel, dim3(1 + nacc), dim3(kJacThreads), params, smem,
                                       st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        LAUNCH(sort_kernel, 1, 1024, 0, st, n, N, a.diag, a.V, values, vectors, ldv);
    }
}

}  // namespace sfdg
