// eigh.cu -- symmetric eigensolver with the jacobi_eigh contract (la_core.cpp:24-80).
//
// The reference runs cyclic Jacobi (row-by-row pair order) until the off-diagonal
// Frobenius norm falls below an absolute tolerance (<= 100 sweeps), then stable-sorts
// eigenpairs by descending eigenvalue. Here the sweep uses the parallel round-robin
// ("tournament") order: each of the N-1 rounds of a sweep rotates N/2 disjoint pairs
// at once. Rotation angles use the reference formula (la_core.cpp:40-44); the stopping
// test is the same off-diagonal norm against the same tolerance, checked at the start
// of every sweep, so the returned spectrum has the same accuracy contract. Any order of
// Jacobi rotations converges to the same eigendecomposition up to roundoff and the
// sign/order of degenerate eigenvectors, to which B^T B is invariant.
//
//  * jacobi_kernel: one CTA keeps the upper triangle packed in shared memory
//    (n <= 232: 216 KB) or L2 (larger n), computes each round's rotations, applies
//    them as independent 2x2 block updates, and logs (c, s) per pair per round.
//  * vapply_kernel: V = J_1 J_2 ... J_R applied row-parallel across the GPU from
//    the log (each row of V evolves independently), off the Jacobi CTA's critical path.
//  * sort_kernel: stable descending order (la_core.cpp:67-78).
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr int kJacThreads = 1024;
constexpr int kMaxSweeps = 100;  // la_core.cpp:31
constexpr int kPackedSmemMax = 232;

__device__ __forceinline__ int pidx(int i, int j) {  // packed upper, i <= j
    return j * (j + 1) / 2 + i;
}

__device__ __forceinline__ void pair_of(int r, int k, int N, int& p, int& q) {
    int a, b;
    if (k == 0) {
        a = N - 1;
        b = r;
    } else {
        a = (r + k) % (N - 1);
        b = (r - k + N - 1) % (N - 1);
    }
    p = min(a, b);
    q = max(a, b);
}

__device__ __forceinline__ double getA(const double* A, int i, int j, int n) {
    if (i >= n || j >= n) return 0.0;
    return i <= j ? A[pidx(i, j)] : A[pidx(j, i)];
}
__device__ __forceinline__ void setA(double* A, int i, int j, int n, double v) {
    if (i >= n || j >= n) return;
    if (i <= j) A[pidx(i, j)] = v;
    else A[pidx(j, i)] = v;
}

__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(const double* __restrict__ K, int n, int ldk,
                                                             double tol_sq, const double* __restrict__ d_fsq,
                                                             double* __restrict__ gpacked,
                                                             int use_smem, double2* __restrict__ rotlog,
                                                             int* __restrict__ nrounds_out,
                                                             double* __restrict__ diag_out, int* __restrict__ err) {
    extern __shared__ double sm[];
    if (d_fsq) {  // svd_top / dense_shrink tolerance 1e-12 * max(|a|_F^2, 1) (la_core.cpp:103, shrink.cpp:53)
        const double off_tol = 1e-12 * fmax(*d_fsq, 1.0);
        tol_sq = off_tol * off_tol;
    }
    double* A = use_smem ? sm : gpacked;
    __shared__ double2 cs[512];
    __shared__ double red[32];
    __shared__ int s_go;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int N = n + (n & 1);
    const int P = N / 2;
    for (int e = tid; e < n * n; e += nt) {
        const int i = e / n, j = e % n;
        if (i <= j) A[pidx(i, j)] = K[(size_t)i * ldk + j];
    }
    __syncthreads();
    int rounds = 0;
    for (int sweep = 0;; ++sweep) {
        // off-diagonal Frobenius norm^2 of the full symmetric matrix (la_core.cpp:14-20)
        double acc = 0.0;
        const int npk = n * (n + 1) / 2;
        for (int e = tid; e < npk; e += nt) {
            // invert packed index: column j with j(j+1)/2 <= e
            int j = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while (j * (j + 1) / 2 > e) --j;
            while ((j + 1) * (j + 2) / 2 <= e) ++j;
            const int i = e - j * (j + 1) / 2;
            if (i != j) acc += 2.0 * A[e] * A[e];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if ((tid & 31) == 0) red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < nt / 32; ++w) s += red[w];
            int go = (s > tol_sq && n > 1) ? 1 : 0;
            if (go && sweep >= kMaxSweeps) {
                atomicOr(err, ERR_JACOBI_NOCONV);
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
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = A[pidx(p, q)];
                    if (apq != 0.0) {
                        const double theta = (A[pidx(q, q)] - A[pidx(p, p)]) / (2.0 * apq);
                        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                cs[k] = make_double2(c, s);
                rotlog[(size_t)rounds * P + k] = make_double2(c, s);
            }
            __syncthreads();
            for (int idx = tid; idx < P * P; idx += nt) {
                const int Kb = idx / P, Lb = idx % P;
                if (Lb < Kb) continue;
                const double2 rk = cs[Kb], rl = cs[Lb];
                if (rk.y == 0.0 && rl.y == 0.0) continue;  // identity on both sides
                int pK, qK, pL, qL;
                pair_of(r, Kb, N, pK, qK);
                pair_of(r, Lb, N, pL, qL);
                if (Kb == Lb) {
                    if (qK >= n) continue;
                    const double app = A[pidx(pK, pK)], aqq = A[pidx(qK, qK)], apq = A[pidx(pK, qK)];
                    const double c = rk.x, s = rk.y;
                    const double y11 = c * app - s * apq, y12 = s * app + c * apq;
                    const double y21 = c * apq - s * aqq, y22 = s * apq + c * aqq;
                    A[pidx(pK, pK)] = c * y11 - s * y21;
                    A[pidx(pK, qK)] = c * y12 - s * y22;
                    A[pidx(qK, qK)] = s * y12 + c * y22;
                } else {
                    const double x11 = getA(A, pK, pL, n), x12 = getA(A, pK, qL, n);
                    const double x21 = getA(A, qK, pL, n), x22 = getA(A, qK, qL, n);
                    const double cl = rl.x, sl = rl.y, ck = rk.x, sk = rk.y;
                    const double y11 = cl * x11 - sl * x12, y12 = sl * x11 + cl * x12;
                    const double y21 = cl * x21 - sl * x22, y22 = sl * x21 + cl * x22;
                    setA(A, pK, pL, n, ck * y11 - sk * y21);
                    setA(A, qK, pL, n, sk * y11 + ck * y21);
                    setA(A, pK, qL, n, ck * y12 - sk * y22);
                    setA(A, qK, qL, n, sk * y12 + ck * y22);
                }
            }
            __syncthreads();
            ++rounds;
        }
    }
    for (int i = tid; i < n; i += nt) diag_out[i] = A[pidx(i, i)];
    if (tid == 0) *nrounds_out = rounds;
}

// V = I * J_1 * ... * J_R, one warp per row of V, row staged in shared memory.
__global__ void vapply_kernel(int n, const double2* __restrict__ rotlog, const int* __restrict__ nrounds,
                              double* __restrict__ V, int ldv) {
    extern __shared__ double rows[];
    const int N = n + (n & 1);
    const int P = N / 2;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * (blockDim.x >> 5) + w;
    double* v = rows + (size_t)w * N;
    for (int j = lane; j < N; j += 32) v[j] = (j == i) ? 1.0 : 0.0;
    __syncwarp();
    const int R = *nrounds;
    if (i < n) {
        for (int r = 0; r < R; ++r) {
            const int rr = r % (N - 1);
            const double2* lg = rotlog + (size_t)r * P;
            for (int k = lane; k < P; k += 32) {
                const double2 cs = lg[k];
                if (cs.y == 0.0) continue;
                int p, q;
                pair_of(rr, k, N, p, q);
                const double vp = v[p], vq = v[q];
                v[p] = cs.x * vp - cs.y * vq;
                v[q] = cs.y * vp + cs.x * vq;
            }
            __syncwarp();
        }
        for (int j = lane; j < n; j += 32) V[(size_t)i * ldv + j] = v[j];
    }
}

// Stable descending sort of eigenpairs (la_core.cpp:67-78); V (n x n) -> out columns.
__global__ void sort_kernel(int n, const double* __restrict__ diag, const double* __restrict__ V, int ldv,
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
        out[(size_t)row * ldo + rank[i]] = V[(size_t)row * ldv + i];
    }
}

}  // namespace

void eigh(const double* K, int n, int ldk, double off_tol, const double* d_fsq, double* values, double* vectors,
          int ldv, int* d_err, Scratch& scr, cudaStream_t st) {
    if (n <= 0) return;
    if (n > 1024) throw invalid_argument("eigh: n > 1024 unsupported");
    const int N = n + (n & 1);
    const int P = N / 2;
    const bool use_smem = n <= kPackedSmemMax;
    const size_t packed = (size_t)n * (n + 1) / 2;
    double* gpk = use_smem ? nullptr : scr.take<double>((int64_t)packed);
    const int64_t max_rounds = (int64_t)kMaxSweeps * (N > 1 ? N - 1 : 1);
    double2* rotlog = scr.take<double2>(std::max<int64_t>(1, max_rounds * P));
    int* nrounds = scr.take<int>(1);
    double* diag = scr.take<double>(n);
    double* V = scr.take<double>((int64_t)n * n);
    static bool attr = false;
    if (!attr) {
        allow_max_dynamic_smem(jacobi_kernel);
        allow_max_dynamic_smem(vapply_kernel);
        attr = true;
    }
    const size_t smem = use_smem ? packed * sizeof(double) : 0;
    {
        ProfScope prof("eigh_jacobi", st);
        LAUNCH(jacobi_kernel, 1, kJacThreads, smem, st, K, n, ldk, off_tol * off_tol, d_fsq, gpk, use_smem ? 1 : 0,
               rotlog, nrounds, diag, d_err);
    }
    const int rows_per_block = 8;
    {
        ProfScope prof("eigh_vectors", st);
        LAUNCH(vapply_kernel, ceil_div(n, rows_per_block), 32 * rows_per_block, rows_per_block * N * sizeof(double),
               st, n, rotlog, nrounds, V, n);
        LAUNCH(sort_kernel, 1, 1024, 0, st, n, diag, V, n, values, vectors, ldv);
    }
}

}  // namespace sfdg
