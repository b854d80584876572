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
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "dense.cuh"

namespace sfdg {

namespace {

constexpr int kJacThreads = 1024;
constexpr int kMaxSweeps = 100;  // la_core.cpp:31
constexpr int kPackedSmemMax = 230;  // N(N+1)/2 doubles + 16.3 KB static smem <= 227 KB

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
    const int* only_if;  // optional: run only when *only_if != 0 (fallback after eigh_tri)
};

// Rotator CTA. SMEM: the packed upper triangle lives in shared memory (else L2 scratch).
// TABLE: the (K, L) block list of a round is precomputed in shared memory (else derived
// from the linear block index). Per pair k the round keeps {p, q, tri[p], tri[q]} so the
// packed index of any element of a 2 x 2 block costs one compare and one add.
template <bool SMEM, bool TABLE>
__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(JacArgs a) {
    pdl_entry();
    if (a.only_if && *a.only_if == 0) return;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int N = a.N, P = N / 2, n = a.n;
    const size_t packed = (size_t)N * (N + 1) / 2;
    double* A = SMEM ? sm : a.gpacked;
    uint32_t* kl = reinterpret_cast<uint32_t*>(sm + (SMEM ? packed : 0));  // TABLE only
    __shared__ double2 cs[512];
    __shared__ int4 pq[512];  // p, q, tri[p], tri[q]
    __shared__ double red[32];
    __shared__ int s_go;
    const int nblk = P * (P + 1) / 2;
    double tol_sq = a.tol_sq;
    if (a.d_fsq) {  // svd_top / dense_shrink tolerance 1e-12 * max(|a|_F^2, 1) (la_core.cpp:103, shrink.cpp:53)
        const double off_tol = 1e-12 * fmax(*a.d_fsq, 1.0);
        tol_sq = off_tol * off_tol;
    }
    for (int j = warp; j < N; j += nw)  // odd n: index n is a zero pad row/column
        for (int i = lane; i <= j; i += 32)
            A[j * (j + 1) / 2 + i] = (i < n && j < n) ? a.K[(size_t)i * a.ldk + j] : 0.0;
    if (TABLE)
        for (int K = warp; K < P; K += nw) {
            const int base = K * P - K * (K - 1) / 2;
            for (int L = K + lane; L < P; L += 32) kl[base + (L - K)] = ((uint32_t)K << 16) | (uint32_t)L;
        }
    __syncthreads();
    int rounds = 0;
    for (int sweep = 0;; ++sweep) {
        // off-diagonal Frobenius norm^2 of the full symmetric matrix (la_core.cpp:14-20)
        double acc = 0.0;
        for (int j = warp; j < N; j += nw)
            for (int i = lane; i < j; i += 32) {
                const double x = A[j * (j + 1) / 2 + i];
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
                const int tp = p * (p + 1) / 2, tq = q * (q + 1) / 2;
                pq[k] = make_int4(p, q, tp, tq);
                double c = 1.0, s = 0.0;
                const double apq = A[tq + p];
                if (apq != 0.0) {  // la_core.cpp:39-44
                    const double theta = (A[tq + q] - A[tp + p]) / (2.0 * apq);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                    c = 1.0 / sqrt(t * t + 1.0);
                    s = t * c;
                }
                cs[k] = make_double2(c, s);
                a.rotlog[(size_t)rounds * P + k] = make_double2(c, s);
            }
            __syncthreads();
            for (int bidx = tid; bidx < nblk; bidx += nt) {
                int Kb, Lb;
                if (TABLE) {
                    const uint32_t e = kl[bidx];
                    Kb = (int)(e >> 16);
                    Lb = (int)(e & 0xffff);
                } else {
                    Kb = (int)floorf((2.0f * P + 1.0f - sqrtf((2.0f * P + 1.0f) * (2.0f * P + 1.0f) - 8.0f * bidx)) *
                                     0.5f);
                    while (Kb > 0 && Kb * P - Kb * (Kb - 1) / 2 > bidx) --Kb;
                    while ((Kb + 1) * P - (Kb + 1) * Kb / 2 <= bidx) ++Kb;
                    Lb = Kb + (bidx - (Kb * P - Kb * (Kb - 1) / 2));
                }
                const double2 rk = cs[Kb], rl = cs[Lb];
                if (rk.y == 0.0 && rl.y == 0.0) continue;  // identity on both sides
                const int4 K4 = pq[Kb];
                if (Lb == Kb) {
                    double* app = A + K4.z + K4.x;
                    double* aqq = A + K4.w + K4.y;
                    double* apq = A + K4.w + K4.x;
                    const double c = rk.x, s = rk.y;
                    const double xpp = *app, xqq = *aqq, xpq = *apq;
                    const double y11 = c * xpp - s * xpq, y12 = s * xpp + c * xpq;
                    const double y21 = c * xpq - s * xqq, y22 = s * xpq + c * xqq;
                    *app = c * y11 - s * y21;
                    *apq = c * y12 - s * y22;
                    *aqq = s * y12 + c * y22;
                } else {
                    const int4 L4 = pq[Lb];
                    // element (i, j) of the symmetric matrix: i <= j ? tri[j] + i : tri[i] + j
                    double* p11 = A + (K4.x <= L4.x ? L4.z + K4.x : K4.z + L4.x);
                    double* p12 = A + (K4.x <= L4.y ? L4.w + K4.x : K4.z + L4.y);
                    double* p21 = A + (K4.y <= L4.x ? L4.z + K4.y : K4.w + L4.x);
                    double* p22 = A + (K4.y <= L4.y ? L4.w + K4.y : K4.w + L4.y);
                    const double x11 = *p11, x12 = *p12, x21 = *p21, x22 = *p22;
                    const double cl = rl.x, sl = rl.y, ck = rk.x, sk = rk.y;
                    const double y11 = cl * x11 - sl * x12, y12 = sl * x11 + cl * x12;
                    const double y21 = cl * x21 - sl * x22, y22 = sl * x21 + cl * x22;
                    *p11 = ck * y11 - sk * y21;
                    *p21 = sk * y11 + ck * y21;
                    *p12 = ck * y12 - sk * y22;
                    *p22 = sk * y12 + ck * y22;
                }
            }
            ++rounds;
            __syncthreads();
        }
    }
    for (int i = tid; i < N; i += nt) a.diag[i] = A[i * (i + 1) / 2 + i];
    if (tid == 0) *a.progress = rounds;
}

// V = I J_1 J_2 ... J_R. Each warp owns one row of V in shared memory (rows evolve
// independently); the CTA stages kChunk rounds of (c, s) from the log into shared memory
// with one coalesced pass, then every warp applies them to its row.
constexpr int kVRows = 16;
constexpr int kChunk = 8;
__global__ void __launch_bounds__(kVRows * 32) vapply_kernel(int n, int N, const double2* __restrict__ rotlog,
                                                             const int* __restrict__ nrounds, double* __restrict__ V,
                                                             const int* __restrict__ only_if) {
    pdl_entry();
    if (only_if && *only_if == 0) return;
    extern __shared__ double sm[];
    const int P = N / 2;
    double2* cs = reinterpret_cast<double2*>(sm);            // kChunk x P
    short2* pq = reinterpret_cast<short2*>(cs + kChunk * P);  // kChunk x P
    double* rows = reinterpret_cast<double*>(pq + kChunk * P + 2);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int row = blockIdx.x * kVRows + w;
    double* v = rows + (size_t)w * N;
    for (int j = lane; j < N; j += 32) v[j] = (j == row) ? 1.0 : 0.0;
    const int R = *nrounds;
    for (int r0 = 0; r0 < R; r0 += kChunk) {
        const int rc = min(kChunk, R - r0);
        __syncthreads();
        for (int e = threadIdx.x; e < rc * P; e += blockDim.x) {
            const int rr = e / P, k = e % P;
            cs[e] = __ldg(rotlog + (size_t)(r0 + rr) * P + k);
            int p, q;
            pair_of((r0 + rr) % (N - 1), k, N, p, q);
            pq[e] = make_short2((short)p, (short)q);
        }
        __syncthreads();
        if (row < N) {
            for (int rr = 0; rr < rc; ++rr) {
                for (int k = lane; k < P; k += 32) {
                    const double2 c = cs[rr * P + k];
                    if (c.y == 0.0) continue;
                    const short2 ij = pq[rr * P + k];
                    const double vp = v[ij.x], vq = v[ij.y];
                    v[ij.x] = c.x * vp - c.y * vq;
                    v[ij.y] = c.y * vp + c.x * vq;
                }
                __syncwarp();
            }
        }
    }
    if (row < N)
        for (int j = lane; j < N; j += 32) V[(size_t)row * N + j] = v[j];
}

// Stable descending sort of eigenpairs (la_core.cpp:67-78); V (N x N) -> out (n x n).
__global__ void sort_kernel(int n, int N, const double* __restrict__ diag, const double* __restrict__ V,
                            double* __restrict__ values, double* __restrict__ out, int ldo,
                            const int* __restrict__ only_if) {
    pdl_entry();
    if (only_if && *only_if == 0) return;
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

void eigh_tri(const double* K, int n, int ldk, double off_tol, const double* d_fsq, int nval, double* values,
              double* vectors, int ldv, int* fallback, Scratch& scr, cudaStream_t st);

void eigh(const double* K, int n, int ldk, double off_tol, const double* d_fsq, double* values, double* vectors,
          int ldv, int* d_err, Scratch& scr, cudaStream_t st, int nval) {
    if (n <= 0) return;
    if (n > 1024) throw invalid_argument("eigh: n > 1024 unsupported");
    if (nval <= 0 || nval > n) nval = n;
    static const int force_jacobi = [] {
        const char* e = std::getenv("SFDG_EIGH");
        return (e && std::string(e) == "jacobi") ? 1 : 0;
    }();
    int* fallback = scr.take<int>(1);
    if (force_jacobi) {
        CK(cudaMemsetAsync(fallback, 0xff, sizeof(int), st));
    } else {
        CK(cudaMemsetAsync(fallback, 0, sizeof(int), st));
        eigh_tri(K, n, ldk, off_tol, d_fsq, nval, values, vectors, ldv, fallback, scr, st);
    }
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
    a.only_if = fallback;
    if (first_on_device((const void*)(jacobi_kernel<true, true>))) {
        allow_max_dynamic_smem(jacobi_kernel<true, true>);
        allow_max_dynamic_smem(jacobi_kernel<true, false>);
        allow_max_dynamic_smem(vapply_kernel);
    }
    const size_t table = (size_t)P * (P + 1) / 2 * sizeof(uint32_t);
    const bool use_table = use_smem && packed * sizeof(double) + table <= 200 * 1024;
    const size_t smem = use_smem ? packed * sizeof(double) + (use_table ? table : 0) : 0;
    const size_t vsmem = (size_t)kChunk * P * (sizeof(double2) + sizeof(short2)) + 8 + (size_t)kVRows * N * sizeof(double);
    {
        ProfScope prof("eigh_jacobi", st);
        if (use_table) LAUNCH((jacobi_kernel<true, true>), 1, kJacThreads, smem, st, a);
        else if (use_smem) LAUNCH((jacobi_kernel<true, false>), 1, kJacThreads, smem, st, a);
        else LAUNCH((jacobi_kernel<false, false>), 1, kJacThreads, smem, st, a);
    }
    {
        ProfScope prof("eigh_vectors", st);
        LAUNCH(vapply_kernel, ceil_div(N, kVRows), kVRows * 32, vsmem, st, n, N, a.rotlog, a.progress, a.V,
               fallback);
        LAUNCH(sort_kernel, 1, 1024, 0, st, n, N, a.diag, a.V, values, vectors, ldv, fallback);
    }
}

}  // namespace sfdg
