// B200 (sm_100a) device kernels for the AeroSketch update path.
// fp64 throughout: the reference computes in fp64 (Eigen MatrixXd) and the
// parity contract compares decision traces, which fp64 keeps bit-stable.
#include <algorithm>
#include <atomic>

#include "aero_common.cuh"
#include "kernels.cuh"
#include "ozaki.cuh"
#include "tiles.cuh"

namespace aero_b200 {

static std::atomic<long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launches_total() { return g_launches.load(); }

// ============================================================================
// fp64 GEMM (column-major): D = alpha op(A) op(B) + beta D, optional row mask
// per output column (rows >= colmask[j] written as 0). Register-blocked DFMA
// with double-buffered shared-memory tiles; micro-tile rows/cols are strided
// so that a warp's shared-memory reads are conflict-free.
// ============================================================================
template <int BM, int BN, int BK, int TM, int TN, bool TA, bool TB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_dgemm(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
            const double* __restrict__ B, int ldb, double beta, double* __restrict__ D, int ldd,
            const int* __restrict__ colmask) {
    constexpr int RT = BM / TM, CT = BN / TN, NT = RT * CT;
    constexpr int LA = (BM * BK) / NT, LB = (BK * BN) / NT;
    static_assert((BM * BK) % NT == 0 && (BK * BN) % NT == 0, "tile/thread mismatch");
    __shared__ double As[2][BK][BM];
    __shared__ double Bs[2][BK][BN];
    const int tid = threadIdx.x;
    const int bm = blockIdx.y * BM, bn = blockIdx.x * BN;
    const int tr = tid % RT, tc = tid / RT;
    double acc[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;
    double ra[LA], rb[LB];
    auto load = [&](int k0) {
#pragma unroll
        for (int s = 0; s < LA; ++s) {
            const int e = tid + s * NT;
            int i, l;
            if (!TA) { i = e % BM; l = e / BM; } else { l = e % BK; i = e / BK; }
            const int gi = bm + i, gl = k0 + l;
            double v = 0.0;
            if (gi < m && gl < k) v = TA ? A[gl + (int64_t)gi * lda] : A[gi + (int64_t)gl * lda];
            ra[s] = v;
        }
#pragma unroll
        for (int s = 0; s < LB; ++s) {
            const int e = tid + s * NT;
            int j, l;
            if (!TB) { l = e % BK; j = e / BK; } else { j = e % BN; l = e / BN; }
            const int gj = bn + j, gl = k0 + l;
            double v = 0.0;
            if (gj < n && gl < k) v = TB ? B[gj + (int64_t)gl * ldb] : B[gl + (int64_t)gj * ldb];
            rb[s] = v;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int s = 0; s < LA; ++s) {
            const int e = tid + s * NT;
            int i, l;
            if (!TA) { i = e % BM; l = e / BM; } else { l = e % BK; i = e / BK; }
            As[buf][l][i] = ra[s];
        }
#pragma unroll
        for (int s = 0; s < LB; ++s) {
            const int e = tid + s * NT;
            int j, l;
            if (!TB) { l = e % BK; j = e / BK; } else { j = e % BN; l = e / BN; }
            Bs[buf][l][j] = rb[s];
        }
    };
    const int nk = (k + BK - 1) / BK;
    if (nk > 0) {
        load(0);
        store(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int cur = kt & 1;
        if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double av[TM], bv[TN];
#pragma unroll
            for (int a = 0; a < TM; ++a) av[a] = As[cur][kk][tr + a * RT];
#pragma unroll
            for (int b = 0; b < TN; ++b) bv[b] = Bs[cur][kk][tc + b * CT];
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        if (kt + 1 < nk) store(cur ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < TN; ++b) {
        const int gj = bn + tc + b * CT;
        if (gj >= n) continue;
        const int lim = colmask ? colmask[gj] : m;
#pragma unroll
        for (int a = 0; a < TM; ++a) {
            const int gi = bm + tr + a * RT;
            if (gi >= m) continue;
            double* p = D + gi + (int64_t)gj * ldd;
            double v = alpha * acc[a][b];
            if (beta != 0.0) v = fma(beta, *p, v);
            if (gi >= lim) v = 0.0;
            *p = v;
        }
    }
}

template <int BM, int BN, int TM, int TN>
static void launch_gemm(cudaStream_t st, bool ta, bool tb, int m, int n, int k, double alpha,
                        const double* A, int lda, const double* B, int ldb, double beta, double* D,
                        int ldd, const int* colmask) {
    constexpr int NT = (BM / TM) * (BN / TN);
    dim3 grid((n + BN - 1) / BN, (m + BM - 1) / BM);
    if (!ta && !tb)
        k_dgemm<BM, BN, 16, TM, TN, false, false><<<grid, NT, 0, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
    else if (ta && !tb)
        k_dgemm<BM, BN, 16, TM, TN, true, false><<<grid, NT, 0, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
    else if (!ta && tb)
        k_dgemm<BM, BN, 16, TM, TN, false, true><<<grid, NT, 0, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
    else
        k_dgemm<BM, BN, 16, TM, TN, true, true><<<grid, NT, 0, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
    AERO_LAUNCHED();
}

void dgemm(cudaStream_t st, bool ta, bool tb, int m, int n, int k, double alpha, const double* A,
           int lda, const double* B, int ldb, double beta, double* D, int ldd,
           const int* colmask) {
    if (m <= 0 || n <= 0) return;
    const long long big = (long long)((m + 63) / 64) * ((n + 63) / 64);
    if (big >= 120)
        launch_gemm<64, 64, 4, 4>(st, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
    else
        launch_gemm<32, 32, 2, 2>(st, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, D, ldd, colmask);
}

// ============================================================================
// ingestion (K1): per-row squared norm + finiteness, one warp per row,
// coalesced 8-byte loads (reference sketch.cpp:83-84, attp.hpp:22)
// ============================================================================
// K1 (ingestion, sketch.cpp:83-85 + attp.hpp:22): squared norm and
// finiteness of each row, one warp per row. VEC: 16-byte loads (rows 16-byte
// aligned, d even) with four independent accumulators so every lane keeps 4
// loads in flight; the per-row sum order is fixed (deterministic).
template <bool VEC>
__global__ void __launch_bounds__(256) k_ingest(const double* __restrict__ rows, int64_t n, int64_t ld, int d,
                                                double* __restrict__ nrm2, int* __restrict__ bad) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const double* a = rows + row * ld;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int nf = 0;
    if (VEC) {
        const double2* a2 = reinterpret_cast<const double2*>(a);
        const int d2 = d >> 1;
        int j = lane;
        for (; j + 96 < d2; j += 128) {
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(a2 + j + 32 * u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                nf |= !isfinite(v[u].x) | !isfinite(v[u].y);
                s[u] = fma(v[u].y, v[u].y, fma(v[u].x, v[u].x, s[u]));
            }
        }
        for (; j < d2; j += 32) {
            const double2 v = __ldcs(a2 + j);
            nf |= !isfinite(v.x) | !isfinite(v.y);
            s[0] = fma(v.y, v.y, fma(v.x, v.x, s[0]));
        }
    } else {
        for (int j = lane; j < d; j += 32) {
            const double v = a[j];
            nf |= !isfinite(v);
            s[0] = fma(v, v, s[0]);
        }
    }
    double t = warp_sum((s[0] + s[1]) + (s[2] + s[3]));
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) {
        nrm2[row] = t;
        bad[row] = nf;
    }
}
void ingest_rows(cudaStream_t st, const double* rows, int64_t n, int64_t ld, int d, double* nrm2,
                 int* bad) {
    if (n <= 0) return;
    const int wpb = 8;
    const bool vec = !(d & 1) && !(ld & 1) && !((uintptr_t)rows & 15);
    if (vec)
        k_ingest<true><<<(unsigned)((n + wpb - 1) / wpb), 32 * wpb, 0, st>>>(rows, n, ld, d, nrm2, bad);
    else
        k_ingest<false><<<(unsigned)((n + wpb - 1) / wpb), 32 * wpb, 0, st>>>(rows, n, ld, d, nrm2, bad);
    AERO_LAUNCHED();
}

// dst[q] = src[idx[q]] for n rows of d doubles (row-major, ld)
__global__ void k_gather_rows(const double* __restrict__ src, int64_t lds, const int64_t* __restrict__ idx,
                              int64_t n, int d, double* __restrict__ dst) {
    const int64_t q = blockIdx.x;
    if (q >= n) return;
    const double* s = src + idx[q] * lds;
    double* o = dst + q * (int64_t)d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) o[j] = s[j];
}
void gather_rows(cudaStream_t st, const double* src, int64_t lds, const int64_t* idx_d, int64_t n, int d,
                 double* dst) {
    if (n <= 0) return;
    k_gather_rows<<<(unsigned)n, 256, 0, st>>>(src, lds, idx_d, n, d, dst);
    AERO_LAUNCHED();
}

// ============================================================================
// CTA-wide cyclic Jacobi for small symmetric matrices in shared memory
// (round-robin parallel ordering; A, V column-major n x n, ld = n).
// On return diag(A) holds the eigenvalues (unsorted) and V the eigenvectors.
// ============================================================================
struct JacobiScratch {
    double* cs;  // >= jacobi_scratch_doubles(n) doubles
};
__device__ int g_jacobi_sweeps = 0;  // diagnostics: max sweeps used (1000 = cap hit)
__host__ __device__ constexpr int jacobi_scratch_doubles(int n) { return 6 * (n / 2 + 3); }
__device__ void cta_jacobi(double* A, double* V, int n, JacobiScratch sc) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < n * n; e += nt) V[e] = (e % (n + 1) == 0) ? 1.0 : 0.0;
    __syncthreads();
    if (n <= 1) return;
    const int np = n + (n & 1);  // players (dummy = n when odd)
    const int half = np / 2;
    double* crs = sc.cs;                                   // c, s, t per pair
    double* tolp = crs + 3 * half;                         // 1 double
    int* pidx = reinterpret_cast<int*>(tolp + 2);          // p, q per pair
    int* flag = pidx + 2 * half + 2;
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (tid == 0) {
            // absolute floor: rotations below ~eps*||A|| are rounding noise
            double sc_max = 0.0;
            for (int i = 0; i < n; ++i) sc_max = fmax(sc_max, fabs(A[i + i * n]));
            *tolp = 1.0e-16 * sc_max;
            *flag = 0;
        }
        __syncthreads();
        const double tol_abs = *tolp;
        for (int step = 0; step < np - 1; ++step) {
            // (a) disjoint pairs of this round-robin step and their rotations
            for (int i = tid; i < half; i += nt) {
                const int pi = (i == 0) ? 0 : ((i - 1 + step) % (np - 1)) + 1;
                const int qi = ((np - 1 - i - 1 + step) % (np - 1)) + 1;
                const int p = min(pi, qi), q = max(pi, qi);
                double c = 1.0, s = 0.0, t = 0.0;
                if (q < n) {
                    const double apq = A[p + q * n];
                    const double app = A[p + p * n], aqq = A[q + q * n];
                    if (fabs(apq) > 1e-300 && fabs(apq) > tol_abs &&
                        fabs(apq) > 2.220446049250313e-16 * sqrt(fabs(app)) * sqrt(fabs(aqq))) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        *flag = 1;
                    }
                }
                crs[3 * i] = c;
                crs[3 * i + 1] = s;
                crs[3 * i + 2] = t;
                pidx[2 * i] = p;
                pidx[2 * i + 1] = q;
            }
            __syncthreads();
            // (b) A <- R^T A R on the 2x2 blocks of pair pairs (diagonal blocks
            // updated exactly, GVL Alg. 8.4.2); V <- V R
            const int nblk = half * half;
            for (int bidx = tid; bidx < nblk + half * n; bidx += nt) {
                if (bidx < nblk) {
                    const int I = bidx % half, J = bidx / half;
                    const int p = pidx[2 * I], q = pidx[2 * I + 1];
                    const int pp = pidx[2 * J], qq = pidx[2 * J + 1];
                    const double cI = crs[3 * I], sI = crs[3 * I + 1];
                    const double cJ = crs[3 * J], sJ = crs[3 * J + 1];
                    const bool qin = q < n, qqin = qq < n;
                    if (I == J) {
                        if (sI != 0.0) {
                            const double tI = crs[3 * I + 2];
                            const double apq = A[p + q * n];
                            A[p + p * n] -= tI * apq;
                            A[q + q * n] += tI * apq;
                            A[p + q * n] = 0.0;
                            A[q + p * n] = 0.0;
                        }
                        continue;
                    }
                    if (sI == 0.0 && sJ == 0.0) continue;
                    const double b00 = A[p + pp * n];
                    const double b01 = qqin ? A[p + qq * n] : 0.0;
                    const double b10 = qin ? A[q + pp * n] : 0.0;
                    const double b11 = (qin && qqin) ? A[q + qq * n] : 0.0;
                    // left: rows (p,q) by R^T = [[c,-s],[s,c]]
                    const double l00 = cI * b00 - sI * b10, l01 = cI * b01 - sI * b11;
                    const double l10 = sI * b00 + cI * b10, l11 = sI * b01 + cI * b11;
                    // right: cols (pp,qq) by R = [[c,s],[-s,c]]
                    A[p + pp * n] = cJ * l00 - sJ * l01;
                    if (qqin) A[p + qq * n] = sJ * l00 + cJ * l01;
                    if (qin) A[q + pp * n] = cJ * l10 - sJ * l11;
                    if (qin && qqin) A[q + qq * n] = sJ * l10 + cJ * l11;
                } else {
                    // consecutive threads walk consecutive rows (conflict-free)
                    const int e = bidx - nblk;
                    const int row = e % n, I = e / n;
                    const int p = pidx[2 * I], q = pidx[2 * I + 1];
                    const double s = crs[3 * I + 1];
                    if (q >= n || s == 0.0) continue;
                    const double c = crs[3 * I];
                    const double vp = V[row + p * n], vq = V[row + q * n];
                    V[row + p * n] = c * vp - s * vq;
                    V[row + q * n] = s * vp + c * vq;
                }
            }
            __syncthreads();
        }
        if (*flag == 0) {
            if (tid == 0) atomicMax(&g_jacobi_sweeps, sweep + 1);
            break;
        }
        __syncthreads();
        if (sweep == 39 && tid == 0) atomicMax(&g_jacobi_sweeps, 1000);
    }
    __syncthreads();
}

// sort eigenpairs descending (stable rank sort) from (A diag, V) into (w, Vout)
// and fix eigenvector signs (largest-magnitude entry positive, first on ties)
__device__ void cta_sort_signfix(const double* A, const double* V, int n, double* w, double* Vout,
                                 int ldvo) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < n; i += nt) {
        const double li = A[i + i * n];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = A[j + j * n];
            rank += (lj > li) || (lj == li && j < i);
        }
        w[rank] = li;
        // sign fix of column i
        int at = 0;
        double best = -1.0;
        for (int r = 0; r < n; ++r) {
            const double v = fabs(V[r + i * n]);
            if (v > best) { best = v; at = r; }
        }
        const double sg = (V[at + i * n] < 0.0) ? -1.0 : 1.0;
        for (int r = 0; r < n; ++r) Vout[r + (int64_t)rank * ldvo] = sg * V[r + i * n];
    }
    __syncthreads();
}

__global__ void k_jacobi_batched(int n, double* A, int lda, int64_t stride, double* w) {
    extern __shared__ double sm[];
    double* sA = sm;
    double* sV = sA + n * n;
    double* cs = sV + n * n;
    double* Ab = A + blockIdx.x * stride;
    double* wb = w + blockIdx.x * (int64_t)n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e % n, j = e / n;
        sA[e] = 0.5 * (Ab[i + (int64_t)j * lda] + Ab[j + (int64_t)i * lda]);
    }
    __syncthreads();
    cta_jacobi(sA, sV, n, JacobiScratch{cs});
    cta_sort_signfix(sA, sV, n, wb, Ab, lda);
}

void eigh_small(cudaStream_t st, int n, double* A, int lda, double* w, int batch, int64_t stride) {
    const size_t smem = sizeof(double) * (2 * n * n + jacobi_scratch_doubles(n)) + 16;
    if (smem > 48 * 1024)
        AERO_CUDA(cudaFuncSetAttribute(k_jacobi_batched, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    k_jacobi_batched<<<batch, n >= 48 ? 512 : 256, smem, st>>>(n, A, lda, stride, w);
    AERO_LAUNCHED();
}

// ============================================================================
// batched power / subspace iteration engine (gate K2 + simul_iter K4)
// ============================================================================
__global__ void k_iter_init(const IterJob* __restrict__ jobs, const double* __restrict__ G, int ldg,
                            double* __restrict__ X, int ldx, int R, int* __restrict__ status,
                            const double* __restrict__ panel) {
    __shared__ double red[32];
    const IterJob jb = jobs[blockIdx.x];
    double tr = 0.0;
    for (int i = threadIdx.x; i < jb.r; i += blockDim.x) tr += G[i + (int64_t)i * ldg];
    tr = block_sum(tr, red);
    const bool zero = (tr == 0.0);
    if (threadIdx.x == 0) status[blockIdx.x] = zero ? JOB_ZERO : JOB_ACTIVE;
    double ss = 0.0;
    const double* pj = (panel && jb.panel >= 0) ? panel + jb.panel : nullptr;
    for (int j = 0; j < jb.k; ++j) {
        double* x = X + (int64_t)(jb.col + j) * ldx;
        for (int i = threadIdx.x; i < R; i += blockDim.x) {
            double v = 0.0;
            // Pi is r x k row-major in draw order (linalg.cpp:141, gaussian_matrix)
            if (i < jb.r && !zero)
                v = pj ? pj[(int64_t)i * jb.k + j] : rng_gaussian_at(jb.rng0, (uint64_t)i * jb.k + j);
            x[i] = v;
            ss = fma(v, v, ss);
        }
    }
    if (jb.type == 0 && !zero) {  // gate: x.normalize() (linalg.cpp:108)
        ss = block_sum(ss, red);
        const double nrm = sqrt(ss);
        double* x = X + (int64_t)jb.col * ldx;
        if (nrm > 0.0)
            for (int i = threadIdx.x; i < jb.r; i += blockDim.x) x[i] = x[i] / nrm;
    }
}
void iter_init(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg,
               double* X, int ldx, int R, int* status, const double* panel) {
    if (njobs <= 0) return;
    k_iter_init<<<njobs, 256, 0, st>>>(jobs, G, ldg, X, ldx, R, status, panel);
    AERO_LAUNCHED();
}

// k x k Gram of two column blocks P (r x k) and Q (r x k), ld, into S (smem, col-major)
template <int KM>
__device__ void cta_gram(const double* P, int ldp, const double* Q, int ldq, int r, int k,
                         double* S, double* red) {
    const int ld = ldp;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int E = k * k;
    if (KM <= 4) {
        // register partials (k <= KM <= 4, compile-time indexed), warp + CTA sums
        double part[KM * KM];
#pragma unroll
        for (int e = 0; e < KM * KM; ++e) part[e] = 0.0;
        // RU rows per thread per round: all their loads in flight before the
        // FMAs (one L2 round trip per round instead of one per row)
        constexpr int RU = (KM <= 16) ? 16 / KM : 1;
        for (int i0 = tid; i0 < r; i0 += RU * nt) {
            double p[RU][KM], q[RU][KM];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int i = i0 + u * nt;
#pragma unroll
                for (int a = 0; a < KM; ++a) {
                    p[u][a] = (i < r && a < k) ? P[i + (int64_t)a * ldp] : 0.0;
                    q[u][a] = (i < r && a < k) ? Q[i + (int64_t)a * ldq] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < RU; ++u)
#pragma unroll
                for (int a = 0; a < KM; ++a)
#pragma unroll
                    for (int b = 0; b < KM; ++b) part[a + b * KM] = fma(p[u][a], q[u][b], part[a + b * KM]);
        }
        const int lane = tid & 31, wid = tid >> 5, nw = (nt + 31) >> 5;
#pragma unroll
        for (int e = 0; e < KM * KM; ++e) {
            const double v = warp_sum(part[e]);
            if (lane == 0) red[wid * 16 + e] = v;
        }
        __syncthreads();
        for (int e = tid; e < E; e += nt) {
            const int a = e % k, b = e / k;
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[w * 16 + a + b * KM];
            S[e] = t;
        }
        __syncthreads();
    } else {
        // one thread per entry, rows streamed (k up to 64; rare path)
        for (int e = tid; e < E; e += nt) {
            const int a = e % k, b = e / k;
            double t = 0.0;
            for (int i = 0; i < r; ++i) t = fma(P[i + (int64_t)a * ld], Q[i + (int64_t)b * ldq], t);
            S[e] = t;
        }
        __syncthreads();
    }
}

// eigendecomposition of a k x k symmetric W (shared memory) -> diag(W), T:
// closed-form 2x2 Jacobi rotation (GVL Alg. 8.4.1) for k <= 2, CTA Jacobi else
__device__ void small_eig(double* W, double* T, int k, double* cs) {
    if (k > 2) {
        cta_jacobi(W, T, k, JacobiScratch{cs});
        return;
    }
    if (threadIdx.x == 0) {
        if (k == 1) {
            T[0] = 1.0;
        } else {
            const double a = W[0], b = W[2], c = W[3];
            double cn = 1.0, sn = 0.0, t = 0.0;
            if (fabs(b) > 1e-300) {
                const double tau = (c - a) / (2.0 * b);
                t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                cn = 1.0 / sqrt(1.0 + t * t);
                sn = t * cn;
            }
            W[0] = a - t * b;
            W[3] = c + t * b;
            W[1] = W[2] = 0.0;
            T[0] = cn;
            T[1] = -sn;
            T[2] = sn;
            T[3] = cn;
        }
    }
    __syncthreads();
}

// WS: Y arrives as `splits` split-K partials in ws (ws[z*sstride + i + c*wsM]),
// summed here in fixed order into shared memory (fuses k_product_reduce)
template <int KM>
__host__ __device__ constexpr size_t normalize_smem_doubles(int R, bool ws) {
    // ws: the job's r x k product, reused as the padded staging of the new iterate (8 r8p <= r + 16 per column)
    return 32 * 16 + 3 * KM * KM + KM + jacobi_scratch_doubles(KM) + (ws ? (size_t)(R + 16) * KM : 0);
}

// one job's normalization after product phase `phase` (body of k_iter_normalize;
// also run inside the persistent k_iterate); sm: normalize_smem_doubles
// dev instrumentation (AERO_I8_PROF): CTA-0 ns per normalization step
__device__ unsigned long long* g_norm_prof = nullptr;
#define NJ_MARK(i)                                                                 \
    if (g_norm_prof && blockIdx.x == 0 && threadIdx.x == 0) {                      \
        unsigned long long t_;                                                     \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
        g_norm_prof[i] += t_ - nj_t;                                               \
        nj_t = t_;                                                                 \
    }

template <int KM, bool WS>
__device__ void normalize_job(const IterJob& jb, int jidx, int phase, double* X,
                              const double* __restrict__ Y, int ldx, double* H,
                              int* __restrict__ status, double* __restrict__ out_sig,
                              double* __restrict__ out_vr, int kv, int* __restrict__ out_clamped,
                              const double* __restrict__ ws, int wsM, int64_t sstride, int splits,
                              double* sm, const OzSliceDst xs = OzSliceDst{}, const OzBulkWs bw = OzBulkWs{},
                              unsigned* bw_use = nullptr) {
    if (phase >= jb.nphase) return;
    const int st = status[jidx];
    const bool last = (phase == jb.nphase - 1);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int r = jb.r, k = jb.k;
    double* x = X + (int64_t)jb.col * ldx;
    double* red = sm;                  // 32*16
    double* S = red + 32 * 16;         // KM*KM
    double* W = S + KM * KM;           // KM*KM
    double* T = W + KM * KM;           // KM*KM
    double* lam = T + KM * KM;         // KM
    double* cs = lam + KM;             // jacobi scratch
    double* ysh = cs + jacobi_scratch_doubles(KM);  // WS: r * k
    unsigned long long nj_t = 0;
    if (g_norm_prof && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(nj_t));
    auto inactive = [&]() {
        if (last && tid == 0) {
            if (jb.type == 0) out_sig[jb.col] = 0.0;
            else
                for (int a = 0; a < k; ++a) out_sig[jb.col + a] = 0.0;
        }
    };
    // WS: the split-K loads are issued before the status is known (the sum
    // is harmless for an inactive job), so the status round trip overlaps them
    if (!WS && st != JOB_ACTIVE) {
        inactive();
        return;
    }
    const double* y;
    int ldy;
    if (WS) {
        const int tot = r * k;
        const int re = (r + 1) & ~1;  // 16-byte multiple per column copy
        const bool bulk = bw.buf && (size_t)splits * k * re <= bw.cap && !(wsM & 1) && !(sstride & 1);
        if (bulk) {
            // the job's split-K partials (k columns x splits) pulled into shared
            // memory by bulk copies (async proxy: all in flight at once, no
            // per-thread load queue), then summed in the same fixed order
            if (tid == 0) {
                mbar_expect_tx(bw.bar, (unsigned)(splits * k * re) * 8u);
                for (int z = 0; z < splits; ++z)
                    for (int a = 0; a < k; ++a)
                        bulk_g2s(smem_u32(bw.buf + (size_t)(z * k + a) * re),
                                 ws + z * sstride + (int64_t)(jb.col + a) * wsM, (unsigned)re * 8u, bw.bar);
            }
            mbar_wait(bw.bar, *bw_use & 1u);
            ++*bw_use;
            if (st == JOB_ACTIVE)
                for (int a = 0; a < k; ++a)
                    for (int i = tid; i < r; i += nt) {
                        double v = 0.0;
                        for (int z = 0; z < splits; z += 4) {
                            double t[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                t[q] = (z + q < splits) ? bw.buf[(size_t)((z + q) * k + a) * re + i] : 0.0;
                            v += (t[0] + t[1]) + (t[2] + t[3]);
                        }
                        ysh[i + a * r] = v;
                    }
        } else {
        // fixed-order split-K sum; 8 entries x 4 splits of loads in flight per
        // thread (a plain per-entry loop serializes one L2 round trip per split)
        constexpr int U = 8;
        for (int e0 = tid; e0 < tot; e0 += U * nt) {
            const double* pp[U];
            bool ok[U];
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * nt;
                ok[u] = e < tot;
                const int ee = ok[u] ? e : 0;
                pp[u] = ws + ee % r + (int64_t)(jb.col + ee / r) * wsM;
                v[u] = 0.0;
            }
            for (int z = 0; z < splits; z += 4) {
                double t[U][4];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < 4; ++q) t[u][q] = (ok[u] && z + q < splits) ? __ldcg(pp[u] + (z + q) * sstride) : 0.0;
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] += (t[u][0] + t[u][1]) + (t[u][2] + t[u][3]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (ok[u]) ysh[e0 + u * nt] = v[u];
        }
        }
        __syncthreads();
        NJ_MARK(0);
        if (st != JOB_ACTIVE) {
            inactive();
            return;
        }
        y = ysh;
        ldy = r;
    } else {
        y = Y + (int64_t)jb.col * ldx;
        ldy = ldx;
    }
    if (jb.type == 0) {
        if (!last) {
            double s = 0.0, mx = 0.0;
            for (int i = tid; i < r; i += nt) {
                const double v = y[i];
                s = fma(v, v, s);
                mx = fmax(mx, fabs(v));
            }
            if (xs.b) {  // max |y| for the slicing scale (max |x| = fl(max|y| / nrm))
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if ((tid & 31) == 0) red[64 + (tid >> 5)] = mx;
            }
            s = block_sum(s, red);
            const double nrm = sqrt(s);
            if (nrm < 1e-300) {  // linalg.cpp:112-116
                if (tid == 0) status[jidx] = JOB_DEAD;
                return;
            }
            int e = 0;
            if (xs.b) {
                mx = 0.0;
                for (int w = 0; w < (nt + 31) / 32; ++w) mx = fmax(mx, red[64 + w]);
                const double xm = mx / nrm;
                e = (xm > 0.0) ? ilogb(xm) + 1 : 0;
                if (tid == 0) xs.fe[jb.col] = e;
            }
            for (int i = tid; i < r; i += nt) x[i] = y[i] / nrm;
            if (xs.b) {  // 8 consecutive entries per thread: one 8-byte store per slice
                const int nkb = xs.Kp / kOzBK, tt = jb.col / kOzBN, rr = jb.col % kOzBN;
                for (int k0 = 8 * tid; k0 < r; k0 += 8 * nt) {
                    double xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) xv[u] = (k0 + u < r) ? y[k0 + u] / nrm : 0.0;
                    uint64_t pk[kOzSlices];
                    ozaki_slice8_pow2<kOzSlices>(xv, e, pk);
                    int8_t* blk = xs.b + ((int64_t)tt * nkb + k0 / kOzBK) * kOzSlices * kOzBN * kOzBK + rr * kOzBK +
                                  ((((k0 % kOzBK) >> 4) ^ ((rr >> 1) & 3)) << 4) + (k0 & 15);
#pragma unroll
                    for (int q = 0; q < kOzSlices; ++q)
                        *reinterpret_cast<uint64_t*>(blk + q * kOzBN * kOzBK) = pk[q];
                }
            }
        } else {
            double s = 0.0;  // sigma1^2 = ||A x||^2 = x^T G x (linalg.cpp:119)
            for (int i = tid; i < r; i += nt) s = fma(x[i], y[i], s);
            s = block_sum(s, red);
            if (tid == 0) out_sig[jb.col] = s;
        }
        return;
    }
    // simul: S = X^T Y (Gram of g = C'^T X), T = S^{-1/2}
    double tq[KM * KM];  // T (scaled), in registers for the update below
    bool fast = false;
    if constexpr (KM == 2) fast = !last;
    if (fast) {
        // k <= 2, not the last phase: the 2x2 Gram reduced once, then every
        // thread evaluates the closed-form eig and the clamp redundantly
        // (the same operations thread 0 runs on the general path: same bits),
        // no serial section and one barrier instead of five
        double part[4] = {0.0, 0.0, 0.0, 0.0};
        constexpr int RUG = 8;
        for (int i0 = tid; i0 < r; i0 += RUG * nt) {
            double p[RUG][2], q[RUG][2];
#pragma unroll
            for (int u = 0; u < RUG; ++u) {
                const int i = i0 + u * nt;
#pragma unroll
                for (int a2 = 0; a2 < 2; ++a2) {
                    p[u][a2] = (i < r && a2 < k) ? x[i + (int64_t)a2 * ldx] : 0.0;
                    q[u][a2] = (i < r && a2 < k) ? y[i + (int64_t)a2 * ldy] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < RUG; ++u)
#pragma unroll
                for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
                    for (int b2 = 0; b2 < 2; ++b2) part[a2 + b2 * 2] = fma(p[u][a2], q[u][b2], part[a2 + b2 * 2]);
        }
        const int lane = tid & 31, wid = tid >> 5, nw = (nt + 31) >> 5;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double v = warp_sum(part[e]);
            if (lane == 0) red[wid * 16 + e] = v;
        }
        __syncthreads();
        double s[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[w * 16 + e];
            s[e] = t;
        }
        NJ_MARK(1);
        double w0, w3, t00, t10, t01, t11;
        if (k == 1) {
            w0 = s[0];
            w3 = 0.0;
            t00 = 1.0;
            t10 = t01 = t11 = 0.0;
        } else {  // small_eig's closed-form 2x2 Jacobi rotation on W = sym(S)
            const double a = 0.5 * (s[0] + s[0]), b = 0.5 * (s[2] + s[1]), cc = 0.5 * (s[3] + s[3]);
            double cn = 1.0, sn = 0.0, t = 0.0;
            if (fabs(b) > 1e-300) {
                const double tau = (cc - a) / (2.0 * b);
                t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                cn = 1.0 / sqrt(1.0 + t * t);
                sn = t * cn;
            }
            w0 = a - t * b;
            w3 = cc + t * b;
            t00 = cn;
            t10 = -sn;
            t01 = sn;
            t11 = cn;
        }
        const double lmax = (k == 1) ? fmax(0.0, w0) : fmax(fmax(0.0, w0), w3);
        const bool ok0 = w0 > 0.0 && w0 > 1e-14 * lmax;
        const double l0 = ok0 ? 1.0 / sqrt(w0) : 0.0;
        double l1 = 0.0;
        if (k == 2) {
            const bool ok1 = w3 > 0.0 && w3 > 1e-14 * lmax;
            l1 = ok1 ? 1.0 / sqrt(w3) : 0.0;
        }
        // T[e] *= lam[e / k]: column b scaled by lam_b
        tq[0] = t00 * l0;
        tq[1] = t10 * l0;
        tq[2] = t01 * l1;
        tq[3] = t11 * l1;
        NJ_MARK(2);
    } else {
    cta_gram<KM>(x, ldx, y, ldy, r, k, S, red);
    NJ_MARK(1);
    for (int e = tid; e < k * k; e += nt) {
        const int a = e % k, b = e / k;
        W[e] = 0.5 * (S[a + b * k] + S[b + a * k]);
    }
    __syncthreads();
    small_eig(W, T, k, cs);  // W -> diag, T -> eigvecs
    // lam_i and T columns scaled by lam^{-1/2} with clamp
    if (tid == 0) {
        double lmax = 0.0;
        for (int i = 0; i < k; ++i) lmax = fmax(lmax, W[i + i * k]);
        int nclamp = 0;
        for (int i = 0; i < k; ++i) {
            const double l = W[i + i * k];
            const bool ok = l > 0.0 && l > 1e-14 * lmax;
            lam[i] = ok ? 1.0 / sqrt(l) : 0.0;
            nclamp += !ok;
        }
        if (last && out_clamped) out_clamped[jidx] = nclamp;
    }
    __syncthreads();
    for (int e = tid; e < k * k; e += nt) T[e] *= lam[e / k];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < KM * KM; ++e) tq[e] = (e < k * k) ? T[e] : 0.0;
    NJ_MARK(2);
    }
    // rows independent: [last: H = X T], X <- Y T; RU rows per thread per
    // round with all their loads issued first (one L2 round trip per round).
    // With xs (not last): the new columns are also sliced for the next product
    // -- from registers when the job fits one round, else reloaded below.
    {
        constexpr int RU = (KM <= 4) ? 16 / KM : 1;
        const bool slice_regs = xs.b && !last && r <= RU * nt;
        double hv[RU][KM], mxb[KM];
#pragma unroll
        for (int b = 0; b < KM; ++b) mxb[b] = 0.0;
        for (int i0 = tid; i0 < r; i0 += RU * nt) {
            double xr[RU][KM], yr[RU][KM];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int i = i0 + u * nt;
#pragma unroll
                for (int a = 0; a < KM; ++a) {
                    if (a < k && i < r) {
                        xr[u][a] = last ? x[i + (int64_t)a * ldx] : 0.0;  // H = X T only in the last phase
                        yr[u][a] = y[i + (int64_t)a * ldy];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int i = i0 + u * nt;
                if (i >= r) break;
#pragma unroll
                for (int b = 0; b < KM; ++b) {
                    if (b >= k) break;
                    double hx = 0.0, hy = 0.0;
#pragma unroll
                    for (int a = 0; a < KM; ++a) {
                        if (a < k) {
                            hx = fma(xr[u][a], tq[a + b * k], hx);
                            hy = fma(yr[u][a], tq[a + b * k], hy);
                        }
                    }
                    if (last) H[i + (int64_t)(jb.col + b) * ldx] = hx;
                    x[i + (int64_t)b * ldx] = hy;
                    hv[u][b] = hy;
                    mxb[b] = fmax(mxb[b], fabs(hy));
                }
            }
        }
        NJ_MARK(3);
        if (slice_regs) {
#pragma unroll
            for (int b = 0; b < KM; ++b) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mxb[b] = fmax(mxb[b], __shfl_xor_sync(0xffffffffu, mxb[b], o));
                if ((tid & 31) == 0) red[64 + b * 32 + (tid >> 5)] = mxb[b];
            }
            __syncthreads();
            // stage the new iterate in shared memory (ysh is free: every thread
            // is past the update loop), then slice 8 consecutive entries per
            // thread into one 8-byte store per slice (was one byte store per
            // slice and entry)
            // (entry i at (i & 7) * r8p + (i >> 3), r8p odd: the 8 consecutive
            // entries a thread slices sit r8p apart, so a warp's reads are
            // consecutive words instead of 64-byte strides -- no bank conflicts)
            const int r8p = ((r + 7) >> 3) | 1;
            int eb[KM];
#pragma unroll
            for (int b = 0; b < KM; ++b) {
                if (b >= k) break;
                double m = 0.0;
                for (int w = 0; w < (nt + 31) / 32; ++w) m = fmax(m, red[64 + b * 32 + w]);
                eb[b] = (m > 0.0) ? ilogb(m) + 1 : 0;
                if (tid == 0) xs.fe[jb.col + b] = eb[b];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const int i = tid + u * nt;
                    if (i < r) ysh[(i & 7) * r8p + (i >> 3) + b * 8 * r8p] = hv[u][b];
                }
            }
            __syncthreads();
            const int nkb = xs.Kp / kOzBK;
#pragma unroll
            for (int b = 0; b < KM; ++b) {
                if (b >= k) break;
                const int cidx = jb.col + b, tt = cidx / kOzBN, rr = cidx % kOzBN;
                for (int k0 = 8 * tid; k0 < r; k0 += 8 * nt) {
                    double xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        xv[u] = (k0 + u < r) ? ysh[u * r8p + (k0 >> 3) + b * 8 * r8p] : 0.0;
                    uint64_t pk[kOzSlices];
                    ozaki_slice8_pow2<kOzSlices>(xv, eb[b], pk);
                    int8_t* blk = xs.b + ((int64_t)tt * nkb + k0 / kOzBK) * kOzSlices * kOzBN * kOzBK + rr * kOzBK +
                                  ((((k0 % kOzBK) >> 4) ^ ((rr >> 1) & 3)) << 4) + (k0 & 15);
#pragma unroll
                    for (int q = 0; q < kOzSlices; ++q)
                        *reinterpret_cast<uint64_t*>(blk + q * kOzBN * kOzBK) = pk[q];
                }
            }
        } else if (xs.b && !last) {
            __syncthreads();
            for (int b = 0; b < k; ++b)
                ozaki_slice_vector<kOzSlices, kOzBN>(x + (int64_t)b * ldx, r, xs.Kp, jb.col + b, xs.b, xs.fe,
                                                     red + 64);
        }
        NJ_MARK(4);
    }
    __syncthreads();
    if (!last) return;
    // Ritz values: eig(w^T w), w = C' g = G H = X (linalg.cpp:145-150)
    cta_gram<KM>(x, ldx, x, ldx, r, k, S, red);
    for (int e = tid; e < k * k; e += nt) {
        const int a = e % k, b = e / k;
        W[e] = 0.5 * (S[a + b * k] + S[b + a * k]);
    }
    __syncthreads();
    small_eig(W, T, k, cs);
    double* vr = out_vr + (int64_t)jb.col * kv;
    cta_sort_signfix(W, T, k, lam, vr, k);
    for (int a = tid; a < k; a += nt) out_sig[jb.col + a] = sqrt(fmax(lam[a], 0.0));
}

template <int KM, bool WS>
__global__ void k_iter_normalize(const IterJob* __restrict__ jobs, int phase, double* X,
                                 const double* __restrict__ Y, int ldx, double* H,
                                 int* __restrict__ status, double* __restrict__ out_sig,
                                 double* __restrict__ out_vr, int kv, int* __restrict__ out_clamped,
                                 const double* __restrict__ ws, int wsM, int64_t sstride,
                                 int splits) {
    extern __shared__ double sm[];
    const IterJob jb = jobs[blockIdx.x];
    normalize_job<KM, WS>(jb, blockIdx.x, phase, X, Y, ldx, H, status, out_sig, out_vr, kv, out_clamped, ws,
                          wsM, sstride, splits, sm);
}

template <int KM, bool WS>
static void launch_normalize(cudaStream_t st, const IterJob* jobs, int njobs, int phase, double* X,
                             const double* Y, int ldx, double* H, int* status, double* out_sig,
                             double* out_vr, int kv, int* out_clamped, const double* ws, int wsM,
                             int64_t sstride, int splits) {
    const size_t smem = sizeof(double) * normalize_smem_doubles<KM>(wsM, WS) + 16;
    if (smem > 48 * 1024)
        AERO_CUDA(cudaFuncSetAttribute(k_iter_normalize<KM, WS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_iter_normalize<KM, WS><<<njobs, 256, smem, st>>>(jobs, phase, X, Y, ldx, H, status, out_sig,
                                                       out_vr, kv, out_clamped, ws, wsM, sstride,
                                                       splits);
    AERO_LAUNCHED();
}

// ---- persistent iteration: every phase of a batch in ONE cooperative launch --
// phase p: [all CTAs] split-K partial products Y_z = G[:, Kz] X[Kz, :] as DMMA
// tiles -> grid barrier -> [CTA per job] fixed-order partial sum + normalize ->
// grid barrier. Replaces (product + reduce + normalize) launches per phase.
struct IterPersistArgs {
    const IterJob* jobs;
    int njobs, maxphase, R, ldg, ldx, kv;
    const double* G;
    double *X, *H, *out_sig, *out_vr, *ws;
    int *status, *out_clamped;
    const int* phase_ncol;    // active columns per phase
    const int* phase_splits;  // split-K factor per phase
    unsigned* bar;
};

template <int KM>
__global__ void __launch_bounds__(tiles::PNT, 2) k_iterate(IterPersistArgs a) {
    using namespace tiles;
    extern __shared__ __align__(16) double smd[];
    unsigned epoch = 0;
    const unsigned G = gridDim.x;
    const int R = a.R;
    const int kt_total = (R + PBK - 1) / PBK;
    for (int p = 0; p < a.maxphase; ++p) {
        const int ncol = a.phase_ncol[p], splits = a.phase_splits[p];
        const int tn = (ncol + PBN - 1) / PBN, tmn = (R + PBM - 1) / PBM;
        const int kchunk = ((kt_total + splits - 1) / splits) * PBK;
        const int items = tn * tmn * splits;
        const int64_t sstride = (int64_t)R * ncol;
        for (int it = blockIdx.x; it < items; it += G) {
            const int tz = it / (tn * tmn), rem = it % (tn * tmn);
            mma_tile<false, false>(rem % tn, rem / tn, tz, R, ncol, R, kchunk, a.G, a.ldg, a.X, a.ldx, a.ws, R,
                                   sstride, nullptr, 0, 1.0, 0.0, smd);
            __syncthreads();
        }
        grid_sync(a.bar, epoch, G);
        for (int j = blockIdx.x; j < a.njobs; j += G) {
            const IterJob jb = a.jobs[j];
            normalize_job<KM, true>(jb, j, p, a.X, nullptr, a.ldx, a.H, a.status, a.out_sig, a.out_vr, a.kv,
                                    a.out_clamped, a.ws, R, sstride, splits, smd);
            __syncthreads();
        }
        grid_sync(a.bar, epoch, G);
    }
}

// ---- persistent iteration with the products on the int8 tensor cores -------
// phase p: [all CTAs] (tile, split) work items of Y = G X (ozaki_tile, TMEM
// allocated once per CTA) -> grid barrier -> [CTA per job] fixed-order split-K
// sum + normalize, then the new iterate columns are sliced for the next
// product -> grid barrier. Same arithmetic as the per-phase launch sequence
// (OzakiGram::product + iter_normalize).
struct IterI8Args {
    const IterJob* jobs;
    int njobs, maxphase, R, ldx, kv, Kp, Rp;
    double *X, *H, *out_sig, *out_vr, *ws;
    int *status, *out_clamped;
    const int* colmask;
    const int* phase_ncol;
    const int* phase_splits;
    unsigned* bar;
    const int8_t* ga;
    const int* gea;
    int8_t* xb;
    int* xfe;
    unsigned long long* prof;  // optional (AERO_I8_PROF): CTA 0 ns per segment
    int smem_bytes;            // dynamic shared memory of the launch
    int bulk_ws;               // split-K partials by bulk copy into shared memory (A/B: AERO_BULK_WS=0)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int KM>
__global__ void __launch_bounds__(256, 1) k_iterate_i8(IterI8Args a) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    double* smd = reinterpret_cast<double*>(sm);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t wsbar;  // split-K partials landed in shared memory (normalize_job)
    constexpr int S = kOzSlices;
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&slot)),
                     "r"(OzCfg<S>::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    if (threadIdx.x == 0) {
        mbar_init(&wsbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = slot;
    unsigned epoch = 0;
    const unsigned G = gridDim.x;
    const int R = a.R, nkb_all = a.Kp / kOzBK, tm = a.Rp / kOzBM;
    const int Rld = (R + 1) & ~1;  // partial columns start 16-byte aligned (bulk copies)
    // shared memory past the normalization scratch receives a job's partials
    const size_t nd = (normalize_smem_doubles<KM>(R, true) + 1) & ~(size_t)1;
    const size_t smd_total = ((size_t)a.smem_bytes - (size_t)(sm - smraw)) / sizeof(double);
    const OzBulkWs bw{a.bulk_ws && smd_total > nd ? smd + nd : nullptr, &wsbar, smd_total > nd ? smd_total - nd : 0};
    unsigned bw_use = 0;
    {  // X slices for phase 0
        const int ncol0 = a.phase_ncol[0], np0 = (ncol0 + kOzBN - 1) / kOzBN * kOzBN;
        for (int c = blockIdx.x; c < np0; c += G) {
            const int lim = (c < ncol0) ? min(a.colmask[c], R) : 0;
            ozaki_slice_vector<S, kOzBN>(a.X + (int64_t)c * a.ldx, lim, a.Kp, c, a.xb, a.xfe, smd);
            __syncthreads();
        }
    }
    grid_sync_async(a.bar, epoch, G);
    // this CTA's first job, read once (jobs are fixed for the whole launch)
    const IterJob jb0 = ((int)blockIdx.x < a.njobs) ? a.jobs[blockIdx.x] : IterJob{};
    const bool pr = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
    unsigned long long tp = pr ? gtimer() : 0;
#define I8_MARK(i)                              \
    if (pr) {                                   \
        const unsigned long long t_ = gtimer(); \
        a.prof[i] += t_ - tp;                   \
        tp = t_;                                \
    }
    for (int p = 0; p < a.maxphase; ++p) {
        // phase_splits[p] = split-K factor | effective slices << 16 (0: all S)
        const int ncol = a.phase_ncol[p], splits = a.phase_splits[p] & 0xffff, se = a.phase_splits[p] >> 16;
        const int tn = (ncol + kOzBN - 1) / kOzBN, per = (nkb_all + splits - 1) / splits;
        const int items = tn * tm * splits;
        const int64_t sstride = (int64_t)Rld * ncol;
        for (int it = blockIdx.x; it < items; it += G) {
            const int z = it / (tn * tm), rem = it % (tn * tm);
            const int kb0 = z * per, nkb = max(0, min(nkb_all - kb0, per));
            if (se == S - 1)
                ozaki_tile<S, S - 1>(R, ncol, nkb_all, rem / tn, rem % tn, kb0, nkb, a.ga, a.xb, a.gea, a.xfe,
                                     a.ws + z * sstride, Rld, nullptr, 0, sm, tmem);
            else
                ozaki_tile<S>(R, ncol, nkb_all, rem / tn, rem % tn, kb0, nkb, a.ga, a.xb, a.gea, a.xfe,
                              a.ws + z * sstride, Rld, nullptr, 0, sm, tmem);
        }
        I8_MARK(0);
        grid_sync_async(a.bar, epoch, G);
        I8_MARK(1);
        for (int j = blockIdx.x; j < a.njobs; j += G) {
            const IterJob jb = (j == (int)blockIdx.x) ? jb0 : a.jobs[j];
            __syncthreads();
            // the normalization also slices the new iterate for the next product
            normalize_job<KM, true>(jb, j, p, a.X, nullptr, a.ldx, a.H, a.status, a.out_sig, a.out_vr, a.kv,
                                    a.out_clamped, a.ws, Rld, sstride, splits, smd, OzSliceDst{a.xb, a.xfe, a.Kp},
                                    bw, &bw_use);
            __syncthreads();
            if (j == 0) I8_MARK(4);
        }
        I8_MARK(2);
        grid_sync_async(a.bar, epoch, G);
        I8_MARK(3);
    }
#undef I8_MARK
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "r"(OzCfg<S>::TMEM_COLS));
    }
}

int ozaki_splits(const OzakiGram& oz, int N, size_t ws_doubles) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        AERO_CUDA(cudaGetDevice(&dev));
        AERO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int tm = oz.Rp / kOzBM, tn = (N + kOzBN - 1) / kOzBN, nkb = oz.Kp / kOzBK;
    int splits = std::max(1, std::min(sms / std::max(tm * tn, 1), nkb / 2));
    static const int max_splits = getenv("AERO_OZ_MAXSPLIT") ? std::max(1, atoi(getenv("AERO_OZ_MAXSPLIT"))) : 1 << 20;
    splits = std::min(splits, max_splits);  // dev knob: fewer splits = less partial traffic, fewer busy CTAs
    while (splits > 1 && (size_t)splits * (oz.R + 1) * N > ws_doubles) --splits;  // padded leading dimension
    const int per = (nkb + splits - 1) / splits;
    return (nkb + per - 1) / per;
}

void iterate_i8_persistent(cudaStream_t st, const IterJob* jobs, int njobs, int maxphase, int R, const OzakiGram& oz,
                           const int* colmask, double* X, int ldx, double* H, int* status, double* out_sig,
                           double* out_vr, int kv, int* out_clamped, double* ws, const int* phase_ncol,
                           const int* phase_splits, unsigned* bar, int max_k, int grid) {
    // the tile pipeline's stages or the normalization's scratch (phases are separate in time)
    // + room for one job's split-K partials (4 splits x max_k columns) when it fits
    const size_t scratch = sizeof(double) * normalize_smem_doubles<4>(R, true) + 1024 + 16;
    const size_t partials = sizeof(double) * 4 * (size_t)std::max(max_k, 2) * (size_t)(R + 2);
    const size_t smem = std::max({(size_t)OzCfg<kOzSlices>::SMEM, scratch,
                                  std::min(scratch + partials, (size_t)227 * 1024 - 4096)});
    static const int bulk_ws = getenv("AERO_BULK_WS") ? atoi(getenv("AERO_BULK_WS")) : 1;
    static size_t attr = 0;
    if (attr < smem) {
        AERO_CUDA(cudaFuncSetAttribute(k_iterate_i8<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AERO_CUDA(cudaFuncSetAttribute(k_iterate_i8<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    AERO_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), st));
    // dev instrumentation (AERO_I8_PROF): CTA-0 ns per segment, printed every 256 launches
    static unsigned long long* prof = nullptr;
    static unsigned long long phases = 0, calls = 0;
    static const bool want = getenv("AERO_I8_PROF") != nullptr;
    static unsigned long long* nprof = nullptr;
    if (want && !prof) {
        AERO_CUDA(cudaMalloc(&prof, 8 * sizeof(unsigned long long)));
        AERO_CUDA(cudaMemset(prof, 0, 8 * sizeof(unsigned long long)));
        AERO_CUDA(cudaMalloc(&nprof, 8 * sizeof(unsigned long long)));
        AERO_CUDA(cudaMemset(nprof, 0, 8 * sizeof(unsigned long long)));
        AERO_CUDA(cudaMemcpyToSymbol(g_norm_prof, &nprof, sizeof(nprof)));
    }
    if (prof && ++calls % 256 == 0) {
        unsigned long long h[8];
        AERO_CUDA(cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost));
        fprintf(stderr, "k_iterate_i8 CTA0 us/phase: tiles %.2f bar1 %.2f normalize %.2f slice %.2f bar2 %.2f (%llu phases)\n",
                h[0] / 1e3 / phases, h[1] / 1e3 / phases, h[4] / 1e3 / phases, h[2] / 1e3 / phases,
                h[3] / 1e3 / phases, phases);
        AERO_CUDA(cudaMemcpy(h, nprof, sizeof(h), cudaMemcpyDeviceToHost));
        fprintf(stderr, "  normalize CTA0 us/phase: ws-sum %.2f gram %.2f eig %.2f update %.2f slice %.2f\n",
                h[0] / 1e3 / phases, h[1] / 1e3 / phases, h[2] / 1e3 / phases, h[3] / 1e3 / phases,
                h[4] / 1e3 / phases);
    }
    phases += (unsigned long long)maxphase;
    IterI8Args a{jobs, njobs, maxphase, R, ldx, kv, oz.Kp, oz.Rp, X, H, out_sig, out_vr, ws, status, out_clamped,
                 colmask, phase_ncol, phase_splits, bar, oz.a, oz.ea, oz.b, oz.fb, prof, (int)smem, bulk_ws};
    void* args[] = {&a};
    note_launch();
    AERO_CUDA(cudaLaunchCooperativeKernel(max_k <= 2 ? (void*)k_iterate_i8<2> : (void*)k_iterate_i8<4>, dim3(grid),
                                          dim3(256), args, smem, st));
}

size_t iterate_smem_bytes(int R) {
    return std::max(tiles::MMA_SMEM, sizeof(double) * normalize_smem_doubles<4>(R, true)) + 16;
}

int iterate_grid(int R) {
    static int grid[2] = {0, 0};
    static int ok_r = -1;
    if (ok_r != R) {
        int dev = 0, sms = 0, per2 = 0, per4 = 0;
        AERO_CUDA(cudaGetDevice(&dev));
        AERO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const size_t smem = iterate_smem_bytes(R);
        AERO_CUDA(cudaFuncSetAttribute(k_iterate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AERO_CUDA(cudaFuncSetAttribute(k_iterate<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AERO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_iterate<2>, tiles::PNT, smem));
        AERO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per4, k_iterate<4>, tiles::PNT, smem));
        grid[0] = sms * std::min(per2, 2);
        grid[1] = sms * std::min(per4, 2);
        ok_r = R;
    }
    return std::min(grid[0], grid[1]);
}

void iterate_persistent(cudaStream_t st, const IterJob* jobs, int njobs, int maxphase, int R, const double* G,
                        int ldg, double* X, int ldx, double* H, int* status, double* out_sig, double* out_vr,
                        int kv, int* out_clamped, double* ws, const int* phase_ncol, const int* phase_splits,
                        unsigned* bar, int max_k, int grid) {
    grid = std::max(1, std::min(grid, iterate_grid(R)));
    AERO_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), st));
    IterPersistArgs a{jobs, njobs, maxphase, R, ldg, ldx, kv, G, X, H, out_sig, out_vr, ws, status, out_clamped,
                      phase_ncol, phase_splits, bar};
    void* args[] = {&a};
    note_launch();
    AERO_CUDA(cudaLaunchCooperativeKernel(max_k <= 2 ? (void*)k_iterate<2> : (void*)k_iterate<4>, dim3(grid),
                                          dim3(tiles::PNT), args, iterate_smem_bytes(R), st));
}

// ---- small buffers (r <= 96, k <= 2): one WARP per job, all phases ----------
// Jobs of a batch only share G (read-only), so with G in shared memory every
// job runs its whole power / subspace iteration independently: lanes own rows
// (i = lane + 32 t), matvecs from shared memory, reductions by shuffles; no
// grid-wide phase synchronisation at all. Same arithmetic as normalize_job.
constexpr int kWarpIterMaxR = 96;
constexpr int kWarpIterWarps = 8;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void eig2_closed(double a, double b, double c, double& l0, double& l1, double T[4]) {
    // GVL Alg. 8.4.1 rotation (same formulas as small_eig)
    double cn = 1.0, sn = 0.0, t = 0.0;
    if (fabs(b) > 1e-300) {
        const double tau = (c - a) / (2.0 * b);
        t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        cn = 1.0 / sqrt(1.0 + t * t);
        sn = t * cn;
    }
    l0 = a - t * b;
    l1 = c + t * b;
    T[0] = cn;
    T[1] = -sn;
    T[2] = sn;
    T[3] = cn;
}

__global__ void __launch_bounds__(32 * kWarpIterWarps) k_iterate_warp(
    const IterJob* __restrict__ jobs, int njobs, const double* __restrict__ G, int ldg, int R,
    double* __restrict__ X, int ldx, double* __restrict__ H, int* __restrict__ status,
    double* __restrict__ out_sig, double* __restrict__ out_vr, int kv, int* __restrict__ out_clamped) {
    extern __shared__ double smw[];
    double* sG = smw;  // R x R, ld R
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xs = smw + (size_t)R * R + (size_t)warp * 2 * R;  // this warp's x (2 columns, ld R)
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) sG[e] = G[e % R + (int64_t)(e / R) * ldg];
    __syncthreads();
    const int j = blockIdx.x * kWarpIterWarps + warp;
    if (j >= njobs) return;
    const IterJob jb = jobs[j];
    const int r = jb.r, k = jb.k;
    double* xg = X + (int64_t)jb.col * ldx;
    if (status[j] != JOB_ACTIVE) {
        if (lane < k) out_sig[jb.col + lane] = 0.0;
        return;
    }
    constexpr int RT = kWarpIterMaxR / 32;
    double x[RT][2], y[RT][2];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int i = lane + 32 * t;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            x[t][a] = (i < r && a < k) ? xg[i + (int64_t)a * ldx] : 0.0;
            if (i < R) xs[i + a * R] = x[t][a];
        }
    }
    __syncwarp();
    for (int p = 0; p < jb.nphase; ++p) {
        const bool last = (p == jb.nphase - 1);
        // y = G x (rows < r)
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int i = lane + 32 * t;
            double y0 = 0.0, y1 = 0.0;
            if (i < r) {
                for (int l = 0; l < r; ++l) {
                    const double g = sG[i + l * R];
                    y0 = fma(g, xs[l], y0);
                    y1 = fma(g, xs[l + R], y1);
                }
            }
            y[t][0] = y0;
            y[t][1] = (k > 1) ? y1 : 0.0;
        }
        if (jb.type == 0) {
            if (!last) {
                double s = 0.0;
#pragma unroll
                for (int t = 0; t < RT; ++t) s = fma(y[t][0], y[t][0], s);
                s = wsum(s);
                const double nrm = sqrt(s);
                if (nrm < 1e-300) {  // linalg.cpp:112-116
                    if (lane == 0) status[j] = JOB_DEAD;
                    return;
                }
                __syncwarp();
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int i = lane + 32 * t;
                    x[t][0] = (i < r) ? y[t][0] / nrm : 0.0;
                    if (i < R) xs[i] = x[t][0];
                }
                __syncwarp();
            } else {
                double s = 0.0;  // sigma1^2 = x^T G x (linalg.cpp:119)
#pragma unroll
                for (int t = 0; t < RT; ++t) s = fma(x[t][0], y[t][0], s);
                s = wsum(s);
                if (lane == 0) out_sig[jb.col] = s;
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int i = lane + 32 * t;
                    if (i < r) xg[i] = x[t][0];
                }
            }
            continue;
        }
        // simul: S = X^T Y, T = S^{-1/2} (closed-form 2x2 / scalar), clamp
        double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            s00 = fma(x[t][0], y[t][0], s00);
            s01 = fma(x[t][0], y[t][1], s01);
            s10 = fma(x[t][1], y[t][0], s10);
            s11 = fma(x[t][1], y[t][1], s11);
        }
        s00 = wsum(s00);
        s01 = wsum(s01);
        s10 = wsum(s10);
        s11 = wsum(s11);
        double Tm[4], l0, l1;
        if (k == 1) {
            l0 = s00;
            l1 = 0.0;
            Tm[0] = 1.0;
            Tm[1] = Tm[2] = 0.0;
            Tm[3] = 1.0;
        } else {
            eig2_closed(s00, 0.5 * (s01 + s10), s11, l0, l1, Tm);
        }
        const double lmax = (k == 1) ? fmax(l0, 0.0) : fmax(fmax(l0, l1), 0.0);
        const bool ok0 = l0 > 0.0 && l0 > 1e-14 * lmax, ok1 = (k > 1) && l1 > 0.0 && l1 > 1e-14 * lmax;
        const double i0 = ok0 ? 1.0 / sqrt(l0) : 0.0, i1 = ok1 ? 1.0 / sqrt(l1) : 0.0;
        if (last && out_clamped && lane == 0) out_clamped[j] = (!ok0) + (k > 1 && !ok1);
        Tm[0] *= i0;
        Tm[1] *= i0;
        Tm[2] *= i1;
        Tm[3] *= i1;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int i = lane + 32 * t;
            const double h0 = fma(x[t][0], Tm[0], (k > 1) ? x[t][1] * Tm[1] : 0.0);
            const double h1 = fma(x[t][0], Tm[2], (k > 1) ? x[t][1] * Tm[3] : 0.0);
            const double n0 = fma(y[t][0], Tm[0], (k > 1) ? y[t][1] * Tm[1] : 0.0);
            const double n1 = fma(y[t][0], Tm[2], (k > 1) ? y[t][1] * Tm[3] : 0.0);
            if (last && i < r) {
                H[i + (int64_t)jb.col * ldx] = h0;
                if (k > 1) H[i + (int64_t)(jb.col + 1) * ldx] = h1;
            }
            x[t][0] = (i < r) ? n0 : 0.0;
            x[t][1] = (i < r && k > 1) ? n1 : 0.0;
            if (i < R) {
                xs[i] = x[t][0];
                xs[i + R] = x[t][1];
            }
        }
        __syncwarp();
        if (!last) continue;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int i = lane + 32 * t;
            if (i < r) {
                xg[i] = x[t][0];
                if (k > 1) xg[i + ldx] = x[t][1];
            }
        }
        // Ritz values: eig(X^T X) (linalg.cpp:145-150), sorted descending, sign-fixed
        double w00 = 0.0, w01 = 0.0, w11 = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            w00 = fma(x[t][0], x[t][0], w00);
            w01 = fma(x[t][0], x[t][1], w01);
            w11 = fma(x[t][1], x[t][1], w11);
        }
        w00 = wsum(w00);
        w01 = wsum(w01);
        w11 = wsum(w11);
        if (lane == 0) {
            double* vr = out_vr + (int64_t)jb.col * kv;
            if (k == 1) {
                out_sig[jb.col] = sqrt(fmax(w00, 0.0));
                vr[0] = 1.0;
            } else {
                double V2[4], a0, a1;
                eig2_closed(w00, w01, w11, a0, a1, V2);
                // rank (descending, ties by index) and sign fix as cta_sort_signfix
                const int r0 = (a1 > a0) ? 1 : 0, r1 = (a0 >= a1) ? 1 : 0;
                const double lam[2] = {a0, a1};
                for (int c = 0; c < 2; ++c) {
                    const int rk = (c == 0) ? r0 : r1;
                    const double v0 = V2[2 * c], v1 = V2[2 * c + 1];
                    const int at = (fabs(v1) > fabs(v0)) ? 1 : 0;
                    const double sg = ((at ? v1 : v0) < 0.0) ? -1.0 : 1.0;
                    vr[0 + rk * 2] = sg * v0;
                    vr[1 + rk * 2] = sg * v1;
                    out_sig[jb.col + rk] = sqrt(fmax(lam[c], 0.0));
                }
            }
        }
    }
}

// Medium buffers (96 < R <= 512; the C3 levels, the C4 sites): a CTA of
// kCtaIterWarps warps runs its jobs (one per warp, k <= 2) through ALL their
// phases with no grid barrier. G (R x R, L2-resident) is streamed once per
// phase per CTA through shared memory in kCtaIterLB-column chunks and shared
// by the CTA's warps; iterates live in registers (lanes over rows). Same
// arithmetic and summation order as k_iterate_warp. The grid-wide persistent
// kernel spends ~26 us per phase on barriers and latency at these sizes.
constexpr int kCtaIterWarps = 4;
constexpr int kCtaIterLB = 32;
constexpr int kCtaIterMaxR = 512;
template <int RT>
__global__ void __launch_bounds__(32 * kCtaIterWarps) k_iterate_cta(
    const IterJob* __restrict__ jobs, int njobs, const double* __restrict__ G, int ldg, int R,
    double* __restrict__ X, int ldx, double* __restrict__ H, int* __restrict__ status,
    double* __restrict__ out_sig, double* __restrict__ out_vr, int kv, int* __restrict__ out_clamped) {
    extern __shared__ double smc[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ int s_r[kCtaIterWarps], s_np[kCtaIterWarps];
    const int j = blockIdx.x * kCtaIterWarps + warp;
    IterJob jb{};
    bool alive = false;
    if (j < njobs) {
        jb = jobs[j];
        alive = status[j] == JOB_ACTIVE;
        if (!alive && lane < jb.k) out_sig[jb.col + lane] = 0.0;
    }
    if (lane == 0) {
        s_r[warp] = alive ? jb.r : 0;
        s_np[warp] = alive ? jb.nphase : 0;
    }
    __syncthreads();
    int rmax = 0, pmax = 0;
#pragma unroll
    for (int w = 0; w < kCtaIterWarps; ++w) {
        rmax = max(rmax, s_r[w]);
        pmax = max(pmax, s_np[w]);
    }
    double* sG = smc;                                                      // rmax x LB chunk
    double* xs = smc + (size_t)R * kCtaIterLB + (size_t)warp * 2 * R;  // this warp's x
    const int r = jb.r, k = jb.k;
    double* xg = X + (int64_t)jb.col * ldx;
    double x[RT][2], y[RT][2];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int i = lane + 32 * t;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            x[t][a] = (alive && i < r && a < k) ? xg[i + (int64_t)a * ldx] : 0.0;
            if (alive && i < R) xs[i + a * R] = x[t][a];
        }
    }
    __syncwarp();
    for (int p = 0; p < pmax; ++p) {
        const bool act = alive && p < jb.nphase;
        const bool last = (p == jb.nphase - 1);
#pragma unroll
        for (int t = 0; t < RT; ++t) y[t][0] = y[t][1] = 0.0;
        // y = G x (rows < r): G streamed in column chunks shared by the warps
        for (int l0 = 0; l0 < rmax; l0 += kCtaIterLB) {
            const int lb = min(kCtaIterLB, rmax - l0);
            __syncthreads();
            for (int e = threadIdx.x; e < rmax * lb; e += blockDim.x) {
                const int ii = e % rmax, ll = e / rmax;
                sG[ii + ll * rmax] = G[ii + (int64_t)(l0 + ll) * ldg];
            }
            __syncthreads();
            if (act) {
                const int le = min(lb, r - l0);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int i = lane + 32 * t;
                    if (i < r) {
                        double y0 = y[t][0], y1 = y[t][1];
                        for (int ll = 0; ll < le; ++ll) {
                            const double g = sG[i + ll * rmax];
                            y0 = fma(g, xs[l0 + ll], y0);
                            y1 = fma(g, xs[l0 + ll + R], y1);
                        }
                        y[t][0] = y0;
                        y[t][1] = y1;
                    }
                }
            }
        }
        if (!act) continue;
        if (k <= 1)
#pragma unroll
            for (int t = 0; t < RT; ++t) y[t][1] = 0.0;
        if (jb.type == 0) {
            if (!last) {
                double s = 0.0;
#pragma unroll
                for (int t = 0; t < RT; ++t) s = fma(y[t][0], y[t][0], s);
                s = wsum(s);
                const double nrm = sqrt(s);
                if (nrm < 1e-300) {  // linalg.cpp:112-116
                    if (lane == 0) status[j] = JOB_DEAD;
                    alive = false;
                    continue;
                }
                __syncwarp();
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int i = lane + 32 * t;
                    x[t][0] = (i < r) ? y[t][0] / nrm : 0.0;
                    if (i < R) xs[i] = x[t][0];
                }
                __syncwarp();
            } else {
                double s = 0.0;  // sigma1^2 = x^T G x (linalg.cpp:119)
#pragma unroll
                for (int t = 0; t < RT; ++t) s = fma(x[t][0], y[t][0], s);
                s = wsum(s);
                if (lane == 0) out_sig[jb.col] = s;
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int i = lane + 32 * t;
                    if (i < r) xg[i] = x[t][0];
                }
            }
            continue;
        }
        // simul: S = X^T Y, T = S^{-1/2} (closed-form 2x2 / scalar), clamp
        double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            s00 = fma(x[t][0], y[t][0], s00);
            s01 = fma(x[t][0], y[t][1], s01);
            s10 = fma(x[t][1], y[t][0], s10);
            s11 = fma(x[t][1], y[t][1], s11);
        }
        s00 = wsum(s00);
        s01 = wsum(s01);
        s10 = wsum(s10);
        s11 = wsum(s11);
        double Tm[4], l0, l1;
        if (k == 1) {
            l0 = s00;
            l1 = 0.0;
            Tm[0] = 1.0;
            Tm[1] = Tm[2] = 0.0;
            Tm[3] = 1.0;
        } else {
            eig2_closed(s00, 0.5 * (s01 + s10), s11, l0, l1, Tm);
        }
        const double lmax = (k == 1) ? fmax(l0, 0.0) : fmax(fmax(l0, l1), 0.0);
        const bool ok0 = l0 > 0.0 && l0 > 1e-14 * lmax, ok1 = (k > 1) && l1 > 0.0 && l1 > 1e-14 * lmax;
        const double i0 = ok0 ? 1.0 / sqrt(l0) : 0.0, i1 = ok1 ? 1.0 / sqrt(l1) : 0.0;
        if (last && out_clamped && lane == 0) out_clamped[j] = (!ok0) + (k > 1 && !ok1);
        Tm[0] *= i0;
        Tm[1] *= i0;
        Tm[2] *= i1;
        Tm[3] *= i1;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int i = lane + 32 * t;
            const double h0 = fma(x[t][0], Tm[0], (k > 1) ? x[t][1] * Tm[1] : 0.0);
            const double h1 = fma(x[t][0], Tm[2], (k > 1) ? x[t][1] * Tm[3] : 0.0);
            const double n0 = fma(y[t][0], Tm[0], (k > 1) ? y[t][1] * Tm[1] : 0.0);
            const double n1 = fma(y[t][0], Tm[2], (k > 1) ? y[t][1] * Tm[3] : 0.0);
            if (last && i < r) {
                H[i + (int64_t)jb.col * ldx] = h0;
                if (k > 1) H[i + (int64_t)(jb.col + 1) * ldx] = h1;
            }
            x[t][0] = (i < r) ? n0 : 0.0;
            x[t][1] = (i < r && k > 1) ? n1 : 0.0;
            if (i < R) {
                xs[i] = x[t][0];
                xs[i + R] = x[t][1];
            }
        }
        __syncwarp();
        if (!last) continue;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int i = lane + 32 * t;
            if (i < r) {
                xg[i] = x[t][0];
                if (k > 1) xg[i + ldx] = x[t][1];
            }
        }
        // Ritz values: eig(X^T X) (linalg.cpp:145-150), sorted descending, sign-fixed
        double w00 = 0.0, w01 = 0.0, w11 = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            w00 = fma(x[t][0], x[t][0], w00);
            w01 = fma(x[t][0], x[t][1], w01);
            w11 = fma(x[t][1], x[t][1], w11);
        }
        w00 = wsum(w00);
        w01 = wsum(w01);
        w11 = wsum(w11);
        if (lane == 0) {
            double* vr = out_vr + (int64_t)jb.col * kv;
            if (k == 1) {
                out_sig[jb.col] = sqrt(fmax(w00, 0.0));
                vr[0] = 1.0;
            } else {
                double V2[4], a0, a1;
                eig2_closed(w00, w01, w11, a0, a1, V2);
                const int r0 = (a1 > a0) ? 1 : 0, r1 = (a0 >= a1) ? 1 : 0;
                const double lam[2] = {a0, a1};
                for (int cc = 0; cc < 2; ++cc) {
                    const int rk = (cc == 0) ? r0 : r1;
                    const double v0 = V2[2 * cc], v1 = V2[2 * cc + 1];
                    const int at = (fabs(v1) > fabs(v0)) ? 1 : 0;
                    const double sg = ((at ? v1 : v0) < 0.0) ? -1.0 : 1.0;
                    vr[0 + rk * 2] = sg * v0;
                    vr[1 + rk * 2] = sg * v1;
                    out_sig[jb.col + rk] = sqrt(fmax(lam[cc], 0.0));
                }
            }
        }
    }
}

bool iterate_cta(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg, int R, double* X,
                 int ldx, double* H, int* status, double* out_sig, double* out_vr, int kv, int* out_clamped,
                 int max_k) {
    if (R > kCtaIterMaxR || max_k > 2 || njobs <= 0) return false;
    const size_t smem = sizeof(double) * ((size_t)R * kCtaIterLB + (size_t)kCtaIterWarps * 2 * R);
    static bool attr = false;
    if (!attr) {
        const int mx = (int)(sizeof(double) * ((size_t)kCtaIterMaxR * kCtaIterLB + (size_t)kCtaIterWarps * 2 * kCtaIterMaxR));
        AERO_CUDA(cudaFuncSetAttribute(k_iterate_cta<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        AERO_CUDA(cudaFuncSetAttribute(k_iterate_cta<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        attr = true;
    }
    const int grid = (njobs + kCtaIterWarps - 1) / kCtaIterWarps;
    if (R <= 256)
        k_iterate_cta<8><<<grid, 32 * kCtaIterWarps, smem, st>>>(jobs, njobs, G, ldg, R, X, ldx, H, status, out_sig,
                                                                 out_vr, kv, out_clamped);
    else
        k_iterate_cta<16><<<grid, 32 * kCtaIterWarps, smem, st>>>(jobs, njobs, G, ldg, R, X, ldx, H, status,
                                                                  out_sig, out_vr, kv, out_clamped);
    AERO_LAUNCHED();
    return true;
}

bool iterate_warp(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg, int R, double* X,
                  int ldx, double* H, int* status, double* out_sig, double* out_vr, int kv, int* out_clamped,
                  int max_k) {
    if (R > kWarpIterMaxR || max_k > 2 || njobs <= 0) return false;
    const size_t smem = sizeof(double) * ((size_t)R * R + (size_t)kWarpIterWarps * 2 * R);
    static bool attr = false;
    if (!attr) {
        AERO_CUDA(cudaFuncSetAttribute(k_iterate_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * (kWarpIterMaxR * kWarpIterMaxR +
                                                               kWarpIterWarps * 2 * kWarpIterMaxR))));
        attr = true;
    }
    k_iterate_warp<<<(njobs + kWarpIterWarps - 1) / kWarpIterWarps, 32 * kWarpIterWarps, smem, st>>>(
        jobs, njobs, G, ldg, R, X, ldx, H, status, out_sig, out_vr, kv, out_clamped);
    AERO_LAUNCHED();
    return true;
}

void iter_normalize(cudaStream_t st, const IterJob* jobs, int njobs, int phase, double* X,
                    const double* Y, int ldx, double* H, int* status, double* out_sig,
                    double* out_vr, int kv, int* out_clamped, int max_k) {
    if (njobs <= 0) return;
    if (max_k <= 2)
        launch_normalize<2, false>(st, jobs, njobs, phase, X, Y, ldx, H, status, out_sig, out_vr, kv,
                                   out_clamped, nullptr, 0, 0, 0);
    else if (max_k <= 4)
        launch_normalize<4, false>(st, jobs, njobs, phase, X, Y, ldx, H, status, out_sig, out_vr, kv,
                                   out_clamped, nullptr, 0, 0, 0);
    else
        launch_normalize<64, false>(st, jobs, njobs, phase, X, Y, ldx, H, status, out_sig, out_vr, kv,
                                    out_clamped, nullptr, 0, 0, 0);
}

void iter_normalize_ws(cudaStream_t st, const IterJob* jobs, int njobs, int phase, double* X,
                       int ldx, const double* ws, int M, int N, int splits, double* H, int* status,
                       double* out_sig, double* out_vr, int kv, int* out_clamped, int max_k) {
    if (njobs <= 0) return;
    const int64_t sstride = (int64_t)M * N;
    if (max_k <= 2)
        launch_normalize<2, true>(st, jobs, njobs, phase, X, nullptr, ldx, H, status, out_sig, out_vr,
                                  kv, out_clamped, ws, M, sstride, splits);
    else
        launch_normalize<4, true>(st, jobs, njobs, phase, X, nullptr, ldx, H, status, out_sig, out_vr,
                                  kv, out_clamped, ws, M, sstride, splits);
}

// ============================================================================
// small helpers
// ============================================================================
__global__ void k_scale_columns(int n, int ncol, double* V, int ld, const double* scale) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * ncol) return;
    const int i = (int)(e % n), j = (int)(e / n);
    V[i + (int64_t)j * ld] *= scale[j];
}
void scale_columns(cudaStream_t st, int n, int ncol, double* V, int ld, const double* scale) {
    const int64_t tot = (int64_t)n * ncol;
    if (tot <= 0) return;
    k_scale_columns<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, ncol, V, ld, scale);
    AERO_LAUNCHED();
}

__global__ void k_scale_rows(int n, int ncol, double* V, int ld, const double* scale) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * ncol) return;
    const int i = (int)(e % n), j = (int)(e / n);
    V[i + (int64_t)j * ld] *= scale[i];
}
void scale_rows(cudaStream_t st, int n, int ncol, double* V, int ld, const double* scale) {
    const int64_t tot = (int64_t)n * ncol;
    if (tot <= 0) return;
    k_scale_rows<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, ncol, V, ld, scale);
    AERO_LAUNCHED();
}

__global__ void k_fd_weights(const double* lam, int n, int ell, int keep, double* w) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= keep) return;
    const double si = sqrt(fmax(lam[i], 0.0));
    double cut = 0.0;
    if (ell <= n) {
        const double se = sqrt(fmax(lam[ell - 1], 0.0));
        cut = se * se;
    }
    const double s2 = si * si - cut;
    w[i] = (s2 > 0.0 && si > 0.0) ? sqrt(s2) / si : 0.0;
}
void fd_weights(cudaStream_t st, const double* lam, int n, int ell, int keep, double* w) {
    k_fd_weights<<<(keep + 127) / 128, 128, 0, st>>>(lam, n, ell, keep, w);
    AERO_LAUNCHED();
}

__global__ void k_fix_signs(int d, double* Z, int ld, double* flips) {
    __shared__ double bv[32];
    __shared__ int bi[32];
    double* z = Z + (int64_t)blockIdx.x * ld;
    double best = -1.0;
    int at = 0x7fffffff;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const double v = fabs(z[i]);
        if (v > best) { best = v; at = i; }
    }
    // warp argmax with first-index tie break
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, at, o);
        if (ov > best || (ov == best && oi < at)) { best = ov; at = oi; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) { bv[wid] = best; bi[wid] = at; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w)
            if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
    }
    __syncthreads();
    const double sg = (bi[0] < d && z[bi[0]] < 0.0) ? -1.0 : 1.0;
    __syncthreads();
    if (sg < 0.0)
        for (int i = threadIdx.x; i < d; i += blockDim.x) z[i] = -z[i];
    if (threadIdx.x == 0 && flips) flips[blockIdx.x] = sg;
}
void fix_column_signs(cudaStream_t st, int d, int k, double* Z, int ld, double* flips) {
    if (k <= 0) return;
    k_fix_signs<<<k, 256, 0, st>>>(d, Z, ld, flips);
    AERO_LAUNCHED();
}

__global__ void k_symmetrize(int n, double* A, int lda) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * n) return;
    const int i = (int)(e % n), j = (int)(e / n);
    if (i >= j) return;
    const double v = 0.5 * (A[i + (int64_t)j * lda] + A[j + (int64_t)i * lda]);
    A[i + (int64_t)j * lda] = v;
    A[j + (int64_t)i * lda] = v;
}
void symmetrize(cudaStream_t st, int n, double* A, int lda) {
    const int64_t tot = (int64_t)n * n;
    if (tot <= 0) return;
    k_symmetrize<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, A, lda);
    AERO_LAUNCHED();
}

__global__ void k_fill(double* p, int64_t count) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < count) p[e] = 0.0;
}
void fill_zero(cudaStream_t st, double* p, int64_t count) {
    if (count <= 0) return;
    k_fill<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(p, count);
    AERO_LAUNCHED();
}

__global__ void k_copy_matrix(int m, int n, const double* A, int lda, double* B, int ldb) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)m * n) return;
    const int i = (int)(e % m), j = (int)(e / m);
    B[i + (int64_t)j * ldb] = A[i + (int64_t)j * lda];
}
void copy_matrix(cudaStream_t st, int m, int n, const double* A, int lda, double* B, int ldb) {
    const int64_t tot = (int64_t)m * n;
    if (tot <= 0) return;
    k_copy_matrix<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(m, n, A, lda, B, ldb);
    AERO_LAUNCHED();
}

void rows_to_cols(cudaStream_t st, const double* rows, int64_t n, int64_t ld, int d, double* Ct,
                  int ldc) {
    if (n <= 0) return;
    AERO_CUDA(cudaMemcpy2DAsync(Ct, sizeof(double) * ldc, rows, sizeof(double) * ld,
                                sizeof(double) * d, n, cudaMemcpyDefault, st));
}

__global__ void k_add_identity(int k, double* A, int lda, double alpha) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) A[i + (int64_t)i * lda] += alpha;
}
void add_identity(cudaStream_t st, int k, double* A, int lda, double alpha) {
    if (k <= 0) return;
    k_add_identity<<<(k + 127) / 128, 128, 0, st>>>(k, A, lda, alpha);
    AERO_LAUNCHED();
}

__global__ void k_shrink_rows(const double* lam, const double* V, int ldv, int d, int ell,
                              double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)ell * d) return;
    const int i = (int)(e / d), j = (int)(e % d);
    double v = 0.0;
    if (i < d) {
        const double cut = (ell <= d) ? fmax(lam[ell - 1], 0.0) : 0.0;
        const double w = fmax(lam[i], 0.0) - cut;
        if (w > 0.0) v = sqrt(w) * V[j + (int64_t)i * ldv];
    }
    out[e] = v;
}
void shrink_rows(cudaStream_t st, const double* lam, const double* V, int ldv, int d, int ell,
                 double* out_rm) {
    const int64_t tot = (int64_t)ell * d;
    if (tot <= 0) return;
    k_shrink_rows<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(lam, V, ldv, d, ell, out_rm);
    AERO_LAUNCHED();
}

// restore contribution K terms: K_s = Mt_s^T Z_s (xi x xi), Y_s = Z_s K_s
__global__ void k_restore_k(int d, const double* __restrict__ Z, const double* __restrict__ Mt,
                            int ld, const int* __restrict__ offsets, const int* __restrict__ widths,
                            double* __restrict__ Y) {
    extern __shared__ double sm[];
    __shared__ double red[32];
    const int off = offsets[blockIdx.x], xi = widths[blockIdx.x];
    double* K = sm;  // xi*xi
    for (int a = 0; a < xi; ++a)
        for (int b = 0; b < xi; ++b) {
            double t = 0.0;
            for (int i = threadIdx.x; i < d; i += blockDim.x)
                t = fma(Mt[i + (int64_t)(off + a) * ld], Z[i + (int64_t)(off + b) * ld], t);
            t = block_sum(t, red);
            if (threadIdx.x == 0) K[a + b * xi] = t;
        }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x)
        for (int b = 0; b < xi; ++b) {
            double t = 0.0;
            for (int a = 0; a < xi; ++a) t = fma(Z[i + (int64_t)(off + a) * ld], K[a + b * xi], t);
            Y[i + (int64_t)(off + b) * ld] = t;
        }
}
void restore_k_terms(cudaStream_t st, int d, const double* Z, const double* Mt, int ld,
                     const int* offsets, const int* widths, int nsnap, double* Y) {
    // widths are bounded by the caller (xi <= kRestoreMaxXi per snapshot)
    if (nsnap <= 0) return;
    const size_t smem = sizeof(double) * 64 * 64;
    k_restore_k<<<nsnap, 256, smem, st>>>(d, Z, Mt, ld, offsets, widths, Y);
    AERO_LAUNCHED();
}

// ============================================================================
// stream generator (DESIGN.md GENERATOR spec): one CTA per row
// ============================================================================
__global__ void k_gen_rows(int d, int k, int k2, const double* __restrict__ U1,
                           const double* __restrict__ U2, double rho, double rho2, double scale2,
                           double noise, double r_max, uint64_t seed, uint64_t stream, int64_t t0,
                           double* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red[32];
    double* coef = sm;          // k + k2
    const int64_t t = t0 + blockIdx.x;
    const uint64_t s0 = rng_state0(seed, (stream << 32) + (uint64_t)t);
    for (int l = threadIdx.x; l < k + k2; l += blockDim.x) coef[l] = rng_gaussian_at(s0, l);
    __syncthreads();
    if (threadIdx.x == 0) {
        double sig = 1.0;
        for (int l = 0; l < k; ++l) { coef[l] *= sig; sig *= rho; }
        sig = scale2;
        for (int l = 0; l < k2; ++l) { coef[k + l] *= sig; sig *= rho2; }
    }
    __syncthreads();
    double* a = out + (int64_t)blockIdx.x * d;
    double ss = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double v = noise * rng_gaussian_at(s0, (uint64_t)(k + k2 + j));
        for (int l = 0; l < k; ++l) v += coef[l] * U1[(int64_t)l * d + j];
        for (int l = 0; l < k2; ++l) v += coef[k + l] * U2[(int64_t)l * d + j];
        a[j] = v;
        ss = fma(v, v, ss);
    }
    ss = block_sum(ss, red);
    const uint64_t g = (uint64_t)(k + k2 + d);
    const double u = rng_uniform_at(s0, 2 * ((g + 1) / 2) + 1);
    const double scale = sqrt(pow(r_max, u) / ss);
    for (int j = threadIdx.x; j < d; j += blockDim.x) a[j] *= scale;
}
void gen_rows(cudaStream_t st, int d, int k, int k2, const double* U1, const double* U2,
              double rho, double rho2, double scale2, double noise, double r_max, uint64_t seed,
              uint64_t stream, int64_t t0, int64_t n, double* out) {
    for (int64_t off = 0; off < n; off += 1 << 20) {
        const int64_t cnt = std::min<int64_t>(n - off, 1 << 20);
        k_gen_rows<<<(unsigned)cnt, 256, sizeof(double) * (k + k2 + 1), st>>>(
            d, k, k2, U1, U2, rho, rho2, scale2, noise, r_max, seed, stream, t0 + off,
            out + off * d);
        AERO_LAUNCHED();
    }
}

__global__ void k_gen_gauss(uint64_t s0, int64_t count, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < count) out[e] = rng_gaussian_at(s0, (uint64_t)e);
}
void gen_gaussian_matrix(cudaStream_t st, uint64_t state0, int64_t count, double* out) {
    if (count <= 0) return;
    k_gen_gauss<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(state0, count, out);
    AERO_LAUNCHED();
}

}  // namespace aero_b200
