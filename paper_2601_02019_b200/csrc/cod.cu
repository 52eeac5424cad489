// CodState -- sliding-window approximate matrix multiplication
// (reference amm.hpp:35-69, amm.cpp:27-122) on the B200.
//
// The reference forms the dense product p = A B^T (dx x dy) every row
// (amm.cpp:65) and runs power_iteration(p) and simul_iter(p), simul_iter(p^T)
// on it. Every randomized estimate there starts in dy- (or dx-) space, so it
// only depends on p itself; p = A B^T is invariant under simultaneous column
// transforms of A and B. We therefore iterate in the column space of the
// buffers: with GA = A^T A, GB = B^T B (c x c, c <= 2 ell),
//   p^T p (B v) = B (GA GB v),     p p^T (A h) = A (GB GA h),
// so each iteration is two c x c products instead of two dx x dy passes, the
// first step maps the dy/dx-space start (x0, Pi) through B^T / A^T, and the
// final Rayleigh-Ritz uses the GA/GB-orthonormal basis (same subspace, same
// Ritz values as the reference's Householder iteration up to rounding).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <deque>
#include <vector>

#include "aero_common.cuh"
#include "engines.hpp"

namespace aero_b200 {

namespace {
constexpr int COD_KMAX = 8;  // in-kernel rank; larger ranks use the host-driven path

struct CodJob {
    int type;   // 0: power_iteration(p); 1: simul_iter(p) (z side); 2: simul_iter(p^T) (h side)
    int c, k, nit;
    uint64_t rng0;
};

constexpr int COD_THREADS = 512;
constexpr int COD_MV_PARTS = 2;  // threads per output row in cta_matvec (split over l)

// y[0:c, 0:k] = G[0:c, 0:c] x[0:c, 0:k] (G global column-major ld, x/y shared,
// ld c). Each output row is shared by COD_MV_PARTS threads over l, 8 loads in
// flight per thread; `part` holds (parts-1) * (blockDim/parts) * COD_KMAX doubles.
__device__ void cta_matvec(const double* __restrict__ G, int ld, int c, int k, const double* x,
                           double* y, double* part) {
    const int R = blockDim.x / COD_MV_PARTS;
    const int ii = threadIdx.x % R, p = threadIdx.x / R;
    const int l0 = (c * p) / COD_MV_PARTS, l1 = (c * (p + 1)) / COD_MV_PARTS;
    for (int i0 = 0; i0 < c; i0 += R) {
        const int i = i0 + ii;
        double acc[COD_KMAX];
#pragma unroll
        for (int j = 0; j < COD_KMAX; ++j) acc[j] = 0.0;
        if (i < c) {
            int l = l0;
            for (; l + 8 <= l1; l += 8) {
                double g[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) g[u] = G[i + (int64_t)(l + u) * ld];
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int j = 0; j < COD_KMAX; ++j)
                        if (j < k) acc[j] = fma(g[u], x[l + u + j * c], acc[j]);
            }
            for (; l < l1; ++l) {
                const double g = G[i + (int64_t)l * ld];
#pragma unroll
                for (int j = 0; j < COD_KMAX; ++j)
                    if (j < k) acc[j] = fma(g, x[l + j * c], acc[j]);
            }
        }
        if (p > 0 && i < c)
#pragma unroll
            for (int j = 0; j < COD_KMAX; ++j)
                if (j < k) part[(p - 1) * R * COD_KMAX + ii + j * R] = acc[j];
        __syncthreads();
        if (p == 0 && i < c)
#pragma unroll
            for (int j = 0; j < COD_KMAX; ++j)
                if (j < k) {
                    double v = acc[j];
                    for (int q = 1; q < COD_MV_PARTS; ++q) v += part[(q - 1) * R * COD_KMAX + ii + j * R];
                    y[i + j * c] = v;
                }
        __syncthreads();
    }
}

// S[a,b] = sum_i x[i,a] y[i,b] (k x k, shared) for shared x, y (ld c)
__device__ void cta_small_gram(const double* x, const double* y, int c, int k, double* S, double* red) {
    for (int e = 0; e < k * k; ++e) {
        const int a = e % k, b = e / k;
        double s = 0.0;
        for (int i = threadIdx.x; i < c; i += blockDim.x) s = fma(x[i + a * c], y[i + b * c], s);
        s = block_sum(s, red);
        if (threadIdx.x == 0) S[e] = s;
    }
    __syncthreads();
}

__device__ void cta_eig_small(double* W, double* V, int k, double* cs);  // below

// x <- x S^{-1/2} for S = x^T M x (k x k, shared); M-inner product given as
// the Gram S computed by the caller; T scratch k*k; lam scratch k
__device__ void cta_orthonormalize(double* x, int c, int k, double* S, double* T, double* lam,
                                   double* cs, double* tmp) {
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int a = e % k, b = e / k;
        tmp[e] = 0.5 * (S[a + b * k] + S[b + a * k]);
    }
    __syncthreads();
    cta_eig_small(tmp, T, k, cs);
    if (threadIdx.x == 0) {
        double lmax = 0.0;
        for (int i = 0; i < k; ++i) lmax = fmax(lmax, tmp[i + i * k]);
        for (int i = 0; i < k; ++i) {
            const double l = tmp[i + i * k];
            lam[i] = (l > 0.0 && l > 1e-14 * lmax) ? 1.0 / sqrt(l) : 0.0;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x) {
        double xr[COD_KMAX];
#pragma unroll
        for (int a = 0; a < COD_KMAX; ++a)
            if (a < k) xr[a] = x[i + a * c];
#pragma unroll
        for (int b = 0; b < COD_KMAX; ++b) {
            if (b >= k) break;
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < COD_KMAX; ++a)
                if (a < k) s = fma(xr[a], T[a + b * k] * lam[b], s);
            x[i + b * c] = s;
        }
    }
    __syncthreads();
}

// one CTA per job. A: dx x c, B: dy x c (column-major, ld dx / dy); GA, GB: c x c (ld cap).
// outputs: sig[k] (gate: sig[0] = sigma1^2), hv (c x k global: the c-space
// basis h V of the Ritz vectors, z = A hv or B hv), status
__global__ void __launch_bounds__(COD_THREADS) k_cod_job(const CodJob* __restrict__ jobs, const double* __restrict__ A, int dx,
                          const double* __restrict__ B, int dy, const double* __restrict__ GA,
                          const double* __restrict__ GB, int cap, double* __restrict__ sig,
                          double* __restrict__ hv, int* __restrict__ status, double* pibuf,
                          int64_t pi_stride) {
    extern __shared__ double sm[];
    const CodJob jb = jobs[blockIdx.x];
    const int c = jb.c, k = jb.k;
    double* red = sm;                       // 32
    double* v = red + 32;                   // c*k
    double* t = v + c * COD_KMAX;           // c*k
    double* S = t + c * COD_KMAX;           // k*k
    double* T = S + COD_KMAX * COD_KMAX;    // k*k
    double* W = T + COD_KMAX * COD_KMAX;    // k*k
    double* lam = W + COD_KMAX * COD_KMAX;  // k
    double* cs = lam + COD_KMAX;            // jacobi scratch (64)
    double* mvp = cs + 64;                  // cta_matvec partials
    double* sig_o = sig + blockIdx.x * COD_KMAX;
    double* hv_o = hv + (int64_t)blockIdx.x * cap * COD_KMAX;
    // zero p <=> trace(GA GB) == 0 (reference checks a.norm() == 0, linalg.cpp:101,131)
    double tr = 0.0;  // trace(GA GB) = sum GA .* GB (GB symmetric)
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
        const int i = e % c, l = e / c;
        tr = fma(GA[i + (int64_t)l * cap], GB[i + (int64_t)l * cap], tr);
    }
    tr = block_sum(tr, red);
    if (tr == 0.0) {
        if (threadIdx.x == 0) {
            status[blockIdx.x] = JOB_ZERO;
            for (int j = 0; j < k; ++j) sig_o[j] = 0.0;
        }
        return;
    }
    if (threadIdx.x == 0) status[blockIdx.x] = JOB_ACTIVE;
    // M1 acts first, M2 second: z side / gate iterate GB then GA on v = B^T x
    // for the gate; the simul z side iterates h <- GB (GA h); the h side GA (GB h)
    const double* Gfirst = (jb.type == 2) ? GB : GA;
    const double* Gsecond = (jb.type == 2) ? GA : GB;
    const double* Mapin = (jb.type == 2) ? A : B;  // dvec-space -> c-space: Mapin^T
    const int dvec = (jb.type == 2) ? dx : dy;
    const int ldm = (jb.type == 2) ? dx : dy;
    // start vectors in dvec space (x0: dvec gaussians; Pi: dvec x k row-major,
    // linalg.cpp:35-40) generated once into global scratch, then mapped to
    // c-space: v = Mapin^T start
    double* pi = pibuf + (int64_t)blockIdx.x * pi_stride;
    for (int e = threadIdx.x; e < dvec * k; e += blockDim.x) pi[e] = rng_gaussian_at(jb.rng0, e);
    __syncthreads();
    {  // warp per buffer column i, lanes over the dvec coordinates
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
        for (int i = wid; i < c; i += nwarp) {
            double acc[COD_KMAX];
#pragma unroll
            for (int j = 0; j < COD_KMAX; ++j) acc[j] = 0.0;
            for (int l = lane; l < dvec; l += 32) {
                const double m = Mapin[l + (int64_t)i * ldm];
#pragma unroll
                for (int j = 0; j < COD_KMAX; ++j)
                    if (j < k) acc[j] = fma(m, pi[l * k + j], acc[j]);
            }
#pragma unroll
            for (int j = 0; j < COD_KMAX; ++j)
                if (j < k) {
                    const double sum = warp_sum(acc[j]);
                    if (lane == 0) v[i + j * c] = sum;
                }
        }
    }
    __syncthreads();
    if (jb.type == 0) {
        // power_iteration(p, kp) (linalg.cpp:96-121) with x = B v after step 0:
        // y = p^T p x = B (GA GB v), ||y||^2 = v'^T GB v', sigma^2 = (GB v)^T GA (GB v)
        double* t1 = t;
        double* t2 = t + c;
        double* t3 = t + 2 * c;
        double s = 0.0;
        for (int l = threadIdx.x; l < dvec; l += blockDim.x) s = fma(pi[l], pi[l], s);
        s = block_sum(s, red);
        const double nx = sqrt(s);
        for (int i = threadIdx.x; i < c; i += blockDim.x) v[i] /= nx;  // u = B^T x0 / ||x0||
        __syncthreads();
        for (int it = 0; it < jb.nit; ++it) {
            if (it == 0) {
                cta_matvec(GA, cap, c, 1, v, t1, mvp);  // y = B (GA u)
            } else {
                cta_matvec(GB, cap, c, 1, v, t2, mvp);
                cta_matvec(GA, cap, c, 1, t2, t1, mvp);  // y = B (GA GB v)
            }
            cta_matvec(GB, cap, c, 1, t1, t3, mvp);
            double n2 = 0.0;
            for (int i = threadIdx.x; i < c; i += blockDim.x) n2 = fma(t1[i], t3[i], n2);
            n2 = block_sum(n2, red);
            const double nrm = sqrt(fmax(n2, 0.0));
            if (nrm < 1e-300) {  // linalg.cpp:112-116
                if (threadIdx.x == 0) {
                    status[blockIdx.x] = JOB_DEAD;
                    sig_o[0] = 0.0;
                }
                return;
            }
            for (int i = threadIdx.x; i < c; i += blockDim.x) v[i] = t1[i] / nrm;
            __syncthreads();
        }
        cta_matvec(GB, cap, c, 1, v, t2, mvp);
        cta_matvec(GA, cap, c, 1, t2, t3, mvp);
        double s2 = 0.0;
        for (int i = threadIdx.x; i < c; i += blockDim.x) s2 = fma(t2[i], t3[i], s2);
        s2 = block_sum(s2, red);
        if (threadIdx.x == 0) sig_o[0] = s2;
        return;
    }
    // simul_iter (linalg.cpp:123-152) in c-space: h0 = v (Mapin^T Pi)
    for (int it = 0; it <= jb.nit; ++it) {
        if (it > 0) {  // h <- Gsecond (Gfirst h)
            cta_matvec(Gfirst, cap, c, k, v, t, mvp);
            cta_matvec(Gsecond, cap, c, k, t, v, mvp);
        }
        cta_small_gram(v, v, c, k, S, red);  // Euclidean re-orthonormalization (span-preserving)
        cta_orthonormalize(v, c, k, S, T, lam, cs, W);
    }
    // final basis orthonormal in the Gfirst inner product (g = Mapout h)
    cta_matvec(Gfirst, cap, c, k, v, t, mvp);
    cta_small_gram(v, t, c, k, S, red);
    cta_orthonormalize(v, c, k, S, T, lam, cs, W);
    // Ritz: w = Map^T ... : w^T w = (Gfirst h)^T Gsecond (Gfirst h)
    cta_matvec(Gfirst, cap, c, k, v, t, mvp);
    double* u2 = hv_o;  // c*k scratch
    cta_matvec(Gsecond, cap, c, k, t, u2, mvp);
    cta_small_gram(t, u2, c, k, S, red);
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int a = e % k, b = e / k;
        W[e] = 0.5 * (S[a + b * k] + S[b + a * k]);
    }
    __syncthreads();
    cta_eig_small(W, T, k, cs);
    // sort descending + sign fix of V (linalg.cpp:146-150)
    if (threadIdx.x == 0) {
        int ord[COD_KMAX];
        for (int i = 0; i < k; ++i) ord[i] = i;
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j)
                if (W[ord[j] + ord[j] * k] > W[ord[i] + ord[i] * k]) {
                    const int x = ord[i];
                    ord[i] = ord[j];
                    ord[j] = x;
                }
        for (int i = 0; i < k; ++i) {
            lam[i] = W[ord[i] + ord[i] * k];
            sig_o[i] = sqrt(fmax(lam[i], 0.0));
            for (int a = 0; a < k; ++a) S[a + i * k] = T[a + ord[i] * k];
        }
    }
    __syncthreads();
    // hv = h V (c x k)
    for (int i = threadIdx.x; i < c; i += blockDim.x)
        for (int b = 0; b < k; ++b) {
            double s = 0.0;
            for (int a = 0; a < k; ++a) s = fma(v[i + a * c], S[a + b * k], s);
            hv_o[i + (int64_t)b * cap] = s;
        }
}

__device__ void cta_eig_small(double* W, double* V, int k, double* cs) {
    // Jacobi sweeps by thread 0 (k <= COD_KMAX)
    if (threadIdx.x == 0) {
        for (int e = 0; e < k * k; ++e) V[e] = (e % (k + 1) == 0) ? 1.0 : 0.0;
        for (int sweep = 0; sweep < 50; ++sweep) {
            bool rot = false;
            for (int p = 0; p < k; ++p)
                for (int q = p + 1; q < k; ++q) {
                    const double apq = W[p + q * k], app = W[p + p * k], aqq = W[q + q * k];
                    if (!(fabs(apq) > 1e-300 && fabs(apq) > 2.2e-16 * sqrt(fabs(app * aqq)))) continue;
                    rot = true;
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    const double cn = 1.0 / sqrt(1.0 + t * t), sn = t * cn;
                    for (int r = 0; r < k; ++r) {  // A <- A R (columns p, q)
                        const double a = W[r + p * k], b = W[r + q * k];
                        W[r + p * k] = cn * a - sn * b;
                        W[r + q * k] = sn * a + cn * b;
                    }
                    for (int r = 0; r < k; ++r) {  // A <- R^T A (rows p, q)
                        const double a = W[p + r * k], b = W[q + r * k];
                        W[p + r * k] = cn * a - sn * b;
                        W[q + r * k] = sn * a + cn * b;
                    }
                    W[p + q * k] = W[q + p * k] = 0.0;
                    for (int r = 0; r < k; ++r) {
                        const double a = V[r + p * k], b = V[r + q * k];
                        V[r + p * k] = cn * a - sn * b;
                        V[r + q * k] = sn * a + cn * b;
                    }
                }
            if (!rot) break;
        }
    }
    __syncthreads();
}

// G[c0 + j, i] = G[i, c0 + j] for i < c0 (mirror the appended columns into rows)
__global__ void k_cod_mirror(int c0, int nb, double* G, int ld) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)c0 * nb) return;
    const int i = (int)(e % c0), j = (int)(e / c0);
    G[(c0 + j) + (int64_t)i * ld] = G[i + (int64_t)(c0 + j) * ld];
}
}  // namespace

constexpr int COD_MAX_BATCH = 128;  // speculative gate jobs per launch

// Snapshot storage: columns of consecutive snapshots packed into chunks of
// kCodChunkCols columns (z, h, zm^T, mh arrays per chunk). Snapshots are born
// and expire in time order, so chunks fill at the back and empty at the front;
// an emptied chunk is kept for reuse (a cudaFree would synchronize the device
// on every expiry -- the first version did 4 cudaMalloc + 4 cudaFree per
// snapshot, and C5 dumps on most rows). Reuse is ordered by the engine stream.
constexpr int kCodChunkCols = 1024;
struct CodChunk {
    double *z = nullptr, *h = nullptr, *zm_t = nullptr, *mh = nullptr;
    int used = 0, live = 0;
};
struct CodSnap {
    int xi;
    int64_t s, t;
    double *z, *h, *zm_t, *mh;  // device: z dx x xi, h dy x xi, zm^T dy x xi, mh dx x xi
    CodChunk* chunk;
};

struct CodEngine::Impl {
    int dx, dy, ell, cap, kp, qz, qh, dev;
    double eps, theta;
    int64_t n, clock = 0, last_dump = 0;
    uint64_t seed, stream, forks = 0;
    int c = 0;
    cudaStream_t st = nullptr, st2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DeviceBuf A, B, GA, GB, A2, B2, sig, hv, work, ws, q1, q2, q3, pib, xs_d, ys_d, gws;
    int batch = 32;         // adaptive speculative batch (rows)
    double fire_ema = 0.0;  // moving average of gate fires (batch pattern prediction)
    CodJob* jobs_d = nullptr;
    int* status_d = nullptr;
    std::deque<CodSnap> snaps;
    // dev instrumentation (AERO_HOST_PROF): wall ms in run() / dumps / reduces
    bool hprof = getenv("AERO_HOST_PROF") != nullptr;
    double t_run = 0, t_dump = 0, t_reduce = 0, t_total = 0, t_eiga = 0, t_eigb = 0, t_eigk = 0;
    int64_t n_run = 0, n_dump = 0, n_reduce = 0, n_rows = 0;
    std::deque<CodChunk*> chunks;  // live chunks, oldest first
    std::vector<CodChunk*> spare;  // emptied chunks kept for reuse
    CodSnap snap_alloc(int xi) {
        if (chunks.empty() || chunks.back()->used + xi > kCodChunkCols) {
            CodChunk* ch;
            if (!spare.empty()) {
                ch = spare.back();
                spare.pop_back();
            } else {
                ch = new CodChunk;
                const size_t nc = kCodChunkCols;
                AERO_CUDA(cudaMalloc(&ch->z, sizeof(double) * dx * nc));
                AERO_CUDA(cudaMalloc(&ch->h, sizeof(double) * dy * nc));
                AERO_CUDA(cudaMalloc(&ch->zm_t, sizeof(double) * dy * nc));
                AERO_CUDA(cudaMalloc(&ch->mh, sizeof(double) * dx * nc));
            }
            ch->used = ch->live = 0;
            chunks.push_back(ch);
        }
        CodChunk* ch = chunks.back();
        const size_t col = (size_t)ch->used;
        ch->used += xi;
        ch->live += xi;
        CodSnap sn{};
        sn.xi = xi;
        sn.chunk = ch;
        sn.z = ch->z + col * dx;
        sn.h = ch->h + col * dy;
        sn.zm_t = ch->zm_t + col * dy;
        sn.mh = ch->mh + col * dx;
        return sn;
    }
    void snap_release(const CodSnap& sn) {
        sn.chunk->live -= sn.xi;
        while (!chunks.empty() && chunks.front()->live == 0 && chunks.front() != chunks.back()) {
            spare.push_back(chunks.front());
            chunks.pop_front();
        }
    }
    void free_chunks() {
        std::vector<CodChunk*> all(chunks.begin(), chunks.end());
        all.insert(all.end(), spare.begin(), spare.end());
        for (CodChunk* ch : all) {
            cudaFree(ch->z);
            cudaFree(ch->h);
            cudaFree(ch->zm_t);
            cudaFree(ch->mh);
            delete ch;
        }
        chunks.clear();
        spare.clear();
    }
    aero_event ev{};

    uint64_t fork_state(uint64_t f) const { return rng_state0(seed, fork_stream(stream, f)); }

    void regram() {  // GA = A^T A, GB = B^T B
        gemm_acc(st, true, false, c, c, dx, 1.0, A.p, dx, A.p, dx, 0.0, GA.p, cap, gws.p, gws.n);
        gemm_acc(st, true, false, c, c, dy, 1.0, B.p, dy, B.p, dy, 0.0, GB.p, cap, gws.p, gws.n);
    }
    // append nb columns (device, contiguous) at c and extend the Grams by the
    // new column block (GA[0:c+nb, c:c+nb] = A^T x_new) and its mirror
    void append(const double* xd, const double* yd, int nb) {
        AERO_CUDA(cudaMemcpyAsync(A.p + (size_t)c * dx, xd, sizeof(double) * dx * nb, cudaMemcpyDeviceToDevice, st));
        AERO_CUDA(cudaMemcpyAsync(B.p + (size_t)c * dy, yd, sizeof(double) * dy * nb, cudaMemcpyDeviceToDevice, st));
        gemm_acc(st, true, false, c + nb, nb, dx, 1.0, A.p, dx, A.p + (size_t)c * dx, dx, 0.0, GA.p + (size_t)c * cap,
                 cap, gws.p, gws.n);
        gemm_acc(st, true, false, c + nb, nb, dy, 1.0, B.p, dy, B.p + (size_t)c * dy, dy, 0.0, GB.p + (size_t)c * cap,
                 cap, gws.p, gws.n);
        if (c > 0) {
            const int64_t tot = (int64_t)c * nb;
            k_cod_mirror<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c, nb, GA.p, cap);
            AERO_LAUNCHED();
            k_cod_mirror<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c, nb, GB.p, cap);
            AERO_LAUNCHED();
        }
        c += nb;
    }

    // run jobs (<= 3) -> sig (host), status (host)
    void run(const CodJob* hj, int nj, double* sig_h, int* status_h) {
        const auto t0 = std::chrono::steady_clock::now();
        struct Acc {
            Impl& s;
            std::chrono::steady_clock::time_point t0;
            ~Acc() {
                if (s.hprof) {
                    s.t_run += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                    s.n_run++;
                }
            }
        } acc{*this, t0};
        AERO_CUDA(cudaMemcpyAsync(jobs_d, hj, sizeof(CodJob) * nj, cudaMemcpyHostToDevice, st));
        const size_t smem = sizeof(double) * (32 + 2 * (size_t)c * COD_KMAX + 3 * COD_KMAX * COD_KMAX +
                                              COD_KMAX + 64 +
                                              (size_t)(COD_MV_PARTS - 1) * (COD_THREADS / COD_MV_PARTS) * COD_KMAX) +
                            16;
        static bool attr = false;
        if (!attr) {
            AERO_CUDA(cudaFuncSetAttribute(k_cod_job, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           100 * 1024));
            attr = true;
        }
        const int64_t pis = (int64_t)std::max(dx, dy) * COD_KMAX;
        pib.alloc((size_t)std::max(nj, 3) * pis);
        k_cod_job<<<nj, COD_THREADS, smem, st>>>(jobs_d, A.p, dx, B.p, dy, GA.p, GB.p, cap, sig.p, hv.p,
                                         status_d, pib.p, pis);
        AERO_LAUNCHED();
        AERO_CUDA(cudaMemcpyAsync(sig_h, sig.p, sizeof(double) * nj * COD_KMAX, cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaMemcpyAsync(status_h, status_d, sizeof(int) * nj, cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaStreamSynchronize(st));
    }

    // cod_reduce (fd.cpp:56-86) in Gram form. With GA = Wa La Wa^T (rank ra),
    // A = Qa Ra, Qa = A Wa La^{-1/2} (orthonormal), Ra = La^{1/2} Wa^T; same for B.
    // The core Ra Rb^T = La^{1/2} (Wa^T Wb) Lb^{1/2} (ra x rb); its SVD u s v^T
    // gives a' = Qa u w, b' = Qb v w with w = sqrt(max(s - s_ell, 0)) (fd.cpp:77-84).
    void cod_reduce() {
        const auto t0 = std::chrono::steady_clock::now();
        struct Acc {
            Impl& s;
            std::chrono::steady_clock::time_point t0;
            ~Acc() {
                if (s.hprof) {
                    cudaStreamSynchronize(s.st);  // destructor: no throw
                    s.t_reduce += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                    s.n_reduce++;
                }
            }
        } acc{*this, t0};
        const int m = c;  // == 2 ell
        q1.alloc((size_t)m * m * 6 + 4 * (size_t)m);
        double* Wa = q1.p;
        double* Wb = Wa + (size_t)m * m;
        double* K = Wb + (size_t)m * m;
        double* T = K + (size_t)m * m;
        double* Ua = T + (size_t)m * m;
        double* Vb = Ua + (size_t)m * m;
        double* la = Vb + (size_t)m * m;
        double* lb = la + m;
        double* ls = lb + m;
        copy_matrix(st, m, m, GA.p, cap, Wa, m);
        copy_matrix(st, m, m, GB.p, cap, Wb, m);
        auto lap = [&](double& acc) {
            if (!hprof) return;
            AERO_CUDA(cudaStreamSynchronize(st));
            static thread_local std::chrono::steady_clock::time_point last;
            const auto now = std::chrono::steady_clock::now();
            acc += std::chrono::duration<double, std::milli>(now - last).count();
            last = now;
        };
        double dummy = 0;
        lap(dummy);
        // the two Gram eigendecompositions are independent: GB's on a second
        // stream, concurrently (each is a latency-bound chain of small launches)
        if (!st2) {
            AERO_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
            AERO_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            AERO_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        AERO_CUDA(cudaEventRecord(ev_fork, st));
        AERO_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
        eigh(st, m, Wa, m, la);
        eigh(st2, m, Wb, m, lb);
        AERO_CUDA(cudaEventRecord(ev_join, st2));
        AERO_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
        lap(t_eiga);
        std::vector<double> ha(m), hb(m);
        AERO_CUDA(cudaMemcpyAsync(ha.data(), la, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaMemcpyAsync(hb.data(), lb, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaStreamSynchronize(st));
        auto rank_of = [&](const std::vector<double>& l) {
            const double lmax = std::max(l[0], 0.0);
            int rk = 0;
            for (int i = 0; i < m; ++i)
                if (l[i] > 1e-10 * lmax && l[i] > 0.0) rk = i + 1;
            return rk;
        };
        const int ra = rank_of(ha), rb = rank_of(hb);
        const int keep = std::max(ell - 1, 1);
        if (ra == 0 || rb == 0) {  // fd.cpp:64-65: a zero factor reduces to zero
            fill_zero(st, A.p, (int64_t)dx * cap);
            fill_zero(st, B.p, (int64_t)dy * cap);
            c = keep;
            regram();
            return;
        }
        std::vector<double> sc((size_t)4 * m, 0.0);  // sa | sb | 1/sa | 1/sb
        for (int i = 0; i < ra; ++i) { sc[i] = std::sqrt(ha[i]); sc[2 * m + i] = 1.0 / sc[i]; }
        for (int i = 0; i < rb; ++i) { sc[m + i] = std::sqrt(hb[i]); sc[3 * m + i] = 1.0 / sc[m + i]; }
        q2.alloc(4 * (size_t)m + 2 * (size_t)keep);
        AERO_CUDA(cudaMemcpyAsync(q2.p, sc.data(), sizeof(double) * 4 * m, cudaMemcpyHostToDevice, st));
        // K = diag(sa) Wa_r^T Wb_r diag(sb)
        dgemm(st, true, false, ra, rb, m, 1.0, Wa, m, Wb, m, 0.0, K, ra);
        scale_rows(st, ra, rb, K, ra, q2.p);
        scale_columns(st, ra, rb, K, ra, q2.p + m);
        // SVD of K via eig(K K^T): u (ra x ra, descending), s^2
        dgemm(st, false, true, ra, ra, rb, 1.0, K, ra, K, ra, 0.0, T, ra);
        lap(dummy);
        eigh(st, ra, T, ra, ls, 1, 0, std::min(ra, keep + 1));  // the kept directions (and the cut)
        lap(t_eigk);
        std::vector<double> hl(ra);
        AERO_CUDA(cudaMemcpyAsync(hl.data(), ls, sizeof(double) * ra, cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaStreamSynchronize(st));
        const int nsv = std::min(ra, rb);
        std::vector<double> sg(nsv);
        for (int i = 0; i < nsv; ++i) sg[i] = std::sqrt(std::max(hl[i], 0.0));
        const double cut = (ell <= nsv) ? sg[ell - 1] : 0.0;
        const int kk = std::min(keep, nsv);
        std::vector<double> wv((size_t)2 * keep, 0.0);  // w | w / s
        for (int i = 0; i < kk; ++i) {
            const double w = std::sqrt(std::max(sg[i] - cut, 0.0));
            wv[i] = w;
            wv[keep + i] = (sg[i] > 0.0) ? w / sg[i] : 0.0;
        }
        AERO_CUDA(cudaMemcpyAsync(q2.p + 4 * m, wv.data(), sizeof(double) * 2 * keep, cudaMemcpyHostToDevice, st));
        // Ua = diag(1/sa) u[:, :kk] diag(w)        (ra x kk)
        copy_matrix(st, ra, kk, T, ra, Ua, ra);
        scale_rows(st, ra, kk, Ua, ra, q2.p + 2 * m);
        scale_columns(st, ra, kk, Ua, ra, q2.p + 4 * m);
        // Vb = diag(1/sb) K^T u[:, :kk] diag(w/s)  (rb x kk)
        dgemm(st, true, false, rb, kk, ra, 1.0, K, ra, T, ra, 0.0, Vb, rb);
        scale_rows(st, rb, kk, Vb, rb, q2.p + 3 * m);
        scale_columns(st, rb, kk, Vb, rb, q2.p + 4 * m + keep);
        // a' = A (Wa_r Ua), b' = B (Wb_r Vb)
        q3.alloc((size_t)m * keep);
        double* tmp = q3.p;
        dgemm(st, false, false, m, kk, ra, 1.0, Wa, m, Ua, ra, 0.0, tmp, m);
        dgemm(st, false, false, dx, kk, m, 1.0, A.p, dx, tmp, m, 0.0, A2.p, dx);
        dgemm(st, false, false, m, kk, rb, 1.0, Wb, m, Vb, rb, 0.0, tmp, m);
        dgemm(st, false, false, dy, kk, m, 1.0, B.p, dy, tmp, m, 0.0, B2.p, dy);
        if (kk < keep) {
            fill_zero(st, A2.p + (size_t)kk * dx, (int64_t)(keep - kk) * dx);
            fill_zero(st, B2.p + (size_t)kk * dy, (int64_t)(keep - kk) * dy);
        }
        std::swap(A.p, A2.p);
        std::swap(A.n, A2.n);
        std::swap(B.p, B2.p);
        std::swap(B.n, B2.n);
        c = keep;
        regram();
    }
};

CodEngine::CodEngine(int dx, int dy, double eps, double theta, int64_t n, uint64_t seed,
                     uint64_t stream, int device)
    : im_(new Impl) {
    if (dx < 1 || dy < 1) {
        delete im_;
        throw InvalidInput("CodState: dimensions must be >= 1");
    }
    if (!(eps > 0.0 && eps <= 1.0)) {
        delete im_;
        throw InvalidInput("CodState: eps out of (0,1]");
    }
    if (theta < 0.0) {
        delete im_;
        throw InvalidInput("CodState: theta must be >= 0");
    }
    if (n < 1) {
        delete im_;
        throw InvalidInput("CodState: window size must be >= 1");
    }
    Impl& s = *im_;
    s.dx = dx;
    s.dy = dy;
    s.eps = eps;
    s.theta = theta;
    s.n = n;
    s.seed = seed;
    s.stream = stream;
    s.dev = device;
    s.ell = static_cast<int>(std::ceil(2.0 / eps));
    s.cap = 2 * s.ell;
    auto pic = [](int b) {
        return static_cast<int>(std::ceil(std::log2(static_cast<double>(std::max(b, 2))))) + 1;
    };
    auto qf = [](int d) {
        return static_cast<int>(std::ceil(std::log2(static_cast<double>(std::max(d, 2))) / 0.4));
    };
    s.kp = pic(s.ell);  // amm.cpp:66 (kp from ell)
    s.qz = qf(dx);      // simul_iter(p): d = rows(p) = dx
    s.qh = qf(dy);      // simul_iter(p^T): d = dy
    AERO_CUDA(cudaSetDevice(device));
    AERO_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    s.A.alloc((size_t)dx * s.cap);
    s.B.alloc((size_t)dy * s.cap);
    s.A2.alloc((size_t)dx * s.cap);
    s.B2.alloc((size_t)dy * s.cap);
    s.GA.alloc((size_t)s.cap * s.cap);
    s.GB.alloc((size_t)s.cap * s.cap);
    s.sig.alloc((size_t)COD_MAX_BATCH * COD_KMAX);
    s.hv.alloc((size_t)COD_MAX_BATCH * s.cap * COD_KMAX);
    s.gws.alloc((size_t)8 * s.cap * COD_MAX_BATCH);
    AERO_CUDA(cudaMalloc(&s.jobs_d, sizeof(CodJob) * COD_MAX_BATCH));
    AERO_CUDA(cudaMalloc(&s.status_d, sizeof(int) * COD_MAX_BATCH));
}

CodEngine::~CodEngine() {
    if (!im_) return;
    cudaSetDevice(im_->dev);
    if (im_->st) cudaStreamSynchronize(im_->st);
    if (im_->hprof && im_->n_rows > 0)
        fprintf(stderr, "cod host: %lld rows %.1f ms total | run %.1f ms (%lld calls) | dumps %.1f ms (%lld) | reduces %.1f ms (%lld): eig GA %.1f GB %.1f core %.1f\n",
                (long long)im_->n_rows, im_->t_total, im_->t_run, (long long)im_->n_run, im_->t_dump,
                (long long)im_->n_dump, im_->t_reduce, (long long)im_->n_reduce, im_->t_eiga, im_->t_eigb,
                im_->t_eigk);
    im_->free_chunks();
    cudaFree(im_->jobs_d);
    cudaFree(im_->status_d);
    if (im_->st) {
        eigh_forget(im_->st);
        cudaStreamDestroy(im_->st);
    }
    if (im_->st2) {
        cudaStreamSynchronize(im_->st2);
        eigh_forget(im_->st2);
        cudaStreamDestroy(im_->st2);
        cudaEventDestroy(im_->ev_fork);
        cudaEventDestroy(im_->ev_join);
    }
    delete im_;
}

// amm.cpp:42-103. Rows are applied in speculative batches: the columns of a
// batch are appended at once (Gram column block by one GEMM), the gates of all
// its rows run as one launch (row j's gate sees the buffer prefix c0 + j + 1
// and fork F + j + 1, exactly what it would see one row at a time if no
// earlier row of the batch fired). The first row whose gate fires is finished
// exactly (paired simul_iter, doubling, dump) and ends the batch; the row that
// fills the buffer (reduce before its gate) always runs alone.
void CodEngine::update_block(const double* xs, const double* ys, int64_t nrows, const int64_t* t,
                             aero_event* log) {
    Impl& s = *im_;
    AERO_CUDA(cudaSetDevice(s.dev));
    if (nrows <= 0) return;
    const auto tu0 = std::chrono::steady_clock::now();
    struct AccU {
        Impl& s;
        std::chrono::steady_clock::time_point t0;
        int64_t n;
        ~AccU() {
            if (s.hprof) {
                s.t_total += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                s.n_rows += n;
            }
        }
    } accu{s, tu0, nrows};
    int64_t good = nrows;
    std::string err;
    int64_t prev = s.clock;
    for (int64_t q = 0; q < nrows && err.empty(); ++q) {
        for (int j = 0; j < s.dx && err.empty(); ++j)
            if (!std::isfinite(xs[q * s.dx + j])) err = "CodState: non-finite input";
        for (int j = 0; j < s.dy && err.empty(); ++j)
            if (!std::isfinite(ys[q * s.dy + j])) err = "CodState: non-finite input";
        if (err.empty() && t[q] <= prev) err = "CodState: timestamp regression";
        if (!err.empty()) good = q;
        prev = t[q];
    }
    if (good > 0) {
        s.xs_d.alloc((size_t)good * s.dx);
        s.ys_d.alloc((size_t)good * s.dy);
        AERO_CUDA(cudaMemcpyAsync(s.xs_d.p, xs, sizeof(double) * good * s.dx, cudaMemcpyHostToDevice, s.st));
        AERO_CUDA(cudaMemcpyAsync(s.ys_d.p, ys, sizeof(double) * good * s.dy, cudaMemcpyHostToDevice, s.st));
    }
    std::vector<double> sig_h((size_t)COD_MAX_BATCH * COD_KMAX);
    std::vector<int> status_h(COD_MAX_BATCH);
    std::vector<CodJob> jobs(COD_MAX_BATCH);

    auto expire = [&](int64_t i) {  // amm.cpp:48
        while (!s.snaps.empty() && s.snaps.front().t + s.n <= i) {
            s.snap_release(s.snaps.front());
            s.snaps.pop_front();
        }
    };
    // the gate fired (amm.cpp:72-101): paired simul_iter with doubling, dump
    // pre: results of the first (k = min(2, kmax)) simul pair when the batch
    // already ran it (z sigma_hat, z status, z / h c-space bases), else null
    auto fired = [&](int64_t i, aero_event& ev, const double* pre_sz, int pre_stz, const double* pre_hvz,
                     const double* pre_hvh) {
        double sig[3 * COD_KMAX];
        int status[3];
        ev.gate_fired = 1;
        const int kmax = std::min({s.ell, s.dx, s.dy, s.c});
        int k = std::min(2, kmax);
        bool have = pre_sz != nullptr;
        while (true) {
            ev.doubling_steps++;
            ev.simul_calls += 2;
            if (k > COD_KMAX) throw InvalidInput("CodState: rank beyond the in-kernel limit");
            const double* sz;  // z side sigma_hat
            const double* hvz;
            const double* hvh;
            int stz;
            if (have) {
                sz = pre_sz;
                stz = pre_stz;
                hvz = pre_hvz;
                hvh = pre_hvh;
                have = false;
            } else {
                CodJob jz{1, s.c, k, s.qz, s.fork_state(++s.forks)};
                CodJob jh{2, s.c, k, s.qh, s.fork_state(++s.forks)};
                CodJob js[2] = {jz, jh};
                s.run(js, 2, sig, status);
                sz = sig;
                stz = status[0];
                hvz = s.hv.p;
                hvh = s.hv.p + (size_t)s.cap * COD_KMAX;
            }
            ev.k_last = k;
            ev.tail_sq = sz[k - 1];
            if (sz[k - 1] < s.theta || k == kmax) {
                int xi = 0;
                for (int j = 0; j < k; ++j) {
                    if (sz[j] >= s.theta) xi = j + 1;
                    else break;
                }
                ev.xi = xi;
                if (xi >= 1) {
                    const auto td0 = std::chrono::steady_clock::now();
                    CodSnap sn = s.snap_alloc(xi);
                    if (stz == JOB_ZERO) {
                        std::vector<double> I((size_t)s.dx * xi, 0.0), J((size_t)s.dy * xi, 0.0);
                        for (int j = 0; j < xi; ++j) {
                            if (j < s.dx) I[j + (size_t)j * s.dx] = 1.0;
                            if (j < s.dy) J[j + (size_t)j * s.dy] = 1.0;
                        }
                        AERO_CUDA(cudaMemcpyAsync(sn.z, I.data(), sizeof(double) * I.size(), cudaMemcpyHostToDevice, s.st));
                        AERO_CUDA(cudaMemcpyAsync(sn.h, J.data(), sizeof(double) * J.size(), cudaMemcpyHostToDevice, s.st));
                        AERO_CUDA(cudaStreamSynchronize(s.st));
                    } else {
                        dgemm(s.st, false, false, s.dx, xi, s.c, 1.0, s.A.p, s.dx, hvz, s.cap, 0.0, sn.z, s.dx);
                        dgemm(s.st, false, false, s.dy, xi, s.c, 1.0, s.B.p, s.dy, hvh, s.cap, 0.0, sn.h, s.dy);
                        fix_column_signs(s.st, s.dx, xi, sn.z, s.dx, nullptr);
                        fix_column_signs(s.st, s.dy, xi, sn.h, s.dy, nullptr);
                    }
                    // zm = z^T p = (z^T A) B^T ; mh = p h = A (B^T h)   (amm.cpp:87-88)
                    s.work.alloc((size_t)2 * s.cap * xi + 64);
                    double* zA = s.work.p;                 // xi x c (ld xi)
                    double* Bh = zA + (size_t)s.cap * xi;  // c x xi (ld cap)
                    dgemm(s.st, true, false, xi, s.c, s.dx, 1.0, sn.z, s.dx, s.A.p, s.dx, 0.0, zA, xi);
                    dgemm(s.st, true, false, s.c, xi, s.dy, 1.0, s.B.p, s.dy, sn.h, s.dy, 0.0, Bh, s.cap);
                    dgemm(s.st, false, true, s.dy, xi, s.c, 1.0, s.B.p, s.dy, zA, xi, 0.0, sn.zm_t, s.dy);
                    dgemm(s.st, false, false, s.dx, xi, s.c, 1.0, s.A.p, s.dx, Bh, s.cap, 0.0, sn.mh, s.dx);
                    // A -= z (z^T A), B -= h (h^T B)   (amm.cpp:92-93)
                    dgemm(s.st, false, false, s.dx, s.c, xi, -1.0, sn.z, s.dx, zA, xi, 1.0, s.A.p, s.dx);
                    dgemm(s.st, true, false, xi, s.c, s.dy, 1.0, sn.h, s.dy, s.B.p, s.dy, 0.0, zA, xi);
                    dgemm(s.st, false, false, s.dy, s.c, xi, -1.0, sn.h, s.dy, zA, xi, 1.0, s.B.p, s.dy);
                    s.regram();
                    sn.s = s.last_dump + 1;
                    sn.t = i;
                    s.last_dump = i;
                    s.snaps.push_back(sn);
                    ev.dumped = 1;
                    if (s.hprof) {
                        AERO_CUDA(cudaStreamSynchronize(s.st));
                        s.t_dump += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - td0).count();
                        s.n_dump++;
                    }
                }
                break;
            }
            k = std::min(2 * k, kmax);
        }
    };
    auto finish = [&](int64_t q, aero_event& ev) {
        s.clock = t[q];
        ev.forks_after = (int64_t)s.forks;
        ev.rows_after = s.c;
        s.ev = ev;
        if (log) log[q] = ev;
    };

    int64_t q = 0;
    while (q < good) {
        const int room = s.cap - s.c;
        const int nb = (int)std::min<int64_t>({(int64_t)s.batch, good - q, (int64_t)room - 1});
        if (nb <= 0) {  // this row fills the buffer: append, reduce, then its gate
            const int64_t i = t[q];
            aero_event ev{};
            ev.t = i;
            ev.theta = s.theta;
            ev.forks_before = (int64_t)s.forks;
            expire(i);
            s.append(s.xs_d.p + (size_t)q * s.dx, s.ys_d.p + (size_t)q * s.dy, 1);
            if (s.c == s.cap) {  // amm.cpp:56-62
                s.cod_reduce();
                ev.reduced = 1;
            }
            CodJob gj{0, s.c, 1, s.kp, s.fork_state(++s.forks)};
            s.run(&gj, 1, sig_h.data(), status_h.data());
            const double s1sq = (status_h[0] == JOB_ACTIVE) ? sig_h[0] : 0.0;
            ev.sigma1_sq = s1sq;
            if (!(std::sqrt(s1sq) < 0.5 * s.theta)) fired(i, ev, nullptr, 0, nullptr, nullptr);
            s.fire_ema = 0.9 * s.fire_ema + 0.1 * ev.gate_fired;
            finish(q, ev);
            ++q;
            continue;
        }
        if (s.fire_ema > 0.5) {  // FIRE1 prediction: gate fires, one k = 2 pair, no dump
            const int c0 = s.c;
            const uint64_t F = s.forks;
            const int nbf = std::min(nb, COD_MAX_BATCH / 3);
            s.append(s.xs_d.p + (size_t)q * s.dx, s.ys_d.p + (size_t)q * s.dy, nbf);
            for (int j = 0; j < nbf; ++j) {
                const int cj = c0 + j + 1;
                const int kj = std::min({2, s.ell, s.dx, s.dy, cj});
                jobs[3 * j] = CodJob{0, cj, 1, s.kp, s.fork_state(F + 3 * j + 1)};
                jobs[3 * j + 1] = CodJob{1, cj, kj, s.qz, s.fork_state(F + 3 * j + 2)};
                jobs[3 * j + 2] = CodJob{2, cj, kj, s.qh, s.fork_state(F + 3 * j + 3)};
            }
            s.run(jobs.data(), 3 * nbf, sig_h.data(), status_h.data());
            int j = 0;
            bool deviated = false;
            for (; j < nbf && !deviated; ++j) {
                const int64_t i = t[q + j];
                aero_event ev{};
                ev.t = i;
                ev.theta = s.theta;
                ev.forks_before = (int64_t)(F + 3 * j);
                expire(i);
                s.c = c0 + j + 1;
                s.forks = F + 3 * j + 1;
                const double s1sq = (status_h[3 * j] == JOB_ACTIVE) ? sig_h[(size_t)3 * j * COD_KMAX] : 0.0;
                ev.sigma1_sq = s1sq;
                if (!(std::sqrt(s1sq) < 0.5 * s.theta)) {
                    s.forks = F + 3 * j + 3;  // the pair of this row ran in the batch
                    const double* sz = sig_h.data() + (size_t)(3 * j + 1) * COD_KMAX;
                    const int kmax = std::min({s.ell, s.dx, s.dy, s.c});
                    const int k = std::min(2, kmax);
                    const bool settled = sz[k - 1] < s.theta || k == kmax;
                    if (!settled || sz[0] >= s.theta) deviated = true;  // doubling or a dump ends the batch
                    fired(i, ev, sz, status_h[3 * j + 1], s.hv.p + (size_t)(3 * j + 1) * s.cap * COD_KMAX,
                          s.hv.p + (size_t)(3 * j + 2) * s.cap * COD_KMAX);
                } else {
                    deviated = true;  // predicted fire, gate stayed quiet: later forks shift
                }
                s.fire_ema = 0.9 * s.fire_ema + 0.1 * ev.gate_fired;
                finish(q + j, ev);
            }
            q += j;
            s.batch = deviated ? std::max(4, 2 * j) : std::min(COD_MAX_BATCH, 2 * s.batch);
            continue;
        }
        const int c0 = s.c;
        const uint64_t F = s.forks;
        s.append(s.xs_d.p + (size_t)q * s.dx, s.ys_d.p + (size_t)q * s.dy, nb);
        for (int j = 0; j < nb; ++j) jobs[j] = CodJob{0, c0 + j + 1, 1, s.kp, s.fork_state(F + j + 1)};
        s.run(jobs.data(), nb, sig_h.data(), status_h.data());
        int fire = -1;
        for (int j = 0; j < nb && fire < 0; ++j) {
            const double s1sq = (status_h[j] == JOB_ACTIVE) ? sig_h[(size_t)j * COD_KMAX] : 0.0;
            if (!(std::sqrt(s1sq) < 0.5 * s.theta)) fire = j;
        }
        const int ncommit = (fire < 0) ? nb : fire + 1;
        for (int j = 0; j < ncommit; ++j) {
            const int64_t i = t[q + j];
            aero_event ev{};
            ev.t = i;
            ev.theta = s.theta;
            ev.forks_before = (int64_t)(F + j);
            expire(i);
            s.c = c0 + j + 1;
            s.forks = F + j + 1;
            ev.sigma1_sq = (status_h[j] == JOB_ACTIVE) ? sig_h[(size_t)j * COD_KMAX] : 0.0;
            if (j == fire) fired(i, ev, nullptr, 0, nullptr, nullptr);
            s.fire_ema = 0.9 * s.fire_ema + 0.1 * ev.gate_fired;
            finish(q + j, ev);
        }
        q += ncommit;
        s.batch = (fire < 0) ? std::min(COD_MAX_BATCH, 2 * s.batch) : std::max(4, 2 * (fire + 1));
    }
    AERO_CUDA(cudaStreamSynchronize(s.st));
    if (good < nrows) throw InvalidInput(err);
}

// amm.cpp:105-114: p = A B^T + sum of cod_restore_contribution (amm.cpp:22-25)
void CodEngine::query_product(double* p_host) {
    Impl& s = *im_;
    AERO_CUDA(cudaSetDevice(s.dev));
    s.q3.alloc((size_t)s.dx * s.dy + 64 * (size_t)s.dx);
    double* P = s.q3.p;
    fill_zero(s.st, P, (int64_t)s.dx * s.dy);
    if (s.c > 0) dgemm(s.st, false, true, s.dx, s.dy, s.c, 1.0, s.A.p, s.dx, s.B.p, s.dy, 0.0, P, s.dx);
    for (const CodSnap& sn : s.snaps) {
        // z zm + mh h^T - z (zm h) h^T
        dgemm(s.st, false, true, s.dx, s.dy, sn.xi, 1.0, sn.z, s.dx, sn.zm_t, s.dy, 1.0, P, s.dx);
        dgemm(s.st, false, true, s.dx, s.dy, sn.xi, 1.0, sn.mh, s.dx, sn.h, s.dy, 1.0, P, s.dx);
        s.work.alloc((size_t)sn.xi * sn.xi + (size_t)s.dx * sn.xi + 64);
        double* K = s.work.p;
        double* zK = K + (size_t)sn.xi * sn.xi;
        dgemm(s.st, true, false, sn.xi, sn.xi, s.dy, 1.0, sn.zm_t, s.dy, sn.h, s.dy, 0.0, K, sn.xi);
        dgemm(s.st, false, false, s.dx, sn.xi, sn.xi, 1.0, sn.z, s.dx, K, sn.xi, 0.0, zK, s.dx);
        dgemm(s.st, false, true, s.dx, s.dy, sn.xi, -1.0, zK, s.dx, sn.h, s.dy, 1.0, P, s.dx);
    }
    if (p_host) {
        std::vector<double> cm((size_t)s.dx * s.dy);
        AERO_CUDA(cudaMemcpyAsync(cm.data(), P, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost, s.st));
        AERO_CUDA(cudaStreamSynchronize(s.st));
        for (int i = 0; i < s.dx; ++i)
            for (int j = 0; j < s.dy; ++j) p_host[(size_t)i * s.dy + j] = cm[i + (size_t)j * s.dx];
    }
}

// amm.cpp:115-121: SVD of the restored p, shrink by sigma_ell
void CodEngine::query(double* astar, double* bstar) {
    Impl& s = *im_;
    query_product(nullptr);
    const int dx = s.dx, dy = s.dy, ell = s.ell;
    const double* P = s.q3.p;
    // eig(p^T p) (dy x dy) -> v, sigma^2 ; u = p v / sigma
    s.q1.alloc((size_t)dy * dy + dy + (size_t)dx * dy);
    double* V = s.q1.p;
    double* lam = V + (size_t)dy * dy;
    double* U = lam + dy;
    dgemm(s.st, true, false, dy, dy, dx, 1.0, P, dx, P, dx, 0.0, V, dy);
    eigh(s.st, dy, V, dy, lam);
    dgemm(s.st, false, false, dx, dy, dy, 1.0, P, dx, V, dy, 0.0, U, dx);
    std::vector<double> hl(dy), hV((size_t)dy * dy), hU((size_t)dx * dy);
    AERO_CUDA(cudaMemcpyAsync(hl.data(), lam, sizeof(double) * dy, cudaMemcpyDeviceToHost, s.st));
    AERO_CUDA(cudaMemcpyAsync(hV.data(), V, sizeof(double) * hV.size(), cudaMemcpyDeviceToHost, s.st));
    AERO_CUDA(cudaMemcpyAsync(hU.data(), U, sizeof(double) * hU.size(), cudaMemcpyDeviceToHost, s.st));
    AERO_CUDA(cudaStreamSynchronize(s.st));
    const int nsv = std::min(dx, dy);
    std::vector<double> sg(nsv);
    for (int i = 0; i < nsv; ++i) sg[i] = std::sqrt(std::max(hl[i], 0.0));
    const double cut = (ell <= nsv) ? sg[ell - 1] : 0.0;
    for (int j = 0; j < ell; ++j) {
        const double w = (j < nsv) ? std::sqrt(std::max(sg[j] - cut, 0.0)) : 0.0;
        for (int i = 0; i < dx; ++i)
            astar[(size_t)i * ell + j] = (w > 0.0 && sg[j] > 0.0) ? w * hU[i + (size_t)j * dx] / sg[j] : 0.0;
        for (int i = 0; i < dy; ++i)
            bstar[(size_t)i * ell + j] = (w > 0.0) ? w * hV[i + (size_t)j * dy] : 0.0;
    }
}

void CodEngine::info(int32_t* ell, int64_t* cols, int64_t* snaps, int64_t* clock) const {
    if (ell) *ell = im_->ell;
    if (cols) *cols = im_->c;
    if (snaps) *snaps = (int64_t)im_->snaps.size();
    if (clock) *clock = im_->clock;
}

double CodEngine::theta() const { return im_->theta; }
void CodEngine::set_theta(double theta) {
    if (theta < 0.0) throw InvalidInput("CodState: theta must be >= 0");
    im_->theta = theta;
}
int64_t CodEngine::window() const { return im_->n; }
int64_t CodEngine::snap_count() const { return (int64_t)im_->snaps.size(); }
int64_t CodEngine::snap_t(int64_t idx) const { return im_->snaps[(size_t)idx].t; }

// ============================================================================
// AdaptiveState
// ============================================================================
// amm.cpp:131-138: main_ takes the constructor rng's first fork, aux_ its
// second; rng_ keeps the parent (forks = 2) for the boundary re-creations.
AdaptiveEngine::AdaptiveEngine(int dx, int dy, double eps, double theta0, int64_t n, uint64_t seed,
                               uint64_t stream, int device)
    : dx_(dx), dy_(dy), dev_(device), eps_(eps), n_(n), seed_(seed), stream_(stream) {
    main_ = std::make_unique<CodEngine>(dx, dy, eps, theta0, n, seed, fork_stream(stream, ++forks_), device);
    aux_ = std::make_unique<CodEngine>(dx, dy, eps, theta0, n, seed, fork_stream(stream, ++forks_), device);
    if (theta0 <= 0.0) throw InvalidInput("AdaptiveState: theta0 must be > 0");
}

// amm.cpp:140-159, one chunk of rows at a time. A chunk [q, e) starts at a
// window boundary or right after an adaptation check and ends
//  * before the next boundary row (the swap precedes that row's update),
//  * at the first row where the main queue could reach level/eps: it grows by
//    at most one snapshot per row (one dump per update),
//  * at the first row where it could fall to (level-1)/eps: the queue never
//    holds fewer than the already-queued snapshots still inside the window.
// Only the chunk's last row can therefore trigger the rule, which is applied
// once after it exactly as after every row of the reference.
void AdaptiveEngine::update_block(const double* xs, const double* ys, int64_t nrows, const int64_t* t,
                                  aero_event* log, int32_t* level_out) {
    int64_t q = 0;
    while (q < nrows) {
        const int64_t i = t[q];
        if (i > 1 && (i % n_) == 1) {  // amm.cpp:143-146: aux becomes main
            const double th = aux_->theta();
            main_ = std::move(aux_);
            aux_ = std::make_unique<CodEngine>(dx_, dy_, eps_, th, n_, seed_, fork_stream(stream_, ++forks_), dev_);
        }
        const int64_t qlen0 = main_->snap_count();
        const double up = static_cast<double>(level_) / eps_;
        const double down = static_cast<double>(level_ - 1) / eps_;
        int64_t e = q + 1, first_live = 0;
        for (; e < nrows; ++e) {
            const int64_t j = e - 1;  // row j is inside the chunk; may row e join it?
            const int64_t tr = t[e];
            if (tr > 1 && (tr % n_) == 1) break;                       // boundary before row e
            if (static_cast<double>(qlen0 + (j - q + 1)) >= up) break;  // row j may reach `up`
            if (level_ > 1) {  // queued snapshots still live after row j (t_s + n > t_j)
                while (first_live < qlen0 && main_->snap_t(first_live) + n_ <= t[j]) ++first_live;
                if (static_cast<double>(qlen0 - first_live) <= down) break;
            }
        }
        try {
            main_->update_block(xs + q * dx_, ys + q * dy_, e - q, t + q, log ? log + q : nullptr);
        } catch (...) {
            // the reference's aux_ saw every row before the failing one
            // (amm.cpp:147-148); no row before it was an adaptation point
            int64_t clk = 0, good = 0;
            main_->info(nullptr, nullptr, nullptr, &clk);
            while (q + good < e && t[q + good] <= clk) ++good;
            if (good > 0) aux_->update_block(xs + q * dx_, ys + q * dy_, good, t + q, nullptr);
            if (level_out)
                for (int64_t r = q; r < q + good; ++r) level_out[r] = level_;
            throw;
        }
        aux_->update_block(xs + q * dx_, ys + q * dy_, e - q, t + q, nullptr);
        const int lv0 = level_;
        const double qlen = static_cast<double>(main_->snap_count());
        if (qlen >= up) {
            ++level_;
            main_->set_theta(2.0 * main_->theta());
            aux_->set_theta(2.0 * aux_->theta());
        } else if (level_ > 1 && qlen <= down) {
            --level_;
            main_->set_theta(0.5 * main_->theta());
            aux_->set_theta(0.5 * aux_->theta());
        }
        if (level_out) {
            for (int64_t r = q; r + 1 < e; ++r) level_out[r] = lv0;
            level_out[e - 1] = level_;
        }
        q = e;
    }
}

}  // namespace aero_b200
