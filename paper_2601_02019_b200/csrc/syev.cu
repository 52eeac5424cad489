// Symmetric eigensolver for n > kSmallEigMax (the FD reduce at C2: n = 2ell =
// 2048; C3/C5: 256; C4: 512; query shrink: n = d). Replaces the reference's
// Eigen SelfAdjointEigenSolver / BDCSVD (linalg.cpp:48-76) on the device:
//
//  1. k_sytrd   -- Householder tridiagonalization Q^T A Q = T in ONE persistent
//                  cooperative kernel: LAPACK-style blocked panels (dlatrd
//                  recurrence, 32 columns) with a grid barrier per phase; the
//                  panel symv reads whole columns of the symmetric trailing
//                  block (coalesced, L2-resident), the syr2k trailing update
//                  runs as 64x64 register tiles over the lower triangle and is
//                  mirrored, so both triangles stay current.
//  2. k_bisect  -- all eigenvalues of T by 33-way multisection (one warp per
//                  eigenvalue, Sturm counts per lane).
//  3. k_twisted -- eigenvectors of T for the top `nvec` eigenvalues from a
//                  twisted LDL^T/UDU^T factorization (one thread per vector,
//                  row-interleaved scratch so the qd sweeps coalesce), then
//                  Gram-Schmidt (twice) inside tight clusters.
//  4. back-transform Z = Q Y with compact-WY blocks of 128 reflectors
//                  (T factor per block, three fp64 GEMMs on the product engine).
// Output convention of eigh(): eigenvalues descending, eigenvector columns
// sign-fixed so the largest-magnitude entry is positive (linalg.cpp:17-26).
#include <cooperative_groups.h>
#include <cuda/atomic>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cfloat>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "aero_common.cuh"
#include "kernels.cuh"
#include "sketch.hpp"  // DeviceBuf

namespace aero_b200 {

namespace {
constexpr int TRD_NB = 32;        // panel width (reflectors per panel)
constexpr int TRD_THREADS = 256;  // 8 warps
constexpr int TRD_TILE = 64;      // trailing-update tile
constexpr int SLOTW = 4;          // doubles per CTA partial slot
constexpr int BT_NB = 128;        // reflectors per back-transform block
constexpr int TRD_DSPLIT = 4;     // warps per panel dot product

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fixed-order block sum (deterministic for a fixed block size)
__device__ double block_sum_d(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
}

// sum of slot field f over all CTAs in a fixed order (every thread gets it)
__device__ double slots_sum(const double* slots, int f, int G, double* red) {
    double v = 0.0;
    if (threadIdx.x < 32) {
        for (int c = threadIdx.x; c < G; c += 32) v += __ldcg(slots + c * SLOTW + f);
        v = warp_sum_d(v);
        if (threadIdx.x == 0) red[32] = v;
    }
    __syncthreads();
    const double s = red[32];
    __syncthreads();
    return s;
}

constexpr int TRD_NW = TRD_THREADS / 32;

struct TrdArgs {
    int n, lda;
    double* A;  // n x n symmetric, both triangles current (overwritten)
    double* V;  // n x n explicit reflectors (ld n, zero-initialized): column j = v_j, v_j[j+1] = 1
    double* W;  // n x TRD_NB panel W (ld n)
    double *d, *e, *tau;
    double *ybuf, *wpre, *y0, *slots, *dots;
    unsigned* bar;
    unsigned long long* prof;  // optional per-phase ns accumulators (CTA 0, dev instrumentation)
};


// LAPACK dsytrd (lower) with the dlatrd panel recurrence and dlarfg reflectors,
// restated for a persistent grid with TWO grid barriers per column: every CTA
// rebuilds the next column (and its reflector) redundantly in shared memory
// from the published partial column y0, so no barrier is spent on the norm,
// and every row-local input is prefetched before the barrier that precedes
// its use (the kernel is L2-latency bound; each phase is one load round).
//  per column j (panel i0, jj = j - i0):
//   R   (all CTAs) beta, tau, v from the column in sx           -> sv[cur]
//   B   y = A(j+1:, j+1:) v (warp per column, 16 B loads), dots V^T v, W^T v;
//       own rows: V(r, k), W(r, k) into registers, panel part of y0
//   -- barrier --
//   C   own rows: w = tau (y - W V^T v - V W^T v); partial w.v; y0
//   -- barrier --
//   A'  alpha2 = -tau/2 w.v; W(:, jj) = w + alpha2 v; x' = y0 - v (w_{j+1} + 2 alpha2)
// W(:, jj) reaches global memory without a barrier before the next column,
// so that column evaluates it as wpre + alpha2 v_prev wherever it needs it.
template <bool VEC>
__global__ void __launch_bounds__(TRD_THREADS, 1) k_sytrd(TrdArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int n = a.n, G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int gw = cta * TRD_NW + warp, GW = G * TRD_NW;
    const int gwi = warp * G + cta;          // CTA-interleaved warp index (row phases)
    const int sub = lane & 7, grp = lane >> 3;  // 8 lanes per row, 4 rows per warp
    const int lda = a.lda;
    const int npad = (n + 3) & ~1;
    double* red = sm;                          // 64
    double* sx = sm + 64;                      // npad: column being reduced, sx[r - j]
    double* svb = sx + npad;                   // 2 x npad: reflectors (ping-pong), sv[c - c0]
    double* srow = svb + 2 * npad;             // 2 * TRD_NB: W(j+1, k) | V(j+1, i0 + k)
    double* sdot = srow + 2 * TRD_NB;          // 2 * TRD_NB: V^T v | W^T v
    double* tl = sdot + 2 * TRD_NB;            // 4 * TRD_TILE * TRD_NB
    double* A = a.A;
    double* V = a.V;
    double* W = a.W;
    unsigned epoch = 0;
    int cur = 0;
    double a2prev = 0.0;  // alpha2 of the previous column (same panel)
    int c0prev = 0;
    double s2p = 0.0;     // this thread's part of ||x[2:]||^2 for the column in sx
    unsigned long long tp = clock64();
#define TRD_MARK(i)                                                   \
    if (a.prof && cta == 0 && tid == 0) {                             \
        const unsigned long long t_ = clock64();                      \
        a.prof[i] += t_ - tp;                                         \
        tp = t_;                                                      \
    }

    for (int r = tid; r < n; r += TRD_THREADS) {  // column 0
        const double x = A[r];
        sx[r] = x;
        if (r >= 2) s2p += x * x;
    }

    for (int i0 = 0; i0 < n - 1; i0 += TRD_NB) {
        const int jb = min(TRD_NB, n - 1 - i0);
        for (int jj = 0; jj < jb; ++jj) {
            const int j = i0 + jj;
            const int m = n - j - 1;  // reflector length: rows j+1 .. n-1
            const bool nxt = jj + 1 < jb;
            // ---- R: reflector (dlarfg) from sx, identical in every CTA
            const double s2 = block_sum_d(s2p, red);
            const double alpha = sx[1];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (s2 > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + s2), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            const int c0 = (j + 1) & ~1;
            double* sv = svb + cur * npad;
            const double* svo = svb + (cur ^ 1) * npad;  // previous reflector (index c - c0prev)
            for (int c = c0 + tid; c < n + 1; c += TRD_THREADS) {
                const int i = c - (j + 1);
                sv[c - c0] = (c >= n || i < 0) ? 0.0 : (i == 0 ? 1.0 : sx[i + 1] * scal);
            }
            if (cta == 0 && tid == 0) {
                a.d[j] = sx[0];
                a.e[j] = beta;
                a.tau[j] = tau;
            }
            __syncthreads();
            if (cta == 0)
                for (int i = tid; i < m; i += TRD_THREADS) V[j + 1 + i + (int64_t)j * n] = sv[j + 1 + i - c0];
            TRD_MARK(0);

            // ---- B: symv on the panel-start trailing block + panel dots
            if (tau != 0.0) {
                const int len = n - c0;
                for (int r = j + 1 + gw; r < n; r += GW) {
                    const double* col = A + (int64_t)r * lda + c0;
                    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
                    if (VEC) {  // 16 x 16 B loads in flight per lane (two L2 round trips per n=2048 column)
                        const double2* c2 = reinterpret_cast<const double2*>(col);
                        const double2* v2 = reinterpret_cast<const double2*>(sv);
                        const int np = len >> 1;
                        for (int p0 = 0; p0 < np; p0 += 32 * 16) {
                            double2 x[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const int idx = p0 + lane + 32 * u;
                                x[u] = (idx < np) ? __ldcg(c2 + idx) : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int u = 0; u < 16; u += 4) {
#pragma unroll
                                for (int w = 0; w < 4; ++w) {
                                    const int idx = p0 + lane + 32 * (u + w);
                                    const double2 y = (idx < np) ? v2[idx] : make_double2(0.0, 0.0);
                                    double& acc = (w == 0) ? acc0 : (w == 1) ? acc1 : (w == 2) ? acc2 : acc3;
                                    acc = fma(x[u + w].x, y.x, fma(x[u + w].y, y.y, acc));
                                }
                            }
                        }
                        if ((len & 1) && lane == 0) acc1 = fma(col[len - 1], sv[len - 1], acc1);
                    } else {
                        int c = lane;
                        for (; c + 96 < len; c += 128) {
                            acc0 = fma(col[c], sv[c], acc0);
                            acc1 = fma(col[c + 32], sv[c + 32], acc1);
                            acc2 = fma(col[c + 64], sv[c + 64], acc2);
                            acc3 = fma(col[c + 96], sv[c + 96], acc3);
                        }
                        for (; c < len; c += 32) acc0 = fma(col[c], sv[c], acc0);
                    }
                    const double acc = warp_sum_d((acc0 + acc1) + (acc2 + acc3));
                    if (lane == 0) a.ybuf[r] = acc;
                }
                // panel dots, each split over TRD_DSPLIT warps (contiguous row
                // quarters; the consumer sums the parts in fixed order)
                for (int qq = GW - 1 - gw; qq < 2 * jj * TRD_DSPLIT; qq += GW) {
                    const int q = qq / TRD_DSPLIT, part = qq % TRD_DSPLIT;
                    const int span = (n - j - 1 + TRD_DSPLIT - 1) / TRD_DSPLIT;
                    const int cs = j + 1 + part * span, ce = min(n, cs + span);
                    double acc0 = 0.0, acc1 = 0.0;
                    if (q < jj) {  // V(:, i0+q)^T v
                        const double* col = V + (int64_t)(i0 + q) * n;
                        for (int c = cs + lane; c < ce; c += 64) {
                            acc0 = fma(__ldcg(col + c), sv[c - c0], acc0);
                            if (c + 32 < ce) acc1 = fma(__ldcg(col + c + 32), sv[c + 32 - c0], acc1);
                        }
                    } else if (q - jj < jj - 1) {  // W(:, k)^T v, final columns
                        const double* col = W + (int64_t)(q - jj) * n;
                        for (int c = cs + lane; c < ce; c += 64) {
                            acc0 = fma(__ldcg(col + c), sv[c - c0], acc0);
                            if (c + 32 < ce) acc1 = fma(__ldcg(col + c + 32), sv[c + 32 - c0], acc1);
                        }
                    } else {  // W(:, jj-1) = wpre + alpha2 v_prev
                        for (int c = cs + lane; c < ce; c += 32)
                            acc0 = fma(__ldcg(a.wpre + c) + a2prev * svo[c - c0prev], sv[c - c0], acc0);
                    }
                    const double acc = warp_sum_d(acc0 + acc1);
                    if (lane == 0) a.dots[qq] = acc;
                }
            }
            // own-row panel values (final before this column) and the panel part of y0
            const int r = j + 1 + 4 * gwi + grp;
            const bool valid = r < n;
            double pv[4], pw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = sub + 8 * u;
                pv[u] = 0.0;
                pw[u] = 0.0;
                if (valid && k < jj) {
                    pv[u] = __ldcg(V + r + (int64_t)(i0 + k) * n);
                    pw[u] = (k == jj - 1) ? __ldcg(a.wpre + r) + a2prev * svo[r - c0prev]
                                          : __ldcg(W + r + (int64_t)k * n);
                }
            }
            const double anext = (valid && sub == 0 && nxt) ? __ldcg(A + r + (int64_t)(j + 1) * lda) : 0.0;
            double ypart = 0.0;
            if (nxt) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = sub + 8 * u;
                    if (k < jj) ypart = fma(pv[u], srow[k], fma(pw[u], srow[TRD_NB + k], ypart));
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) ypart += __shfl_xor_sync(0xffffffffu, ypart, o);
            }
            TRD_MARK(1);
            grid_sync(a.bar, epoch, G);
            TRD_MARK(2);

            // ---- C: own rows
            if (tid < 2 * jj) {
                double v = 0.0;
                if (tau != 0.0)
#pragma unroll
                    for (int pt = 0; pt < TRD_DSPLIT; ++pt) v += __ldcg(a.dots + tid * TRD_DSPLIT + pt);
                sdot[tid] = v;
            }
            const double yb = (valid && sub == 0 && tau != 0.0) ? __ldcg(a.ybuf + r) : 0.0;
            __syncthreads();
            double t = 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = sub + 8 * u;
                if (k < jj) t = fma(pw[u], sdot[k], fma(pv[u], sdot[jj + k], t));
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            double wv = 0.0, wr = 0.0;
            if (valid && sub == 0) {
                wr = (tau != 0.0) ? tau * (yb - t) : 0.0;
                a.wpre[r] = wr;
                wv = wr * sv[r - c0];
                if (nxt) a.y0[r] = anext - ypart - wr;
            }
            wv = block_sum_d(wv, red);
            if (tid == 0) a.slots[cta * SLOTW + 1] = wv;
            TRD_MARK(3);
            grid_sync(a.bar, epoch, G);
            TRD_MARK(4);

            // ---- A': finish W(:, jj) (own rows), next column into sx
            double yv[16];
            const double wj1 = nxt ? __ldcg(a.wpre + j + 1) : 0.0;
            // row j+2 of the panel for the next column's y0 (srow), loaded with the rest
            const bool pre = nxt && tid <= jj && j + 2 < n;
            const double wj2 = (pre && tid == jj) ? __ldcg(a.wpre + j + 2) : 0.0;
            const double sr_w = (pre && tid < jj) ? __ldcg(W + j + 2 + (int64_t)tid * n) : 0.0;
            const double sr_v = pre ? __ldcg(V + j + 2 + (int64_t)(i0 + tid) * n) : 0.0;
            if (nxt) {
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int rr = j + 1 + tid + u * TRD_THREADS;
                    yv[u] = (rr < n) ? __ldcg(a.y0 + rr) : 0.0;
                }
            }
            const double a2 = -0.5 * tau * slots_sum(a.slots, 1, G, red);
            if (valid && sub == 0) W[r + (int64_t)jj * n] = wr + a2 * sv[r - c0];
            if (nxt) {
                const double coef = wj1 + 2.0 * a2;
                s2p = 0.0;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int rr = j + 1 + tid + u * TRD_THREADS;
                    if (rr < n) {
                        const double x = yv[u] - sv[rr - c0] * coef;
                        sx[rr - j - 1] = x;
                        if (rr >= j + 3) s2p += x * x;
                    }
                }
                if (pre) {
                    srow[tid] = (tid == jj) ? wj2 + a2 * sv[j + 2 - c0] : sr_w;
                    srow[TRD_NB + tid] = sr_v;
                }
                a2prev = a2;
                c0prev = c0;
            } else {
                a2prev = 0.0;
            }
            cur ^= 1;
            TRD_MARK(5);
        }
        grid_sync(a.bar, epoch, G);
        TRD_MARK(6);
        const int t0 = i0 + jb, mt = n - t0;
        if (mt > 0) {
            const int nt = (mt + TRD_TILE - 1) / TRD_TILE;
            const int ntiles = nt * (nt + 1) / 2;
            double* sVr = tl;                       // [k][64] rows R of V
            double* sWr = sVr + TRD_NB * TRD_TILE;  // rows R of W
            double* sVc = sWr + TRD_NB * TRD_TILE;  // rows C of V
            double* sWc = sVc + TRD_NB * TRD_TILE;  // rows C of W
            const int tr = tid & 15, tc = tid >> 4;  // 16 x 16 threads, 4 x 4 each
            for (int t = cta; t < ntiles; t += G) {
                int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);  // t = bi(bi+1)/2 + bj
                while (bi * (bi + 1) / 2 > t) --bi;
                while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
                const int bj = t - bi * (bi + 1) / 2;
                const int R0 = t0 + bi * TRD_TILE, C0 = t0 + bj * TRD_TILE;
                __syncthreads();
                for (int idx = tid; idx < TRD_NB * TRD_TILE; idx += TRD_THREADS) {
                    const int k = idx / TRD_TILE, i = idx % TRD_TILE;
                    const bool kin = k < jb;
                    const int rr = R0 + i, c = C0 + i;
                    sVr[idx] = (kin && rr < n) ? __ldcg(V + rr + (int64_t)(i0 + k) * n) : 0.0;
                    sWr[idx] = (kin && rr < n) ? __ldcg(W + rr + (int64_t)k * n) : 0.0;
                    sVc[idx] = (kin && c < n) ? __ldcg(V + c + (int64_t)(i0 + k) * n) : 0.0;
                    sWc[idx] = (kin && c < n) ? __ldcg(W + c + (int64_t)k * n) : 0.0;
                }
                __syncthreads();
                double acc[4][4];
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
                for (int k = 0; k < jb; ++k) {
                    double vr[4], wr4[4], vc[4], wc[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        vr[p] = sVr[k * TRD_TILE + tr + 16 * p];
                        wr4[p] = sWr[k * TRD_TILE + tr + 16 * p];
                        vc[p] = sVc[k * TRD_TILE + tc + 16 * p];
                        wc[p] = sWc[k * TRD_TILE + tc + 16 * p];
                    }
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[p][q] = fma(vr[p], wc[q], fma(wr4[p], vc[q], acc[p][q]));
                }
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const int rr = R0 + tr + 16 * p;
                    if (rr >= n) continue;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = C0 + tc + 16 * q;
                        if (c >= n) continue;
                        A[rr + (int64_t)c * lda] -= acc[p][q];
                        if (bi != bj) A[c + (int64_t)rr * lda] -= acc[p][q];
                    }
                }
            }
        }
        TRD_MARK(7);
        grid_sync(a.bar, epoch, G);
        s2p = 0.0;
        for (int rr = t0 + tid; rr < n; rr += TRD_THREADS) {
            const double x = __ldcg(A + rr + (int64_t)t0 * lda);
            sx[rr - t0] = x;
            if (rr >= t0 + 2) s2p += x * x;
        }
        __syncthreads();
        TRD_MARK(8);
    }
    if (cta == 0 && tid == 0) a.d[n - 1] = sx[0];
#undef TRD_MARK
}

// Medium n (kSytrdSmall < n <= 512): unblocked dsytd2 by ONE thread-block
// cluster with the matrix distributed over the CTAs' shared memory (columns
// [q cw, (q+1) cw) in CTA q, both triangles) and exchanged through DSMEM:
// two cluster barriers per column, no global round trips on the critical path.
template <int CS>
__global__ void __launch_bounds__(256, 1) k_sytrd_cluster(int n, const double* __restrict__ Ain, int lda,
                                                          double* __restrict__ V, double* __restrict__ d,
                                                          double* __restrict__ e, double* __restrict__ tau,
                                                          unsigned long long* prof) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    const int q = (int)cl.block_rank();
    const int cw = (n + CS - 1) / CS;
    const int c_lo = q * cw, c_hi = min(n, c_lo + cw);
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    // reflector, p values and partials are double-buffered by column parity, so
    // the owner of column j+1 can push before slower CTAs finish column j
    double* Al = sm;                     // cw x n, column c at (c - c_lo) * n
    double* svb = Al + (size_t)cw * n;   // 2 n: reflector, PUSHED here by its owner
    double* pwb = svb + 2 * n;           // 2 n: p values of all columns, pushed by their owners
    double* w = pwb + 2 * n;             // n
    double* partsb = w + n;              // 2 (CS + 4): partial p.v (pushed) | [CS] tau (pushed)
    double* red = partsb + 2 * (CS + 4); // 64
    for (int idx = tid; idx < (c_hi - c_lo) * n; idx += nt) {
        const int c = c_lo + idx / n, r = idx % n;
        Al[idx] = Ain[r + (int64_t)c * lda];
    }
    cl.sync();
    unsigned long long tp = clock64();
#define CL_MARK(i)                                          \
    if (prof && q == 0 && tid == 0) {                       \
        const unsigned long long t_ = clock64();            \
        prof[i] += t_ - tp;                                 \
        tp = t_;                                            \
    }
    for (int j = 0; j < n - 1; ++j) {
        const int owner = j / cw;
        const int m = n - j - 1;
        double* sv = svb + (j & 1) * n;
        double* pw = pwb + (j & 1) * n;
        double* parts = partsb + (j & 1) * (CS + 4);
        if (q == owner) {  // reflector of column j (warp 0 reduces), pushed to every CTA
            const double* x = Al + (size_t)(j - c_lo) * n;
            if (warp == 0) {
                double s2 = 0.0;
                for (int r = j + 2 + lane; r < n; r += 32) s2 += x[r] * x[r];
                s2 = warp_sum_d(s2);
                if (lane == 0) {
                    const double alpha = x[j + 1];
                    double tj = 0.0, beta = alpha, scal = 0.0;
                    if (s2 > 0.0) {
                        beta = -copysign(sqrt(alpha * alpha + s2), alpha);
                        tj = (beta - alpha) / beta;
                        scal = 1.0 / (alpha - beta);
                    }
                    red[40] = tj;
                    red[41] = scal;
                    d[j] = x[j];
                    e[j] = beta;
                    tau[j] = tj;
                }
            }
            __syncthreads();
            const double tj = red[40], scal = red[41];
            for (int i = tid; i < m; i += nt) {
                const double v = (i == 0) ? 1.0 : x[j + 1 + i] * scal;
                V[j + 1 + i + (int64_t)j * n] = v;
                for (int r = 0; r < CS; ++r) cl.map_shared_rank(sv, r)[i] = v;
            }
            if (tid < CS) cl.map_shared_rank(parts, tid)[CS] = tj;
        }
        CL_MARK(0);
        cl.sync();
        CL_MARK(1);
        const double tj = parts[CS];
        if (tj == 0.0) continue;  // H = I: nothing to update (uniform over the cluster)
        // p_c = tau A(j+1:, c) . v for own columns c > j (warp per column), pushed to all CTAs
        double pv = 0.0;
        for (int c = max(c_lo, j + 1) + warp; c < c_hi; c += nw) {
            const double* col = Al + (size_t)(c - c_lo) * n + j + 1;
            double acc = 0.0;
            for (int i = lane; i < m; i += 32) acc = fma(col[i], sv[i], acc);
            acc = warp_sum_d(acc) * tj;
            if (lane < CS) cl.map_shared_rank(pw, lane)[c] = acc;
            if (lane == 0) pv += acc * sv[c - j - 1];
        }
        pv = block_sum_d(pv, red);
        if (tid < CS) cl.map_shared_rank(parts, tid)[q] = pv;
        CL_MARK(3);
        cl.sync();
        CL_MARK(4);
        double tot = 0.0;
        for (int r = 0; r < CS; ++r) tot += parts[r];  // fixed order
        const double K = -0.5 * tj * tot;
        for (int i = tid; i < m; i += nt) w[i] = pw[j + 1 + i] + K * sv[i];
        __syncthreads();
        CL_MARK(5);
        // own columns: A(j+1:, c) -= v w_c + w v_c
        const int cfirst = max(c_lo, j + 1);
        const int ncols = c_hi - cfirst;
        for (int idx = tid; idx < ncols * m; idx += nt) {
            const int c = cfirst + idx / m, i = idx % m;
            const int ic = c - j - 1;
            Al[(size_t)(c - c_lo) * n + j + 1 + i] -= sv[i] * w[ic] + w[i] * sv[ic];
        }
        __syncthreads();  // the owner of column j+1 reads its (updated) column next
        CL_MARK(6);
    }
#undef CL_MARK
    if (q == (n - 1) / cw && tid == 0) d[n - 1] = Al[(size_t)(n - 1 - c_lo) * n + n - 1];
    cl.sync();
}

size_t sytrd_cluster_smem(int n, int cs) {
    const int cw = (n + cs - 1) / cs;
    return sizeof(double) * ((size_t)cw * n + 5 * (size_t)n + 2 * (cs + 4) + 64);
}

// n in (512, 2048]: unblocked dsytd2 (same arithmetic as k_sytrd_small) with
// the matrix RESIDENT IN SHARED MEMORY, distributed by rows: CTA q owns rows
// q, q + G, q + 2G, ... (cyclic, so every CTA keeps work until the end; at
// n = 2048 and G = 148 that is 14 full rows = 224 KiB). Every vector indexed by
// the column (x = the column being reduced, v, w) lives in registers of the
// thread owning that column index (cc = tid + SR_NT m), identically in every
// CTA, so per column there is ONE grid barrier and no other global round trip:
//   1. reflector v_j from x_j: block reduction of |x|^2, redundant per CTA
//   2. ONE fused pass over the own rows: apply the pending rank-2 update of
//      reflector j-1 (A -= v w^T + w v^T) and accumulate y = A v_j
//   3. publish y (own rows) and row j+1 (the next column, updates <= j-1);
//      -- grid barrier --
//   4. every CTA loads y and row j+1 (one L2 round), w = tau y,
//      alpha = -tau/2 w.v, w += alpha v, and x_{j+1} = row j+1 - v w_{j+1} - w v_{j+1}
// y and the next column are double-buffered by column parity: a CTA can only
// overwrite a buffer after every CTA passed the barrier that follows its reads.
constexpr int SR_R = 14;    // rows per CTA (smem: 14 x 2048 doubles)
constexpr int SR_NWMAX = 16;  // warps per CTA (<= 512 threads)
constexpr int kSytrdRowsMax = 2048;

size_t sytrd_rows_smem(int n, int R) {
    return sizeof(double) * ((size_t)R * n + SR_NWMAX * 16 + 2 * SR_NWMAX + 2 * SR_R + 8);
}

struct SrArgs {
    int n, lda, R;
    const double* A;  // n x n symmetric (both triangles), column-major
    double *V, *d, *e, *tau;
    double *ypub, *cpub;  // 2 x n each
    unsigned* bar;
    unsigned long long* prof;  // optional (AERO_SYTRD_PROF): CTA 0 ns per segment
};

// sum of 16 per-thread values over a warp by recursive halving (16 shuffles
// instead of 80): returns the total of value idx(lane) (lanes 2i, 2i+1 hold it)
__device__ __forceinline__ double warp_sum16(double (&v)[16], int lane) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const bool up = lane & 16;
        const double send = up ? v[i] : v[i + 8];
        const double keep = up ? v[i + 8] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool up = lane & 8;
        const double send = up ? v[i] : v[i + 4];
        const double keep = up ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const bool up = lane & 4;
        const double send = up ? v[i] : v[i + 2];
        const double keep = up ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {
        const bool up = lane & 2;
        const double send = up ? v[0] : v[1];
        const double keep = up ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
__device__ __forceinline__ int warp_sum16_index(int lane) {
    return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// one-barrier block sum: the caller alternates buffers so that a buffer is
// rewritten only after another __syncthreads (fixed order: deterministic)
template <int NW>
__device__ __forceinline__ double block_sum1(double v, double* buf) {
    v = warp_sum_d(v);
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += buf[w];
    return s;
}

template <int SR_NT>
__global__ void __launch_bounds__(SR_NT, 1) k_sytrd_rows(SrArgs a) {
    constexpr int SR_M = kSytrdRowsMax / SR_NT;  // column indices per thread
    constexpr int SR_NW = SR_NT / 32;
    extern __shared__ __align__(16) double sm[];
    const int n = a.n, G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int R = a.R;
    const int nr = (n - cta + G - 1) / G;  // own rows r_k = cta + G k, k < nr (<= R)
    double* As = sm;                        // nr x n, row k at As + k n
    double* red = sm + (size_t)R * n;       // SR_NW x 16 (row sums)
    double* rs2 = red + SR_NWMAX * 16;      // SR_NW: reflector norm partials
    double* rdot = rs2 + SR_NWMAX;          // SR_NW: w.v partials
    double* rv = rdot + SR_NWMAX;           // v_{j-1}(r_k)
    double* rw = rv + SR_R;                 // w_{j-1}(r_k)
    double* bc = rw + SR_R;                 // broadcast scalars
    for (int k = 0; k < nr; ++k) {
        const double* src = a.A + (int64_t)(cta + G * k) * a.lda;  // row r = column r (symmetric)
        for (int cc = tid; cc < n; cc += SR_NT) As[(size_t)k * n + cc] = src[cc];
    }
    if (tid < SR_R) rv[tid] = rw[tid] = 0.0;
    double xr[SR_M], vr[SR_M], wr[SR_M];
#pragma unroll
    for (int m = 0; m < SR_M; ++m) {
        const int cc = tid + SR_NT * m;
        xr[m] = (cc < n) ? a.A[cc] : 0.0;  // column 0
        vr[m] = wr[m] = 0.0;
    }
    unsigned epoch = 0;
    const bool pr = a.prof && cta == 0 && tid == 0;
    unsigned long long tp = 0;
    if (pr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp));
#define SR_MARK(i)                                                   \
    if (pr) {                                                        \
        unsigned long long t_;                                       \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));       \
        a.prof[i] += t_ - tp;                                        \
        tp = t_;                                                     \
    }
    for (int j = 0; j < n - 1; ++j) {
        // ---- 1. reflector (dlarfg) from x_j, rows j+1 ..
        double s2 = 0.0;
#pragma unroll
        for (int m = 0; m < SR_M; ++m) {
            const int cc = tid + SR_NT * m;
            if (cc >= j + 2 && cc < n) s2 = fma(xr[m], xr[m], s2);
            if (cc == j) bc[0] = xr[m];
            if (cc == j + 1) bc[1] = xr[m];
        }
        s2 = block_sum1<SR_NW>(s2, rs2);  // the sync also publishes bc
        const double dj = bc[0], alpha = bc[1];
        double tj = 0.0, beta = alpha, scal = 0.0;
        if (s2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s2), alpha);
            tj = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        double vn[SR_M];
#pragma unroll
        for (int m = 0; m < SR_M; ++m) {
            const int cc = tid + SR_NT * m;
            const double vv = (cc == j + 1) ? 1.0 : (cc >= j + 2 && cc < n) ? xr[m] * scal : 0.0;
            if (cta == 0 && cc > j && cc < n) a.V[cc + (int64_t)j * n] = vv;
            vn[m] = (tj != 0.0) ? vv : 0.0;
        }
        if (cta == 0 && tid == 0) {
            a.d[j] = dj;
            a.e[j] = beta;
            a.tau[j] = tj;
        }
        SR_MARK(0);
        // ---- 2. fused pass: pending update j-1, then y = A v_j (own rows >= j+1)
        const int k0 = (j + 1 <= cta) ? 0 : (j + 1 - cta + G - 1) / G;  // first own row >= j+1
        double acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.0;
        bool act[SR_M];
#pragma unroll
        for (int m = 0; m < SR_M; ++m) act[m] = (tid + SR_NT * m >= j + 1) && (tid + SR_NT * m < n);
#pragma unroll
        for (int k = 0; k < SR_R; ++k) {
            if (k >= k0 && k < nr) {
                // row factors once per row (stores to As could alias them otherwise)
                const double rvk = rv[k], rwk = rw[k];
                double* rowp = As + (size_t)k * n + tid;
#pragma unroll
                for (int m = 0; m < SR_M; ++m) {
                    if (act[m]) {
                        double* p = rowp + SR_NT * m;
                        const double x = fma(-rwk, vr[m], fma(-rvk, wr[m], *p));
                        *p = x;
                        acc[k] = fma(x, vn[m], acc[k]);
                    }
                }
            }
        }
        SR_MARK(1);
        // row j+1 after updates <= j-1 is the next column (symmetry): publish it
        double* cpub = a.cpub + (size_t)(j & 1) * n;
        double* ypub = a.ypub + (size_t)(j & 1) * n;
        if ((j + 1) % G == cta) {
            const int k1 = (j + 1) / G;
#pragma unroll
            for (int m = 0; m < SR_M; ++m) {
                const int cc = tid + SR_NT * m;
                if (cc >= j + 1 && cc < n) __stcg(cpub + cc, As[(size_t)k1 * n + cc]);
            }
        }
        // ---- 3. y(r_k) = block sum of acc[k], publish
        {
            const double ws = warp_sum16(acc, lane);
            const int idx = warp_sum16_index(lane);
            if (!(lane & 1)) red[warp * 16 + idx] = ws;
            __syncthreads();
            if (tid < nr && tid >= k0) {
                double y = 0.0;
                for (int w = 0; w < SR_NW; ++w) y += red[w * 16 + tid];
                __stcg(ypub + cta + G * tid, y);
            }
        }
        SR_MARK(2);
        grid_sync(a.bar, epoch, G);
        SR_MARK(3);
        // ---- 4. w = tau y; alpha = -tau/2 w.v; w += alpha v; next column
        double yv[SR_M], cv[SR_M];
#pragma unroll
        for (int m = 0; m < SR_M; ++m) {
            const int cc = tid + SR_NT * m;
            const bool act = cc >= j + 1 && cc < n;
            yv[m] = act ? __ldcg(ypub + cc) : 0.0;
            cv[m] = act ? __ldcg(cpub + cc) : 0.0;
        }
        double dot = 0.0;
#pragma unroll
        for (int m = 0; m < SR_M; ++m) {
            yv[m] *= tj;
            dot = fma(yv[m], vn[m], dot);
            if (tid + SR_NT * m == j + 1) bc[2] = yv[m];
        }
        dot = block_sum1<SR_NW>(dot, rdot);
        const double al = -0.5 * tj * dot;
        const double vj1 = (tj != 0.0) ? 1.0 : 0.0;
        const double wj1 = bc[2] + al * vj1;
#pragma unroll
        for (int m = 0; m < SR_M; ++m) {
            const int cc = tid + SR_NT * m;
            const double wn = fma(al, vn[m], yv[m]);
            xr[m] = (cc >= j + 1 && cc < n) ? fma(-wn, vj1, fma(-vn[m], wj1, cv[m])) : 0.0;
            vr[m] = vn[m];
            wr[m] = wn;
            if (cc < n && cc % G == cta) {  // own rows: the pending update's row factors
                rv[cc / G] = vn[m];
                rw[cc / G] = wn;
            }
        }
        SR_MARK(4);
    }
#undef SR_MARK
    // x_{n-1}(n-1): the last diagonal element
#pragma unroll
    for (int m = 0; m < SR_M; ++m)
        if (cta == 0 && tid + SR_NT * m == n - 1) a.d[n - 1] = xr[m];
}

// Small n (<= kSytrdSmall): unblocked dsytd2 by ONE CTA with the whole matrix
// in shared memory (no grid barriers). Same outputs as k_sytrd.
constexpr int kSytrdSmall = 128;
constexpr int kSytrdClusterMax = 512;
__global__ void __launch_bounds__(512, 1) k_sytrd_small(int n, const double* __restrict__ Ain, int lda,
                                                        double* __restrict__ V, double* __restrict__ d,
                                                        double* __restrict__ e, double* __restrict__ tau) {
    extern __shared__ __align__(16) double sa[];  // n*n matrix (ld n), v[n], w[n], red[64]
    double* sv = sa + n * n;
    double* sw = sv + n;
    double* red = sw + n;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int idx = tid; idx < n * n; idx += nt) sa[idx] = Ain[idx % n + (int64_t)(idx / n) * lda];
    __syncthreads();
    for (int j = 0; j < n - 1; ++j) {
        const int m = n - j - 1;  // rows j+1 .. n-1
        double s2 = 0.0;
        for (int i = j + 2 + tid; i < n; i += nt) s2 += sa[i + j * n] * sa[i + j * n];
        s2 = block_sum_d(s2, red);
        const double alpha = sa[j + 1 + j * n];
        double tj = 0.0, beta = alpha, scal = 0.0;
        if (s2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s2), alpha);
            tj = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        for (int i = tid; i < m; i += nt) {
            const double v = (i == 0) ? 1.0 : sa[j + 1 + i + j * n] * scal;
            sv[i] = v;
            V[j + 1 + i + (int64_t)j * n] = v;
        }
        if (tid == 0) {
            d[j] = sa[j + j * n];
            e[j] = beta;
            tau[j] = tj;
        }
        __syncthreads();
        if (tj == 0.0) continue;
        // p = tau A22 v  (A22 = sa[j+1:, j+1:]; consecutive threads take consecutive rows)
        for (int r = tid; r < m; r += nt) {
            const double* row = sa + (j + 1 + r) + (j + 1) * n;
            double acc = 0.0;
            for (int c = 0; c < m; ++c) acc = fma(row[c * n], sv[c], acc);
            sw[r] = tj * acc;
        }
        __syncthreads();
        double pv = 0.0;
        for (int i = tid; i < m; i += nt) pv += sw[i] * sv[i];
        pv = block_sum_d(pv, red);
        const double K = -0.5 * tj * pv;
        for (int i = tid; i < m; i += nt) sw[i] += K * sv[i];
        __syncthreads();
        // A22 -= v w^T + w v^T
        for (int idx = tid; idx < m * m; idx += nt) {
            const int r = idx % m, c = idx / m;
            sa[(j + 1 + r) + (j + 1 + c) * n] -= sv[r] * sw[c] + sw[r] * sv[c];
        }
        __syncthreads();
    }
    if (tid == 0) d[n - 1] = sa[(n - 1) + (n - 1) * n];
}

// Gershgorin interval, pivmin, ||T||; T is split into unreduced blocks where
// e_i^2 <= eps^2 |d_i d_{i+1}| + safmin or |e_i| <= eps ||T|| (LAPACK dstebz /
// dsteqr criterion): e_i is set to 0 there. blk[i] = first row of i's block,
// blk[n + i] = one past its last row. One CTA.
__global__ void k_tri_prep(int n, const double* __restrict__ d, double* __restrict__ e,
                           double* __restrict__ e2, double* __restrict__ bounds, int* __restrict__ blk) {
    __shared__ double smin[32], smax[32], se[32];
    __shared__ double s_tnorm;
    double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double el = (i > 0) ? fabs(e[i - 1]) : 0.0;
        const double er = (i < n - 1) ? fabs(e[i]) : 0.0;
        lo = fmin(lo, d[i] - el - er);
        hi = fmax(hi, d[i] + el + er);
        if (i < n - 1) emax = fmax(emax, e[i] * e[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        smin[wid] = lo;
        smax[wid] = hi;
        se[wid] = emax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) {
            lo = fmin(lo, smin[w]);
            hi = fmax(hi, smax[w]);
            emax = fmax(emax, se[w]);
        }
        const double tnorm = fmax(fabs(lo), fabs(hi));
        const double pivmin = DBL_MIN * fmax(1.0, emax);
        const double pad = 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
        bounds[0] = lo - pad;
        bounds[1] = hi + pad;
        bounds[2] = pivmin;
        bounds[3] = tnorm;
        s_tnorm = tnorm;
    }
    __syncthreads();
    const double tnorm = s_tnorm;
    for (int i = threadIdx.x; i < n - 1; i += blockDim.x) {
        const double ei = e[i];
        const bool split = ei * ei <= DBL_EPSILON * DBL_EPSILON * fabs(d[i] * d[i + 1]) + DBL_MIN ||
                           fabs(ei) <= (double)n * DBL_EPSILON * tnorm;
        if (split) e[i] = 0.0;
        e2[i] = split ? 0.0 : ei * ei;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // block boundaries: warp scans over 32-row chunks (ballot masks)
        int carry = 0;         // first row of the block open at the chunk start
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const bool f = i < n && (i == n - 1 || e[i] == 0.0);  // a block ends at row i
            const unsigned m = __ballot_sync(0xffffffffu, f);
            const unsigned below = m & ((1u << lane) - 1u);
            if (i < n) blk[i] = below ? base + (31 - __clz(below)) + 1 : carry;
            if (m) carry = base + (31 - __clz(m)) + 1;
        }
        int carry2 = n;  // one past the end of the block continuing after the chunk
        for (int base = ((n - 1) / 32) * 32; base >= 0; base -= 32) {
            const int i = base + lane;
            const bool f = i < n && (i == n - 1 || e[i] == 0.0);
            const unsigned m = __ballot_sync(0xffffffffu, f);
            const unsigned here = m & ~((1u << lane) - 1u);
            if (i < n) blk[n + i] = here ? base + __ffs(here) : carry2;
            if (m) carry2 = base + __ffs(m);
        }
    }
}

// Sturm count over rows [s, t): eigenvalues of that block strictly below x
// reciprocal on the Sturm recurrence's critical path: hardware approximation
// plus two Newton steps (~1 ulp; |q| >= pivmin >= DBL_MIN, so no subnormals) --
// about a third of the latency of the correctly rounded __drcp_rn
__device__ __forceinline__ double rcp_nr(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = fma(r, fma(-q, r, 1.0), r);
    return fma(r, fma(-q, r, 1.0), r);
}

__device__ __forceinline__ int sturm_count(int s, int t, const double* d, const double* e2, double x,
                                           double pivmin) {
    int cnt = 0;
    double q = d[s] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = s + 1; i < t; ++i) {
        q = d[i] - x - e2[i - 1] * rcp_nr(q);
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// coarse cut: global Sturm counts at 1023 evenly spaced points x_m (one
// thread each, spread over 32 CTAs so the division chains run on 32 SMs);
// k_bisect derives from them the largest x_m with count(x_m) <= kc (a lower
// bound of the kc-th smallest eigenvalue) -- bounds[5] = 1 marks them valid,
// bounds[6] = kc
__global__ void __launch_bounds__(32) k_cut_coarse(int n, int kc, const double* __restrict__ d,
                                                   const double* __restrict__ e2, double* __restrict__ bounds,
                                                   int* __restrict__ hist) {
    const double lo = bounds[0], hi = bounds[1], pivmin = bounds[2];
    const int m = blockIdx.x * 32 + threadIdx.x;
    if (m < 1023) hist[m] = sturm_count(0, n, d, e2, lo + (hi - lo) * (double)(m + 1) / 1024.0, pivmin);
    if (m == 0) {
        bounds[5] = 1.0;
        bounds[6] = (double)kc;
    }
}

// one warp per row p: the (p - s)-th smallest eigenvalue of p's block [s, t),
// by 33-way multisection of the Gershgorin interval; d, e^2 in shared memory
__global__ void k_bisect(int n, const double* __restrict__ d, const double* __restrict__ e2,
                         const double* __restrict__ bounds, const int* __restrict__ blk,
                         double* __restrict__ lam, const int* __restrict__ hist) {
    extern __shared__ double sde[];
    double* sd = sde;
    double* se = sde + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sd[i] = d[i];
        se[i] = (i < n - 1) ? e2[i] : 0.0;
    }
    __syncthreads();
    const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n) return;
    const int bs = blk[p], bt = blk[n + p], k = p - bs;
    if (bt - bs == 1) {
        if (lane == 0) lam[p] = sd[p];
        return;
    }
    const double pivmin = bounds[2];
    double lo = bounds[0], hi = bounds[1];
    // below the cut (only the top eigenvalues are wanted): park at the lower bound
    double xcut = -DBL_MAX;
    if (bounds[5] > 0.5) {  // largest coarse point with count <= kc (k_cut_coarse)
        const int kc = (int)bounds[6];
        int a = 0, b = 1023;  // first m with hist[m] > kc (1023: none)
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (hist[mid] > kc) b = mid;
            else a = mid + 1;
        }
        xcut = (a == 0) ? lo : lo + (hi - lo) * (double)a / 1024.0;
    }
    if (sturm_count(bs, bt, sd, se, xcut, pivmin) > k) {
        if (lane == 0) lam[p] = lo;
        return;
    }
    for (int round = 0; round < 64; ++round) {
        const double tol = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin;
        if (hi - lo <= tol) break;
        const double h = (hi - lo) / 33.0;
        const double x = fmin(lo + h * (lane + 1), hi);
        const int c = sturm_count(bs, bt, sd, se, x, pivmin);
        const unsigned above = __ballot_sync(0xffffffffu, c > k);
        double nlo = lo, nhi = hi;
        if (above) {
            const int f = __ffs(above) - 1;
            nhi = __shfl_sync(0xffffffffu, x, f);
            const double xp = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
            if (f > 0) nlo = xp;
        } else {
            nlo = __shfl_sync(0xffffffffu, x, 31);
        }
        if (nlo == lo && nhi == hi) break;  // interval can no longer be split
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) lam[p] = 0.5 * (lo + hi);
}

// descending order of all eigenvalues (ties by row): order[q] = row, w[q] = lambda
__global__ void k_order(int n, const double* __restrict__ lam, int* __restrict__ order, double* __restrict__ w) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double lp = lam[p];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
        const double li = lam[i];
        rank += (li > lp) || (li == lp && i < p);
    }
    order[rank] = p;
    w[rank] = lp;
}

// eigenvector (descending index q) of its unreduced block [s, t) by a twisted
// factorization; zero outside the block. Scratch Dp and output Z are
// row-interleaved: element i of vector q at [i * nvec + q], so consecutive
// threads touch consecutive addresses.
__global__ void k_twisted(int n, int nvec, const double* __restrict__ d, const double* __restrict__ e,
                          const double* __restrict__ lam, const double* __restrict__ wdesc,
                          const int* __restrict__ order, const int* __restrict__ blk,
                          const double* __restrict__ bounds, double* __restrict__ Dp, double* __restrict__ L1,
                          double* __restrict__ L2, double* __restrict__ L3, double* __restrict__ Z, int usm) {
    extern __shared__ double sde[];
    double* sd = sde;
    double* se = sde + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sd[i] = d[i];
        se[i] = (i < n - 1) ? e[i] : 0.0;
    }
    __syncthreads();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nvec) return;
    const int p = order[q];
    const int bs = blk[p], bt = blk[n + p];
    const double lv = lam[p];
    const double pivmin = bounds[2];
    auto safe = [&](double x) { return (fabs(x) < pivmin) ? -pivmin : x; };
    // per-thread scratch in shared memory when it fits (usm), else interleaved in global
    double* sDp = sde + 2 * n + threadIdx.x;
    double* sZ = sDp + (size_t)n * blockDim.x;
    auto DP = [&](int i) -> double& { return usm ? sDp[(size_t)i * blockDim.x] : Dp[(int64_t)i * nvec + q]; };
    auto ZZ = [&](int i) -> double& { return usm ? sZ[(size_t)i * blockDim.x] : Z[(int64_t)i * nvec + q]; };
    if (bt - bs == 1) {
        for (int i = 0; i < n; ++i) Z[(int64_t)i * nvec + q] = (i == bs) ? 1.0 : 0.0;
        return;
    }
    for (int i = 0; i < bs; ++i) ZZ(i) = 0.0;
    for (int i = bt; i < n; ++i) ZZ(i) = 0.0;
    // top-down stationary qd: D+(i)
    double dp = safe(sd[bs] - lv);
    DP(bs) = dp;
    for (int i = bs; i < bt - 1; ++i) {
        dp = safe(sd[i + 1] - lv - (se[i] * se[i]) * rcp_nr(dp));  // reciprocal off the divide path
        DP(i + 1) = dp;
    }
    // numerically repeated eigenvalue (gap to a neighbour < 1e-12 ||T||): a twisted
    // vector is not determined; LAPACK dstein-style inverse iteration instead --
    // shift perturbed below the earlier equal members of the block, pivoted LU
    // (dlagtf / dlagts) in the interleaved scratch, pseudo-random start, two
    // solves; k_cluster_orth then orthonormalizes the run
    const double tdeg = 1e-12 * bounds[3];
    const bool degen = (q > 0 && wdesc[q - 1] - wdesc[q] < tdeg) || (q + 1 < nvec && wdesc[q] - wdesc[q + 1] < tdeg);
    if (degen) {
        if (usm) {
            for (int i = 0; i < bs; ++i) Z[(int64_t)i * nvec + q] = 0.0;
            for (int i = bt; i < n; ++i) Z[(int64_t)i * nvec + q] = 0.0;
        }
        int cnt = 0;
        for (int j = q - 1; j >= 0 && wdesc[j] - wdesc[q] < 1e-10 * bounds[3]; --j) cnt += blk[order[j]] == bs;
        const double shift = lv - cnt * 10.0 * DBL_EPSILON * bounds[3];
        const double tiny = DBL_EPSILON * bounds[3] + pivmin;
        double* la = Dp;   // U diagonal
        double* lb = L1;   // U first super-diagonal
        double* ll = L2;   // multipliers, sign bit of L3 = pivot
        double* ld2 = L3;  // U second super-diagonal
        auto at = [&](double* a, int k) -> double& { return a[(int64_t)(bs + k) * nvec + q]; };
        const int len = bt - bs;
        for (int k = 0; k < len; ++k) {
            at(la, k) = sd[bs + k] - shift;
            at(lb, k) = (k < len - 1) ? se[bs + k] : 0.0;
        }
        // partial pivoting: |multiplier| <= 1, so a row swap is recorded as multiplier +- 4
        for (int k = 0; k < len - 1; ++k) {
            const double ck = se[bs + k];
            double ak = at(la, k);
            at(ld2, k) = 0.0;
            if (fabs(ak) >= fabs(ck)) {
                if (ak == 0.0) {
                    ak = tiny;
                    at(la, k) = tiny;
                }
                const double mult = ck / ak;
                at(ll, k) = mult;
                at(la, k + 1) -= mult * at(lb, k);
            } else {
                const double mult = ak / ck;
                at(ll, k) = mult >= 0.0 ? mult + 4.0 : mult - 4.0;
                at(la, k) = ck;
                const double tmp = at(la, k + 1);
                at(la, k + 1) = at(lb, k) - mult * tmp;
                if (k < len - 2) {
                    at(ld2, k) = at(lb, k + 1);
                    at(lb, k + 1) = -mult * at(ld2, k);
                }
                at(lb, k) = tmp;
            }
        }
        if (at(la, len - 1) == 0.0) at(la, len - 1) = tiny;
        double nrm2 = 0.0;
        for (int k = 0; k < len; ++k) {
            uint64_t h = (uint64_t)(q + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)(bs + k + 7) * 0xBF58476D1CE4E5B9ull;
            h ^= h >> 31;
            h *= 0x94D049BB133111EBull;
            h ^= h >> 29;
            const double v = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
            at(Z, k) = v;
        }
        for (int it = 0; it < 2; ++it) {
            for (int k = 0; k < len - 1; ++k) {  // P L y = x
                double m = at(ll, k);
                const bool sw = fabs(m) > 2.0;
                if (sw) m = m >= 0.0 ? m - 4.0 : m + 4.0;
                const double xk = at(Z, k), xk1 = at(Z, k + 1);
                if (!sw) {
                    at(Z, k + 1) = xk1 - m * xk;
                } else {
                    at(Z, k) = xk1;
                    at(Z, k + 1) = xk - m * xk1;
                }
            }
            nrm2 = 0.0;
            for (int k = len - 1; k >= 0; --k) {  // U z = y
                double v = at(Z, k);
                if (k < len - 1) v -= at(lb, k) * at(Z, k + 1);
                if (k < len - 2) v -= at(ld2, k) * at(Z, k + 2);
                v /= at(la, k);
                at(Z, k) = v;
                nrm2 += v * v;
            }
            const double sc = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
            for (int k = 0; k < len; ++k) at(Z, k) *= sc;
        }
        return;
    }
    // bottom-up: D-(i) into Z, twist index by min |gamma|. The loads that do
    // not depend on the recurrence are issued 8 ahead (global scratch is L2).
    constexpr int PF = 8;
    double dm = safe(sd[bt - 1] - lv);
    ZZ(bt - 1) = dm;
    int r = bt - 1;
    double best = fabs(dp);  // gamma at the last row = D+(last)
    for (int ib = bt - 2; ib >= bs; ib -= PF) {
        double pre[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) pre[u] = (ib - u >= bs) ? DP(ib - u) : 0.0;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = ib - u;
            if (i < bs) break;
            dm = safe(sd[i] - lv - (se[i] * se[i]) * rcp_nr(dm));
            ZZ(i) = dm;
            const double g = pre[u] + dm - (sd[i] - lv);
            if (fabs(g) < best) {
                best = fabs(g);
                r = i;
            }
        }
    }
    // solve outward from r
    double nrm2 = 1.0, z = 1.0;
    for (int ib = r; ib < bt - 1; ib += PF) {  // z_{i+1} = -(e_i / D-(i+1)) z_i
        double pre[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) pre[u] = (ib + u < bt - 1) ? ZZ(ib + u + 1) : 1.0;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = ib + u;
            if (i >= bt - 1) break;
            z = -(se[i] / pre[u]) * z;
            ZZ(i + 1) = z;
            nrm2 += z * z;
        }
    }
    ZZ(r) = 1.0;
    z = 1.0;
    for (int ib = r - 1; ib >= bs; ib -= PF) {  // z_i = -(e_i / D+(i)) z_{i+1}
        double pre[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) pre[u] = (ib - u >= bs) ? DP(ib - u) : 1.0;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = ib - u;
            if (i < bs) break;
            z = -(se[i] / pre[u]) * z;
            ZZ(i) = z;
            nrm2 += z * z;
        }
    }
    const double sc = 1.0 / sqrt(nrm2);
    // normalize: 16 loads in flight per thread (the scratch is L2 when !usm;
    // one dependent L2 round trip per element was a third of the kernel)
    for (int i0 = bs; i0 < bt; i0 += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (i0 + u < bt) ? ZZ(i0 + u) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (i0 + u < bt) ZZ(i0 + u) = v[u] * sc;
    }
    if (usm)
        for (int i = 0; i < n; ++i) Z[(int64_t)i * nvec + q] = ZZ(i);
}

// re-orthonormalize the vectors of each cluster of close eigenvalues
// (classical Gram-Schmidt applied twice, one CTA per cluster leader; clusters
// longer than kMaxCluster are cut into consecutive groups of that length).
// Vectors of different unreduced blocks have disjoint support (exactly
// orthogonal); inside a block the eigenvalues are distinct.
constexpr int kMaxCluster = 128;
// Long runs (the noise floor of the AMM cod_reduce Grams: ~200 linked
// eigenvalues at n = 256 cost 7 ms vector by vector from L2) are
// re-orthonormalized by block classical Gram-Schmidt applied twice (BCGS2):
// panels of PB vectors staged in shared memory, projected against all earlier
// run members with two passes over them (W = Q^T P, P -= Q W), then
// CGS2-orthonormalized inside the panel. Same span, orthonormal to working
// precision; ~20x fewer dependent steps.
constexpr int kPanelMin = 32, kPanelMaxN = 512, kPanelMaxRun = 512;
__host__ __device__ constexpr int cluster_panel_width(int n) { return n <= 256 ? 32 : 16; }
size_t cluster_orth_smem(int n) {
    const int pb = cluster_panel_width(n);
    // panel (n x PB) + W (run x PB, run <= nvec <= n): 128 KiB at n = 256 or 512
    return sizeof(double) * (n <= kPanelMaxN ? std::max<size_t>((size_t)n, (size_t)2 * n * pb) : n);
}
__device__ void cluster_orth_panels(int n, int nvec, int q, int end, double* __restrict__ Z, double* sm,
                                    double* red) {
    const int PB = cluster_panel_width(n);
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    double* P = sm;           // n x PB, row t at P + t * PB
    double* W = P + n * PB;   // (run) x PB, row a at W + a * PB
    for (int p0 = q; p0 < end; p0 += PB) {
        const int pb = min(PB, end - p0), prev = p0 - q;
        for (int e = tid; e < n * PB; e += nt) {
            const int t = e / PB, j = e % PB;
            P[e] = (j < pb) ? Z[(int64_t)t * nvec + p0 + j] : 0.0;
        }
        __syncthreads();
        for (int pass = 0; pass < 2 && prev > 0; ++pass) {
            // W[a][j] = sum_t Z[t][q + a] P[t][j]: thread per earlier member a
            for (int a = tid; a < prev; a += nt) {
                double acc[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = 0.0;
                const double* zc = Z + q + a;
                for (int t = 0; t < n; ++t) {
                    const double z = zc[(int64_t)t * nvec];
                    const double* pr = P + t * PB;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < PB) acc[j] = fma(z, pr[j], acc[j]);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < PB) W[a * PB + j] = acc[j];
            }
            __syncthreads();
            // P[t][j] -= sum_a Z[t][q + a] W[a][j]: thread per row t
            for (int t = tid; t < n; t += nt) {
                double acc[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = (j < PB) ? P[t * PB + j] : 0.0;
                const double* zr = Z + (int64_t)t * nvec + q;
                for (int a = 0; a < prev; ++a) {
                    const double z = zr[a];
                    const double* wr = W + a * PB;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < PB) acc[j] = fma(-z, wr[j], acc[j]);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < PB) P[t * PB + j] = acc[j];
            }
            __syncthreads();
        }
        // CGS2 inside the panel (shared memory)
        for (int j = 0; j < pb; ++j) {
            for (int pass = 0; pass < 2 && j > 0; ++pass) {
                for (int i = warp; i < j; i += nw) {  // d_i = P[:, i] . P[:, j]
                    double d = 0.0;
                    for (int t = lane; t < n; t += 32) d = fma(P[t * PB + i], P[t * PB + j], d);
                    d = warp_sum_d(d);
                    if (lane == 0) red[i] = d;
                }
                __syncthreads();
                for (int t = tid; t < n; t += nt) {
                    double acc = P[t * PB + j];
                    for (int i = 0; i < j; ++i) acc = fma(-red[i], P[t * PB + i], acc);
                    P[t * PB + j] = acc;
                }
                __syncthreads();
            }
            double nr = 0.0;
            for (int t = tid; t < n; t += nt) nr = fma(P[t * PB + j], P[t * PB + j], nr);
            nr = block_sum_d(nr, red + 32);
            const double sc = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
            for (int t = tid; t < n; t += nt) P[t * PB + j] *= sc;
            __syncthreads();
        }
        for (int e = tid; e < n * PB; e += nt) {
            const int t = e / PB, j = e % PB;
            if (j < pb) Z[(int64_t)t * nvec + p0 + j] = P[e];
        }
        __syncthreads();
    }
}
__global__ void __launch_bounds__(256) k_cluster_orth(int n, int nvec, const double* __restrict__ wdesc,
                                                      const double* __restrict__ bounds, double* __restrict__ Z) {
    __shared__ double red[64];
    extern __shared__ double dots[];  // n
    const int q = blockIdx.x;
    const double thr = 1e-6 * bounds[3] + bounds[2];
    auto linked = [&](int i) { return i > 0 && wdesc[i - 1] - wdesc[i] <= thr; };
    // the whole run of linked eigenvalues around q
    int st = q;
    while (st > 0 && linked(st)) --st;
    int fend = st + 1;
    while (fend < nvec && linked(fend)) ++fend;
    bool degenerate = false;
    for (int i = st + 1; i < fend; ++i) degenerate |= (wdesc[i - 1] - wdesc[i]) < 1e-12 * bounds[3];
    int end;
    if (degenerate) {  // one CTA handles the whole run (members made orthogonal to all earlier ones)
        if (q != st) return;
        end = fend;
    } else {  // independent groups of at most kMaxCluster
        if ((q - st) % kMaxCluster != 0) return;
        end = min(fend, q + kMaxCluster);
    }
    if (end - q < 2) return;
    // numerically null clusters (|lambda| <= 1e-10 ||T||): every caller weights
    // these directions by sqrt(lambda) or cuts them at its rank threshold
    if (fabs(wdesc[q]) <= 1e-10 * bounds[3]) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (end - q > kPanelMin && n <= kPanelMaxN && end - q <= min(kPanelMaxRun, n)) {
        cluster_orth_panels(n, nvec, q, end, Z, dots, red);
        return;
    }
    for (int i = q + 1; i < end; ++i) {
        for (int pass = 0; pass < 2; ++pass) {
            for (int p = q + warp; p < i; p += 8) {
                double dot = 0.0;
                for (int t = lane; t < n; t += 32) dot = fma(Z[(int64_t)t * nvec + p], Z[(int64_t)t * nvec + i], dot);
                dot = warp_sum_d(dot);
                if (lane == 0) dots[p - q] = dot;
            }
            __syncthreads();
            for (int t = tid; t < n; t += blockDim.x) {
                const double* zr = Z + (int64_t)t * nvec;
                double acc = zr[i];
                for (int p = q; p < i; ++p) acc = fma(-dots[p - q], zr[p], acc);
                Z[(int64_t)t * nvec + i] = acc;
            }
            __syncthreads();
        }
        double nr = 0.0;
        for (int t = tid; t < n; t += blockDim.x) nr += Z[(int64_t)t * nvec + i] * Z[(int64_t)t * nvec + i];
        nr = block_sum_d(nr, red);
        const double sc = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
        for (int t = tid; t < n; t += blockDim.x) Z[(int64_t)t * nvec + i] *= sc;
        __syncthreads();
    }
}

// Y (n x nvec column-major) = Z^T view (Z row-interleaved n x nvec)
__global__ void k_interleaved_to_cols(int n, int nvec, const double* __restrict__ Z, double* __restrict__ Y,
                                      int ldy) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, q0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, q = q0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < n && q < nvec) ? Z[(int64_t)i * nvec + q] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int q = q0 + r, i = i0 + threadIdx.x;
        if (q < nvec && i < n) Y[i + (int64_t)q * ldy] = tile[threadIdx.x][r];
    }
}

// dlarft (forward, columnwise) for every back-transform block at once: one
// CTA per block b, T_b (nb x nb upper) from S_b = V_b^T V_b and tau, T in smem
__global__ void k_larft(int nref, const double* __restrict__ S, const double* __restrict__ tau,
                        double* __restrict__ T) {
    extern __shared__ double sT[];  // BT_NB x BT_NB T, then S strictly-upper packed by column
    const int b = blockIdx.x;
    const int j0 = b * BT_NB, nb = min(BT_NB, nref - j0);
    const double* Sb = S + (size_t)b * BT_NB * BT_NB;
    double* sS = sT + BT_NB * BT_NB;  // column i at offset i(i-1)/2, rows 0..i-1
    for (int idx = threadIdx.x; idx < BT_NB * BT_NB; idx += blockDim.x) {
        sT[idx] = 0.0;
        const int r = idx % BT_NB, c = idx / BT_NB;
        if (r < c) sS[c * (c - 1) / 2 + r] = Sb[r + (size_t)c * BT_NB];
    }
    __syncthreads();
    // T(0:i, i) = -tau_i T(0:i, 0:i) S(0:i, i): 4 threads per row split the sum
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    for (int i = 0; i < nb; ++i) {
        const double ti = tau[j0 + i];
        const double* scol = sS + i * (i - 1) / 2;
        double acc = 0.0;
        if (r < i)
            for (int c = r + part; c < i; c += 4) acc = fma(sT[r + c * BT_NB], scol[c], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (r < i && part == 0) sT[r + i * BT_NB] = -ti * acc;
        if (threadIdx.x == 0) sT[i + i * BT_NB] = ti;
        __syncthreads();
    }
    double* Tb = T + (size_t)b * BT_NB * BT_NB;
    for (int idx = threadIdx.x; idx < BT_NB * BT_NB; idx += blockDim.x) Tb[idx] = sT[idx];
}

// small n (<= 128): apply the reflectors directly, warp per eigenvector
// (v_j from V in L2, dot by shuffles), then the sign fix and the output copy:
// one launch instead of larft + 4 GEMMs per 128-reflector block
__global__ void k_backtransform_small(int n, int nvec, const double* __restrict__ V, const double* __restrict__ tau,
                                      const double* __restrict__ Z, double* __restrict__ A, int lda) {
    extern __shared__ double zb[];  // per warp: n
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int q = blockIdx.x * nw + warp;
    if (q >= nvec) return;
    double* z = zb + (size_t)warp * n;
    for (int i = lane; i < n; i += 32) z[i] = Z[(int64_t)i * nvec + q];
    __syncwarp();
    for (int j = n - 2; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const double* v = V + (int64_t)j * n;
        double s = 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) s = fma(v[i], z[i], s);
        s = warp_sum_d(s) * tj;
        for (int i = j + 1 + lane; i < n; i += 32) z[i] -= s * v[i];
        __syncwarp();
    }
    double best = -1.0;
    int at = n;
    for (int i = lane; i < n; i += 32)
        if (fabs(z[i]) > best) {
            best = fabs(z[i]);
            at = i;
        }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, at, o);
        if (ob > best || (ob == best && oa < at)) {
            best = ob;
            at = oa;
        }
    }
    const double sg = (z[at] < 0.0) ? -1.0 : 1.0;
    for (int i = lane; i < n; i += 32) A[i + (int64_t)q * lda] = sg * z[i];
}

struct Work {
    DeviceBuf V, W, vec, Z, Dp, L, Y, S, T, M1, M2, ws, pub;
    unsigned* bar = nullptr;
    int grid = 0;
};
std::mutex g_mu;
std::unordered_map<cudaStream_t, Work> g_work;

size_t trd_smem(int n) {
    const size_t npad = (size_t)((n + 3) & ~1);
    return sizeof(double) * (64 + 3 * npad + 4 * TRD_NB + 4 * (size_t)TRD_TILE * TRD_NB);
}
}  // namespace

constexpr int kEighLargeMax = 4096;  // shared-memory bound of k_sytrd (3 n + tiles doubles)

void eigh_large(cudaStream_t st, int n, double* A, int lda, double* w, int nvec) {
    if (n > kEighLargeMax) throw InvalidInput("eigh: n beyond the device solver limit");
    if (nvec <= 0 || nvec > n) nvec = n;
    Work* wp;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        wp = &g_work[st];
    }
    Work& wk = *wp;
    int dev = 0;
    AERO_CUDA(cudaGetDevice(&dev));
    const size_t smem = trd_smem(n);
    if (!wk.bar) {
        AERO_CUDA(cudaMalloc(&wk.bar, 64));
        const size_t smax = trd_smem(kEighLargeMax);
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_cluster<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sytrd_cluster_smem(256, 8)));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_cluster<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sytrd_cluster_smem(kSytrdClusterMax, 16)));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_cluster<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_rows<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sytrd_rows_smem(kSytrdRowsMax, SR_R)));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_rows<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sytrd_rows_smem(kSytrdRowsMax, SR_R)));
        AERO_CUDA(cudaFuncSetAttribute(k_sytrd_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * (kSytrdSmall * kSytrdSmall + 2 * kSytrdSmall + 64))));
        AERO_CUDA(cudaFuncSetAttribute(k_bisect, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(2 * sizeof(double) * kEighLargeMax)));
        AERO_CUDA(cudaFuncSetAttribute(k_twisted, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
        AERO_CUDA(cudaFuncSetAttribute(k_cluster_orth, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max({sizeof(double) * kEighLargeMax, cluster_orth_smem(256), cluster_orth_smem(kPanelMaxN)})));
        AERO_CUDA(cudaFuncSetAttribute(k_larft, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * (BT_NB * BT_NB + BT_NB * (BT_NB - 1) / 2))));
        int sms = 0;
        AERO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        wk.grid = sms;  // one CTA per SM (cooperative residency)
    }
    // CTAs: enough that the symv columns spread, few enough that barriers stay cheap
    // CTAs: enough that the symv columns spread (and 4 rows per warp cover n),
    // few enough that barriers stay cheap
    static const int g_env = getenv("AERO_SYTRD_CTAS") ? atoi(getenv("AERO_SYTRD_CTAS")) : 0;  // dev sweep
    const int G = std::max((n + 31) / 32, std::min(g_env > 0 ? g_env : wk.grid, (n + 13) / 14));
    const size_t n2 = (size_t)n * n;
    wk.V.alloc(n2);
    wk.W.alloc((size_t)n * TRD_NB);
    wk.vec.alloc((size_t)11 * n + (size_t)SLOTW * wk.grid + 2 * TRD_NB * TRD_DSPLIT + 8 + 512);
    double* d = wk.vec.p;
    double* e = d + n;
    double* tau = e + n;
    double* y0 = tau + n;
    double* wpre = y0 + n;
    double* ybuf = wpre + n;
    double* e2 = ybuf + n;
    double* lam = e2 + n;
    double* slots = lam + n + n;
    double* dots = slots + SLOTW * wk.grid;
    double* bounds = dots + 2 * TRD_NB * TRD_DSPLIT;
    int* blk = reinterpret_cast<int*>(bounds + 8);       // 2n ints
    int* order = blk + 2 * n;                            // n ints
    int* hist = order + n;                               // 1024 ints: coarse Sturm counts
    fill_zero(st, wk.V.p, (int64_t)n2);
    fill_zero(st, e, n);
    fill_zero(st, tau, n);
    AERO_CUDA(cudaMemsetAsync(wk.bar, 0, sizeof(unsigned), st));

    static const bool trd_prof = getenv("AERO_SYTRD_PROF") != nullptr;
    unsigned long long* prof = nullptr;
    if (trd_prof) {
        AERO_CUDA(cudaMalloc(&prof, 16 * sizeof(unsigned long long)));
        AERO_CUDA(cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), st));
    }
    TrdArgs ta{n, lda, A, wk.V.p, wk.W.p, d, e, tau, ybuf, wpre, y0, slots, dots, wk.bar, prof};
    void* args[] = {&ta};
    const bool vec = !(lda & 1) && !((uintptr_t)A & 15);
    static const bool no_rows = getenv("AERO_SYTRD_ROWS") && atoi(getenv("AERO_SYTRD_ROWS")) == 0;  // dev A/B
    note_launch();
    if (n <= kSytrdSmall) {
        k_sytrd_small<<<1, n <= 64 ? 128 : 512, sizeof(double) * ((size_t)n * n + 2 * n + 64), st>>>(n, A, lda, wk.V.p,
                                                                                                      d, e, tau);
        AERO_LAUNCHED();
    } else if (n <= kSytrdClusterMax) {
        const int cs = (n <= 256) ? 8 : 16;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = sytrd_cluster_smem(n, cs);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        static const bool cl_prof = getenv("AERO_SYTRD_PROF") != nullptr;
        unsigned long long* cprof = nullptr;
        if (cl_prof) {
            AERO_CUDA(cudaMalloc(&cprof, 8 * sizeof(unsigned long long)));
            AERO_CUDA(cudaMemsetAsync(cprof, 0, 8 * sizeof(unsigned long long), st));
        }
        if (cs == 8)
            AERO_CUDA(cudaLaunchKernelEx(&cfg, k_sytrd_cluster<8>, n, (const double*)A, lda, wk.V.p, d, e, tau, cprof));
        else
            AERO_CUDA(cudaLaunchKernelEx(&cfg, k_sytrd_cluster<16>, n, (const double*)A, lda, wk.V.p, d, e, tau, cprof));
        if (cprof) {
            unsigned long long h[8];
            AERO_CUDA(cudaMemcpyAsync(h, cprof, sizeof(h), cudaMemcpyDeviceToHost, st));
            AERO_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "sytrd_cluster n=%d cs=%d kcycles: own %.0f sync1 %.0f - %.0f symv %.0f sync2 %.0f w %.0f upd %.0f\n",
                    n, cs, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, h[6] / 1e3);
            cudaFree(cprof);
        }
    } else if (n <= kSytrdRowsMax && (n + wk.grid - 1) / wk.grid <= SR_R && !no_rows) {
        // matrix resident in shared memory, one grid barrier per column
        const int Gr = wk.grid, R = (n + Gr - 1) / Gr;
        wk.pub.alloc((size_t)4 * n);
        SrArgs sa{n, lda, R, A, wk.V.p, d, e, tau, wk.pub.p, wk.pub.p + 2 * (size_t)n, wk.bar, prof};
        void* sargs[] = {&sa};
        static const int nt_env = getenv("AERO_SYTRD_NT") ? atoi(getenv("AERO_SYTRD_NT")) : 512;  // dev A/B
        if (nt_env == 256)
            AERO_CUDA(cudaLaunchCooperativeKernel((void*)k_sytrd_rows<256>, dim3(Gr), dim3(256), sargs,
                                                  sytrd_rows_smem(n, R), st));
        else
            AERO_CUDA(cudaLaunchCooperativeKernel((void*)k_sytrd_rows<512>, dim3(Gr), dim3(512), sargs,
                                                  sytrd_rows_smem(n, R), st));
    } else {
        AERO_CUDA(cudaLaunchCooperativeKernel(vec ? (void*)k_sytrd<true> : (void*)k_sytrd<false>, dim3(G),
                                              dim3(TRD_THREADS), args, smem, st));
    }
    if (prof && n <= kSytrdRowsMax && !no_rows) {
        unsigned long long h[16];
        AERO_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "sytrd_rows n=%d us: reflector %.0f pass %.0f rowsum+publish %.0f barrier %.0f update+next %.0f\n",
                n, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3);
        cudaFree(prof);
        prof = nullptr;
    }
    if (prof) {
        unsigned long long h[16];
        AERO_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st));
        AERO_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "sytrd n=%d G=%d kcycles: R %.0f B %.0f bar1 %.0f C %.0f bar2 %.0f A' %.0f bar3 %.0f trail %.0f bar4+load %.0f\n",
                n, G, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, h[6] / 1e3,
                h[7] / 1e3, h[8] / 1e3);
        cudaFree(prof);
    }

    note_launch();
    k_tri_prep<<<1, 1024, 0, st>>>(n, d, e, e2, bounds, blk);
    AERO_LAUNCHED();
    const size_t sde = 2 * sizeof(double) * (size_t)n;
    note_launch();
    if (nvec < n - 1 && n >= 256) {  // only the top nvec + 1 eigenvalues are needed
        note_launch();
        k_cut_coarse<<<32, 32, 0, st>>>(n, n - nvec - 1, d, e2, bounds, hist);
        AERO_LAUNCHED();
    } else {
        const double nocut[3] = {-DBL_MAX, 0.0, 0.0};  // bounds[4..6]: no cut, no coarse counts
        AERO_CUDA(cudaMemcpyAsync(bounds + 4, nocut, sizeof(nocut), cudaMemcpyHostToDevice, st));
    }
    k_bisect<<<(n * 32 + 127) / 128, 128, sde, st>>>(n, d, e2, bounds, blk, lam, hist);
    AERO_LAUNCHED();
    note_launch();
    k_order<<<(n + 127) / 128, 128, 0, st>>>(n, lam, order, w);
    AERO_LAUNCHED();

    // eigenvectors of T for the top nvec eigenvalues
    wk.Dp.alloc((size_t)n * nvec);
    wk.Z.alloc((size_t)n * nvec);
    note_launch();
    wk.L.alloc((size_t)3 * n * nvec);
    {  // per-thread scratch in shared memory when 2 n x threads doubles fit
        // per-thread qd scratch (2n doubles) in shared memory: 32 vectors per CTA
        // when they fit, else as many as fit (>= 2), else interleaved in global
        // memory (L2); eigh n = 1024: 11.66 -> 11.34 ms, n = 512: 4.87 -> 4.71 ms
        static const bool tw_global = getenv("AERO_TWISTED_GLOBAL") != nullptr;  // dev A/B switch
        const size_t per_vec = 2 * sizeof(double) * (size_t)n, budget = 200 * 1024;
        int tb = 32;
        if (sde + per_vec * tb > budget) tb = (budget > sde) ? (int)std::min<size_t>(32, (budget - sde) / per_vec) : 0;
        // (only while the vectors still run in one wave: at n = 2048 the 5-lane
        // CTAs need several waves and the one-wave global variant wins, 1.55 vs 2.7 ms)
        const bool usm = !tw_global && tb >= 2 && (nvec + tb - 1) / tb <= wk.grid;
        if (!usm) tb = 32;
        const size_t sm_tw = sde + (usm ? per_vec * tb : 0);
        k_twisted<<<(nvec + tb - 1) / tb, tb, sm_tw, st>>>(n, nvec, d, e, lam, w, order, blk, bounds, wk.Dp.p,
                                                          wk.L.p, wk.L.p + (size_t)n * nvec,
                                                          wk.L.p + (size_t)2 * n * nvec, wk.Z.p, usm ? 1 : 0);
    }
    AERO_LAUNCHED();
    note_launch();
    k_cluster_orth<<<nvec, 256, cluster_orth_smem(n), st>>>(n, nvec, w, bounds, wk.Z.p);
    AERO_LAUNCHED();
    if (n <= 128) {  // direct reflector application + sign fix, warp per vector
        note_launch();
        k_backtransform_small<<<(nvec + 7) / 8, 256, sizeof(double) * 8 * (size_t)n, st>>>(n, nvec, wk.V.p, tau,
                                                                                          wk.Z.p, A, lda);
        AERO_LAUNCHED();
        return;
    }
    // Y = columns; then back-transform Y <- Q Y, Q = H_0 ... H_{n-2}
    const int ldy = (n + 1) & ~1;
    wk.Y.alloc((size_t)ldy * nvec);
    double* Y = wk.Y.p;
    note_launch();
    k_interleaved_to_cols<<<dim3((n + 31) / 32, (nvec + 31) / 32), dim3(32, 8), 0, st>>>(n, nvec, wk.Z.p, Y, ldy);
    AERO_LAUNCHED();
    const int nref = n - 1;  // reflectors j = 0 .. n-2 (rows j+1 ..)
    const int nblk = (nref + BT_NB - 1) / BT_NB;
    wk.S.alloc((size_t)nblk * BT_NB * BT_NB);
    wk.T.alloc((size_t)nblk * BT_NB * BT_NB);
    wk.M1.alloc((size_t)BT_NB * nvec);
    wk.M2.alloc((size_t)BT_NB * nvec);
    const size_t wsn = std::max((size_t)8 * BT_NB * std::max(nvec, BT_NB), (size_t)4 * n * nvec);  // split-K partials
    wk.ws.alloc(wsn);
    // row j0 of block b is zero in every reflector of the block: start there (keeps 16 B alignment)
    for (int b = 0; b < nblk; ++b) {
        const int j0 = b * BT_NB, nb = std::min(BT_NB, nref - j0), mr = n - j0;
        const double* Vb = wk.V.p + j0 + (size_t)j0 * n;
        gemm_acc(st, true, false, nb, nb, mr, 1.0, Vb, n, Vb, n, 0.0, wk.S.p + (size_t)b * BT_NB * BT_NB, BT_NB,
                 wk.ws.p, wsn);
    }
    note_launch();
    k_larft<<<nblk, 4 * BT_NB, sizeof(double) * (BT_NB * BT_NB + BT_NB * (BT_NB - 1) / 2), st>>>(nref, wk.S.p, tau, wk.T.p);
    AERO_LAUNCHED();
    for (int b = nblk - 1; b >= 0; --b) {
        const int j0 = b * BT_NB, nb = std::min(BT_NB, nref - j0), mr = n - j0;
        const double* Vb = wk.V.p + j0 + (size_t)j0 * n;  // mr x nb, ld n
        const double* Tb = wk.T.p + (size_t)b * BT_NB * BT_NB;
        // M1 = Vb^T Y[j0:, :] ; M2 = T M1 ; Y[j0:, :] -= Vb M2
        gemm_acc(st, true, false, nb, nvec, mr, 1.0, Vb, n, Y + j0, ldy, 0.0, wk.M1.p, BT_NB, wk.ws.p, wsn);
        gemm_acc(st, false, false, nb, nvec, nb, 1.0, Tb, BT_NB, wk.M1.p, BT_NB, 0.0, wk.M2.p, BT_NB,
                 wk.ws.p, wsn);
        gemm_acc(st, false, false, mr, nvec, nb, -1.0, Vb, n, wk.M2.p, BT_NB, 1.0, Y + j0, ldy, wk.ws.p, wsn);
    }
    copy_matrix(st, n, nvec, Y, ldy, A, lda);
    fix_column_signs(st, n, nvec, A, lda, nullptr);
}

void eigh_large_forget(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_work.find(st);
    if (it == g_work.end()) return;
    if (it->second.bar) cudaFree(it->second.bar);
    g_work.erase(it);
}

}  // namespace aero_b200
