// The large fp64 contractions of the update path, led by the dominant one:
// the batched power / subspace iteration product Y = G X (G: R x R Gram of the
// row buffer, X: R x N job columns; reference linalg.cpp:109-118 and :141-143
// in Gram form), plus the buffer-append Gram block (C'^T C'_new, K = d) and
// the FD-reduce rotation / re-Gram.
// fp64 DFMA, 128x64 CTA tile, 8x8 register micro-tile per thread (DFMA-bound,
// shared memory at ~50%), 3-stage cp.async pipeline over 16-deep K slices, and
// a deterministic split-K (fixed-order reduction) so skinny shapes fill all
// 148 SMs with two CTAs each. Column-major; op(A) = A or A^T, op(B) = B or B^T.
// Rows >= colmask[j] of output column j are written as 0 (job prefix lengths).
#include <algorithm>
#include <cstdlib>

#include "aero_common.cuh"
#include "kernels.cuh"
#include "tiles.cuh"

namespace aero_b200 {

namespace {
using namespace tiles;
constexpr int kMaxSplits = 32;
// A tile: !TA -> a[k][m] (m contiguous); TA -> a[m][k] (k contiguous, ld KLD)
// B tile: !TB -> b[n][k] (k contiguous, ld KLD); TB -> b[k][n] (n contiguous)
template <bool TA, bool TB>
__global__ void __launch_bounds__(PNT, 2)
    k_product(int M, int N, int K, int kchunk, const double* __restrict__ A, int lda,
              const double* __restrict__ B, int ldb, double* __restrict__ out, int ldo,
              int64_t split_stride, const int* __restrict__ colmask, int direct, double alpha,
              double beta) {
    extern __shared__ __align__(16) double smd[];
    double* sa = smd;
    double* sb = smd + PST * A_TILE;
    const int tid = threadIdx.x, tr = tid % 16, tc = tid / 16;
    const int bm = blockIdx.y * PBM, bn = blockIdx.x * PBN;
    const int k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
    const int nk = (k1 > k0) ? (k1 - k0 + PBK - 1) / PBK : 0;

    auto load_tile = [&](int stage, int kt) {
        const int kb = k0 + kt * PBK;
        double* ta = sa + stage * A_TILE;
        double* tb = sb + stage * B_TILE;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // A: 1024 16-byte chunks
            const int idx = tid + i * PNT;
            int gm, gk, bytes = 0;
            double* dst;
            if (!TA) {  // column gk of A: 128 contiguous m
                const int col = idx >> 6, r2 = idx & 63;
                gk = kb + col;
                gm = bm + 2 * r2;
                dst = ta + col * PBM + 2 * r2;
                if (gk < k1 && gm < M) bytes = (M - gm >= 2) ? 16 : 8;
            } else {  // row gm of op(A): 16 contiguous k
                const int row = idx >> 3, k2 = idx & 7;
                gm = bm + row;
                gk = kb + 2 * k2;
                dst = ta + row * KLD + 2 * k2;
                if (gm < M && gk < k1) bytes = (k1 - gk >= 2) ? 16 : 8;
            }
            const double* src = bytes ? (TA ? A + gk + (int64_t)gm * lda : A + gm + (int64_t)gk * lda) : A;
            cp_async16(dst, src, bytes);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // B: 512 16-byte chunks
            const int idx = tid + i * PNT;
            int gn, gk, bytes = 0;
            double* dst;
            if (!TB) {  // column gn of B: 16 contiguous k
                const int col = idx >> 3, k2 = idx & 7;
                gn = bn + col;
                gk = kb + 2 * k2;
                dst = tb + col * KLD + 2 * k2;
                if (gn < N && gk < k1) bytes = (k1 - gk >= 2) ? 16 : 8;
            } else {  // row gk of op(B): 64 contiguous n
                const int row = idx >> 5, n2 = idx & 31;
                gk = kb + row;
                gn = bn + 2 * n2;
                dst = tb + row * PBN + 2 * n2;
                if (gk < k1 && gn < N) bytes = (N - gn >= 2) ? 16 : 8;
            }
            const double* src = bytes ? (TB ? B + gn + (int64_t)gk * ldb : B + gk + (int64_t)gn * ldb) : B;
            cp_async16(dst, src, bytes);
        }
    };

    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

#pragma unroll
    for (int s0 = 0; s0 < PST - 1; ++s0) {
        if (s0 < nk) load_tile(s0, s0);
        cp_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % PST;
        cp_wait<PST - 2>();  // tile kt has landed
        __syncthreads();     // and every warp is done with the stage reloaded below
        if (kt + PST - 1 < nk) load_tile((kt + PST - 1) % PST, kt + PST - 1);
        cp_commit();
        const double* ta = sa + st * A_TILE;
        const double* tb = sb + st * B_TILE;
#pragma unroll
        for (int kk = 0; kk < PBK; ++kk) {
            double av[8], bv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                av[i] = TA ? ta[(tr + 16 * i) * KLD + kk] : ta[kk * PBM + tr + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                bv[j] = TB ? tb[kk * PBN + tc + 8 * j] : tb[(tc + 8 * j) * KLD + kk];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
    }
    cp_wait<0>();

    double* o = out + (direct ? 0 : (int64_t)blockIdx.z * split_stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int gn = bn + tc + 8 * j;
        if (gn >= N) continue;
        const int lim = (direct && colmask) ? colmask[gn] : M;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int gm = bm + tr + 16 * i;
            if (gm >= M) continue;
            double* dst = o + gm + (int64_t)gn * ldo;
            if (!direct || (alpha == 1.0 && beta == 0.0)) *dst = (gm < lim) ? acc[i][j] : 0.0;
            else *dst = (gm < lim) ? fma(alpha, acc[i][j], beta == 0.0 ? 0.0 : beta * *dst) : 0.0;
        }
    }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(PNT, 2)
    k_product_mma(int M, int N, int K, int kchunk, const double* __restrict__ A, int lda,
                  const double* __restrict__ B, int ldb, double* __restrict__ out, int ldo,
                  int64_t split_stride, const int* __restrict__ colmask, int direct, double alpha,
                  double beta) {
    extern __shared__ __align__(16) double smd[];
    mma_tile<TA, TB>(blockIdx.x, blockIdx.y, blockIdx.z, M, N, K, kchunk, A, lda, B, ldb, out, ldo,
                     split_stride, colmask, direct, alpha, beta, smd);
}

// fixed-order sum of the split-K partials + row mask
__global__ void k_product_reduce(int M, int N, int splits, const double* __restrict__ ws,
                                 int64_t split_stride, double* __restrict__ Y, int ldy,
                                 const int* __restrict__ colmask, double alpha, double beta) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)M * N) return;
    const int i = (int)(e % M), j = (int)(e / M);
    double v = 0.0;
    for (int z = 0; z < splits; ++z) v += ws[z * split_stride + e];
    double* dst = Y + i + (int64_t)j * ldy;
    if (alpha != 1.0 || beta != 0.0) v = fma(alpha, v, beta == 0.0 ? 0.0 : beta * *dst);
    if (colmask && i >= colmask[j]) v = 0.0;
    *dst = v;
}

bool use_mma() {
    static const int v = getenv("AERO_PRODUCT_DFMA") ? 0 : 1;  // dev A/B switch
    return v;
}

template <bool TA, bool TB>
void launch(cudaStream_t st, dim3 grid, int M, int N, int K, int kchunk, const double* A, int lda,
            const double* B, int ldb, double* out, int ldo, int64_t sstride, const int* colmask,
            int direct, double alpha, double beta) {
    if (use_mma()) {
        static bool attr_m = false;
        if (!attr_m) {
            AERO_CUDA(cudaFuncSetAttribute(k_product_mma<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)MMA_SMEM));
            attr_m = true;
        }
        k_product_mma<TA, TB><<<grid, PNT, MMA_SMEM, st>>>(M, N, K, kchunk, A, lda, B, ldb, out, ldo, sstride,
                                                           colmask, direct, alpha, beta);
        AERO_LAUNCHED();
        return;
    }
    static bool attr = false;
    if (!attr) {
        AERO_CUDA(cudaFuncSetAttribute(k_product<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)PROD_SMEM));
        attr = true;
    }
    k_product<TA, TB><<<grid, PNT, PROD_SMEM, st>>>(M, N, K, kchunk, A, lda, B, ldb, out, ldo,
                                                    sstride, colmask, direct, alpha, beta);
    AERO_LAUNCHED();
}
}  // namespace

size_t product_workspace_doubles(int M, int N) { return (size_t)kMaxSplits * M * N; }

namespace {
bool gemm_core(cudaStream_t st, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
               int lda, const double* B, int ldb, double beta, double* Y, int ldy, const int* colmask,
               double* ws, size_t ws_doubles, int* splits_used, bool defer_reduce) {
    if (M <= 0 || N <= 0) return true;
    // 16-byte cp.async needs even leading dimensions and aligned bases
    if ((lda & 1) || (ldb & 1) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15)) return false;
    const int tiles = ((M + PBM - 1) / PBM) * ((N + PBN - 1) / PBN);
    // split-K so the grid fills ~2 CTAs per SM (148 SMs), up to 32 ways, each
    // split >= 4 K slices, partials must fit the workspace
    int splits = std::max(1, std::min(kMaxSplits, (296 + tiles / 2) / tiles));
    const int kt_total = (K + PBK - 1) / PBK;
    splits = std::min(splits, std::max(1, kt_total / 4));
    if (!ws) splits = 1;
    while (splits > 1 && (size_t)splits * M * N > ws_doubles) --splits;
    const int kchunk = ((kt_total + splits - 1) / splits) * PBK;
    dim3 grid((N + PBN - 1) / PBN, (M + PBM - 1) / PBM, splits);
    const int64_t sstride = (int64_t)M * N;
    double* o = splits == 1 ? Y : ws;
    const int ldo = splits == 1 ? ldy : M;
    const int direct = splits == 1;
    if (!ta && !tb) launch<false, false>(st, grid, M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride, colmask, direct, alpha, beta);
    else if (ta && !tb) launch<true, false>(st, grid, M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride, colmask, direct, alpha, beta);
    else if (!ta && tb) launch<false, true>(st, grid, M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride, colmask, direct, alpha, beta);
    else launch<true, true>(st, grid, M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride, colmask, direct, alpha, beta);
    if (splits_used) *splits_used = splits;
    if (splits > 1 && !defer_reduce) {
        const int64_t tot = (int64_t)M * N;
        k_product_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, splits, ws, sstride, Y,
                                                                        ldy, colmask, alpha, beta);
        AERO_LAUNCHED();
    }
    return true;
}
}  // namespace

bool gemm_big(cudaStream_t st, bool ta, bool tb, int M, int N, int K, const double* A, int lda,
              const double* B, int ldb, double* Y, int ldy, const int* colmask, double* ws,
              size_t ws_doubles, int* splits_used, bool defer_reduce) {
    return gemm_core(st, ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, Y, ldy, colmask, ws, ws_doubles,
                     splits_used, defer_reduce);
}

void gemm_acc(cudaStream_t st, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
              int lda, const double* B, int ldb, double beta, double* Y, int ldy, double* ws,
              size_t ws_doubles) {
    if (!gemm_core(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Y, ldy, nullptr, ws, ws_doubles,
                   nullptr, false))
        dgemm(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Y, ldy);
}

void gemm_product(cudaStream_t st, int M, int N, int K, const double* A, int lda, const double* B,
                  int ldb, double* Y, int ldy, const int* colmask, double* ws, size_t ws_doubles) {
    if (!gemm_big(st, false, false, M, N, K, A, lda, B, ldb, Y, ldy, colmask, ws, ws_doubles))
        dgemm(st, false, false, M, N, K, 1.0, A, lda, B, ldb, 0.0, Y, ldy, colmask);
}

}  // namespace aero_b200
