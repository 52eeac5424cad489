// The dominant kernel of the update path: the batched power / subspace
// iteration product Y = G X (G: R x R Gram of the row buffer, X: R x N job
// columns; reference linalg.cpp:109-118 and :141-143 in Gram form).
// fp64 DFMA, 128x64 CTA tile, 8x8 register micro-tile per thread (DFMA-bound,
// shared memory at ~50%), cp.async double-buffered 16-deep K slices, and a
// deterministic split-K (fixed-order reduction) so that R ~ 2048, N ~ 192
// fills all 148 SMs. Column-major throughout; rows >= colmask[j] of output
// column j are written as 0 (each job's prefix length).
#include "aero_common.cuh"
#include "kernels.cuh"

namespace aero_b200 {

namespace {
constexpr int PBM = 128, PBN = 64, PBK = 16, PNT = 128, PST = 3;  // PST cp.async stages
constexpr int BLD = PBK + 2;  // padded k-stride of the B tile (conflict-free)
struct ProdSmem {
    double a[PST][PBK][PBM];
    double b[PST][PBN][BLD];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__global__ void __launch_bounds__(PNT, 2)
    k_product(int M, int N, int K, int kchunk, const double* __restrict__ A, int lda,
              const double* __restrict__ B, int ldb, double* __restrict__ out, int ldo,
              int64_t split_stride, const int* __restrict__ colmask, int direct) {
    extern __shared__ __align__(16) unsigned char smraw[];
    ProdSmem& s = *reinterpret_cast<ProdSmem*>(smraw);
    const int tid = threadIdx.x, tr = tid % 16, tc = tid / 16;
    const int bm = blockIdx.y * PBM, bn = blockIdx.x * PBN;
    const int k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
    const int nk = (k1 > k0) ? (k1 - k0 + PBK - 1) / PBK : 0;

    auto load_tile = [&](int stage, int kt) {
        const int kb = k0 + kt * PBK;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // A: 16 k-columns x 64 double2
            const int idx = tid + i * PNT;
            const int col = idx >> 6, r2 = idx & 63;
            const int gk = kb + col, gm = bm + 2 * r2;
            int bytes = 0;
            const double* src = A;
            if (gk < k1 && gm < M) {
                bytes = (M - gm >= 2) ? 16 : 8;
                src = A + gm + (int64_t)gk * lda;
            }
            cp_async16(&s.a[stage][col][2 * r2], src, bytes);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // B: 64 n-columns x 8 double2 (k)
            const int idx = tid + i * PNT;
            const int col = idx >> 3, k2 = idx & 7;
            const int gn = bn + col, gk = kb + 2 * k2;
            int bytes = 0;
            const double* src = B;
            if (gn < N && gk < k1) {
                bytes = (k1 - gk >= 2) ? 16 : 8;
                src = B + gk + (int64_t)gn * ldb;
            }
            cp_async16(&s.b[stage][col][2 * k2], src, bytes);
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
#pragma unroll
        for (int kk = 0; kk < PBK; ++kk) {
            double av[8], bv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) av[i] = s.a[st][kk][tr + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) bv[j] = s.b[st][tc + 8 * j][kk];
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
            o[gm + (int64_t)gn * ldo] = (gm < lim) ? acc[i][j] : 0.0;
        }
    }
}

// fixed-order sum of the split-K partials + row mask
__global__ void k_product_reduce(int M, int N, int splits, const double* __restrict__ ws,
                                 int64_t split_stride, double* __restrict__ Y, int ldy,
                                 const int* __restrict__ colmask) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)M * N) return;
    const int i = (int)(e % M), j = (int)(e / M);
    double v = 0.0;
    for (int z = 0; z < splits; ++z) v += ws[z * split_stride + e];
    if (colmask && i >= colmask[j]) v = 0.0;
    Y[i + (int64_t)j * ldy] = v;
}
}  // namespace

size_t product_workspace_doubles(int M, int N) { return (size_t)8 * M * N; }

void gemm_product(cudaStream_t st, int M, int N, int K, const double* A, int lda, const double* B,
                  int ldb, double* Y, int ldy, const int* colmask, double* ws, size_t ws_doubles) {
    if (M <= 0 || N <= 0) return;
    static bool attr = false;
    if (!attr) {
        AERO_CUDA(cudaFuncSetAttribute(k_product, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(ProdSmem)));
        attr = true;
    }
    const int tiles = ((M + PBM - 1) / PBM) * ((N + PBN - 1) / PBN);
    // two resident CTAs per SM (2 x 77 KB shared memory): target 296 CTAs
    int splits = std::max(1, std::min(8, (296 + tiles / 2) / tiles));
    const int kt_total = (K + PBK - 1) / PBK;
    splits = std::min(splits, std::max(1, kt_total / 4));  // >= 4 K slices per split
    if ((size_t)splits * M * N > ws_doubles) splits = 1;
    const int kchunk = ((kt_total + splits - 1) / splits) * PBK;
    dim3 grid((N + PBN - 1) / PBN, (M + PBM - 1) / PBM, splits);
    if (splits == 1) {
        k_product<<<grid, PNT, sizeof(ProdSmem), st>>>(M, N, K, kchunk, A, lda, B, ldb, Y, ldy, 0,
                                                       colmask, 1);
        AERO_LAUNCHED();
        return;
    }
    const int64_t sstride = (int64_t)M * N;
    k_product<<<grid, PNT, sizeof(ProdSmem), st>>>(M, N, K, kchunk, A, lda, B, ldb, ws, M, sstride,
                                                   nullptr, 0);
    AERO_LAUNCHED();
    const int64_t tot = (int64_t)M * N;
    k_product_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, splits, ws, sstride, Y,
                                                                    ldy, colmask);
    AERO_LAUNCHED();
}

}  // namespace aero_b200
