// Shared device building blocks of the fp64 products: tile constants, cp.async
// helpers and the DMMA (mma.sync.m8n8k4.f64) 128 x 64 tile used by
// k_product_mma (product.cu) and the persistent iteration kernel (kernels.cu).
#pragma once

#include "aero_common.cuh"

namespace aero_b200 {
namespace tiles {
constexpr int PBM = 128, PBN = 64, PBK = 16, PNT = 128, PST = 3;  // PST cp.async stages
constexpr int KLD = PBK + 2;  // padded k-stride for k-contiguous tiles (16B aligned rows)
constexpr int A_TILE = (PBM * KLD > PBK * PBM) ? PBM * KLD : PBK * PBM;
constexpr int B_TILE = (PBN * KLD > PBK * PBN) ? PBN * KLD : PBK * PBN;
constexpr size_t PROD_SMEM = sizeof(double) * (size_t)PST * (A_TILE + B_TILE);

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

// ---- fp64 tensor-core (DMMA, mma.sync.m8n8k4.f64) variant -----------------
// Same CTA tile (128 x 64), loader and split-K as k_product; 4 warps as 2 x 2,
// warp tile 64 x 32 = 8 x 4 m8n8 fragments, 64 fp64 accumulators per lane.
// Shared tiles padded so the fragment loads of a warp take the minimum two
// wavefronts: [k][m] ld 136, [m|n][k] ld 20, [k][n] ld 72.
constexpr int MLDM = PBM + 8, MLDN = PBN + 8, MKLD = PBK + 4;
constexpr int MA_TILE = (PBK * MLDM > PBM * MKLD) ? PBK * MLDM : PBM * MKLD;
constexpr int MB_TILE = (PBK * MLDN > PBN * MKLD) ? PBK * MLDN : PBN * MKLD;
constexpr size_t MMA_SMEM = sizeof(double) * (size_t)PST * (MA_TILE + MB_TILE);

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// one 128 x 64 output tile (tile coordinates tn, tm, split tz) by the first
// 128 threads of a CTA; smd: MMA_SMEM bytes of shared memory
template <bool TA, bool TB>
__device__ __forceinline__ void mma_tile(int tn, int tm, int tz, int M, int N, int K, int kchunk,
                                         const double* __restrict__ A, int lda, const double* __restrict__ B,
                                         int ldb, double* __restrict__ out, int ldo, int64_t split_stride,
                                         const int* __restrict__ colmask, int direct, double alpha, double beta,
                                         double* smd) {
    double* sa = smd;
    double* sb = smd + PST * MA_TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;
    const int bm = tm * PBM, bn = tn * PBN;
    const int k0 = tz * kchunk, k1 = min(K, k0 + kchunk);
    const int nk = (k1 > k0) ? (k1 - k0 + PBK - 1) / PBK : 0;

    auto load_tile = [&](int stage, int kt) {
        const int kb = k0 + kt * PBK;
        double* ta = sa + stage * MA_TILE;
        double* tb = sb + stage * MB_TILE;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // A: 1024 16-byte chunks
            const int idx = tid + i * PNT;
            int gm, gk, bytes = 0;
            double* dst;
            if (!TA) {
                const int col = idx >> 6, r2 = idx & 63;
                gk = kb + col;
                gm = bm + 2 * r2;
                dst = ta + col * MLDM + 2 * r2;
                if (gk < k1 && gm < M) bytes = (M - gm >= 2) ? 16 : 8;
            } else {
                const int row = idx >> 3, k2 = idx & 7;
                gm = bm + row;
                gk = kb + 2 * k2;
                dst = ta + row * MKLD + 2 * k2;
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
            if (!TB) {
                const int col = idx >> 3, k2 = idx & 7;
                gn = bn + col;
                gk = kb + 2 * k2;
                dst = tb + col * MKLD + 2 * k2;
                if (gn < N && gk < k1) bytes = (k1 - gk >= 2) ? 16 : 8;
            } else {
                const int row = idx >> 5, n2 = idx & 31;
                gk = kb + row;
                gn = bn + 2 * n2;
                dst = tb + row * MLDN + 2 * n2;
                if (gk < k1 && gn < N) bytes = (N - gn >= 2) ? 16 : 8;
            }
            const double* src = bytes ? (TB ? B + gn + (int64_t)gk * ldb : B + gk + (int64_t)gn * ldb) : B;
            cp_async16(dst, src, bytes);
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s0 = 0; s0 < PST - 1; ++s0) {
        if (s0 < nk) load_tile(s0, s0);
        cp_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % PST;
        cp_wait<PST - 2>();
        __syncthreads();
        if (kt + PST - 1 < nk) load_tile((kt + PST - 1) % PST, kt + PST - 1);
        cp_commit();
        const double* ta = sa + st * MA_TILE;
        const double* tb = sb + st * MB_TILE;
#pragma unroll
        for (int kk = 0; kk < PBK; kk += 4) {
            const int k = kk + tg;
            double af[8], bf[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int m = wm + 8 * i + g;
                af[i] = TA ? ta[m * MKLD + k] : ta[k * MLDM + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = wn + 8 * j + g;
                bf[j] = TB ? tb[k * MLDN + n] : tb[n * MKLD + k];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_wait<0>();

    double* o = out + (direct ? 0 : (int64_t)tz * split_stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gn = bn + wn + 8 * j + 2 * tg + h;
            if (gn >= N) continue;
            const int lim = (direct && colmask) ? colmask[gn] : M;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int gm = bm + wm + 8 * i + g;
                if (gm >= M) continue;
                double* dst = o + gm + (int64_t)gn * ldo;
                const double v = acc[i][j][h];
                if (!direct || (alpha == 1.0 && beta == 0.0)) *dst = (gm < lim) ? v : 0.0;
                else *dst = (gm < lim) ? fma(alpha, v, beta == 0.0 ? 0.0 : beta * *dst) : 0.0;
            }
        }
    }
}

}  // namespace tiles
}  // namespace aero_b200
