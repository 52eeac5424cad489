// Device side of the exact int8 slicing (Ozaki scheme) shared by the slicing
// kernel (ozaki.cu) and the iteration normalization (kernels.cu), which
// slices each new iterate column as it writes it.
#pragma once

#include <cstdint>

#include "aero_common.cuh"
#include "ozaki_slice.h"

namespace aero_b200 {

constexpr int kOzSlices = 6;  // balanced signed 8-bit slices per fp64 value (46 bits + sign, ozaki_slice.h)
constexpr int kOzBK = 64;     // K bytes per tiled block (one pipeline stage)
constexpr int kOzBM = 128;    // G-tile rows (UMMA M)
constexpr int kOzBN = 64;     // X-tile columns (UMMA N)

// cut 8 values (|x| < 2^e) into S balanced signed 8-bit slices, packed 8 per
// uint64 (ozaki_slice.h)
template <int S>
__device__ __forceinline__ void ozaki_slice8(const double (&x)[8], int e, uint64_t (&pk)[S]) {
    ozaki_slice8_int<S>(x, e, pk);
}
template <int S>
__device__ __forceinline__ void ozaki_slice8_pow2(const double (&x)[8], int e, uint64_t (&pk)[S]) {
    ozaki_slice8_int<S>(x, e, pk);
}

template <int S, int TR, int NV>
__device__ inline void ozaki_slice_vectors(const double* __restrict__ v0, int ldv, int lim, int Kp, int i0,
                                           int8_t* __restrict__ out, int* __restrict__ ex, double* red) {
    const int tid = threadIdx.x, nt = blockDim.x, span = 8 * nt, nw = nt / 32;
    const int nkb = Kp / kOzBK;
    auto load8 = [&](const double* v, int k0, double (&x)[8]) {
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = (k0 + u < lim) ? v[k0 + u] : 0.0;
    };
    auto store8 = [&](int i, int k0, const uint64_t (&pk)[S]) {
        const int t = i / TR, r = i % TR;
        const int b = k0 / kOzBK, kk = k0 % kOzBK, kc = kk >> 4;
        int8_t* blk = out + ((int64_t)t * nkb + b) * S * TR * kOzBK + r * kOzBK + ((kc ^ ((r >> 1) & 3)) << 4) +
                      (kk & 15);
#pragma unroll
        for (int p = 0; p < S; ++p) *reinterpret_cast<uint64_t*>(blk + p * TR * kOzBK) = pk[p];
    };
    const int k00 = tid * 8;
    double x0[NV][8], m[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        load8(v0 + (int64_t)c * ldv, k00, x0[c]);
        m[c] = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) m[c] = fmax(m[c], fabs(x0[c][u]));
    }
    for (int k0 = k00 + span; k0 < lim; k0 += span)  // long vectors (Kp > span): extra chunks
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            double x[8];
            load8(v0 + (int64_t)c * ldv, k0, x);
#pragma unroll
            for (int u = 0; u < 8; ++u) m[c] = fmax(m[c], fabs(x[u]));
        }
#pragma unroll
    for (int c = 0; c < NV; ++c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m[c] = fmax(m[c], __shfl_xor_sync(0xffffffffu, m[c], o));
    __syncthreads();
    if ((tid & 31) == 0)
#pragma unroll
        for (int c = 0; c < NV; ++c) red[c * nw + (tid >> 5)] = m[c];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        double mm = 0.0;
        for (int w = 0; w < nw; ++w) mm = fmax(mm, red[c * nw + w]);
        const int e = (mm > 0.0) ? ilogb(mm) + 1 : 0;  // |v| < 2^e
        if (tid == 0) ex[i0 + c] = e;
        uint64_t pk[S];
        if (k00 < Kp) {
            ozaki_slice8<S>(x0[c], e, pk);
            store8(i0 + c, k00, pk);
        }
        for (int k0 = k00 + span; k0 < Kp; k0 += span) {
            double x[8];
            load8(v0 + (int64_t)c * ldv, k0, x);
            ozaki_slice8<S>(x, e, pk);
            store8(i0 + c, k0, pk);
        }
    }
}

// Destination of slices written as a side effect of the normalization (the
// X image of the next product); b == nullptr: none
struct OzSliceDst {
    int8_t* b = nullptr;
    int* fe = nullptr;
    int Kp = 0;
};

// Shared-memory landing zone of one job's split-K partials (normalize_job in
// k_iterate_i8): buf holds cap doubles, bar is an mbarrier (count 1) reused
// with alternating parity; buf == nullptr: partials are read with plain loads
struct OzBulkWs {
    double* buf = nullptr;
    uint64_t* bar = nullptr;
    size_t cap = 0;
};

// the S slices of one value x (|x| < 2^e) at K index k of vector i, as bytes
// of the tiled image (TR vectors per tile)
template <int S, int TR>
__device__ __forceinline__ void ozaki_store_value(int8_t* __restrict__ out, int Kp, int i, int k, double x, int e) {
    const int nkb = Kp / kOzBK, t = i / TR, r = i % TR, b = k / kOzBK, kk = k % kOzBK, kc = kk >> 4;
    int8_t* base = out + ((int64_t)t * nkb + b) * S * TR * kOzBK + r * kOzBK + ((kc ^ ((r >> 1) & 3)) << 4) + (kk & 15);
    int8_t dg[S];
    ozaki_slice1_int<S>(x, e, dg);
#pragma unroll
    for (int p = 0; p < S; ++p) base[p * TR * kOzBK] = dg[p];
}

// Slice vector i (v[0..lim), zero beyond; padded to Kp) into the product
// kernel's tiled image: tiles of TR vectors; block (tile t, K block b) at
// out + (t * nkb + b) * S * TR * 64 holds slice p at p * TR * 64, vector row r
// at 64 r, its 16-byte chunk c at chunk c ^ ((r >> 1) & 3) (64-byte swizzle).
// ex[i] = e with max|v| < 2^e. Whole CTA; red: blockDim.x / 32 doubles (x NV
// for ozaki_slice_vectors, which slices NV vectors v0 + c*ldv at once). Each
// thread owns 8 consecutive entries per 8 * blockDim.x: for Kp <= that span
// the vector is read once (registers), max-reduced, sliced and stored.
template <int S, int TR>
__device__ inline void ozaki_slice_vector(const double* __restrict__ v, int lim, int Kp, int i,
                                          int8_t* __restrict__ out, int* __restrict__ ex, double* red) {
    ozaki_slice_vectors<S, TR, 1>(v, 0, lim, Kp, i, out, ex, red);
}

template <int S>
struct OzCfg {
    static constexpr int A_BYTES = S * kOzBM * kOzBK;
    static constexpr int B_BYTES = S * kOzBN * kOzBK;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    // pipeline stages: as many as fit beside the barriers (3 at S = 6: two
    // bulk loads in flight behind the stage the tensor pipe is reading)
    static constexpr int NST = (3 * STAGE + 2048 + kOzBN * 12 <= 225 * 1024) ? 3 : 2;
    static constexpr int SMEM = NST * STAGE + 1024 + 128 + kOzBN * 12;  // + alignment slack, barriers, column scales
    static constexpr int TMEM_COLS = (S * kOzBN <= 256) ? 256 : 512;
};

// UMMA instruction descriptor: D s32, A/B signed int8, both K-major, M=128, N=64
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOzBN >> 3) << 17) |
                              ((uint32_t)(kOzBM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor, K-major with the 64-byte swizzle: a tile
// is rows x 64 B (row m at 64 m, its 16-byte chunk c stored at chunk
// c ^ ((m >> 1) & 3)); 8-row atoms of 512 B (SBO), LBO unused; the K step of
// 32 bytes inside the atom advances the start address (the hardware applies
// the XOR on address bits [4:5] ^= [7:8], so tiles are 1024-byte aligned);
// descriptor version 1 (sm_100), layout type 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdescI8), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// bulk global -> shared copy completing on an mbarrier (bytes multiple of 16)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15])
        : "r"(taddr));
}


// One work item of the product: rows [bm, bm+128) of G times job columns
// [bn, bn+64) of X over K blocks [kb0, kb0 + nkb), written (fp64) to
// o[m + n*ldo] for rows m < min(M, clim) (clim: direct && colmask ? colmask[n]
// : M). `sm` is 1024-byte aligned shared memory of OzCfg<S>::SMEM - 1024
// bytes, `tmem` an allocation of OzCfg<S>::TMEM_COLS columns; 256 threads.
// Barriers are initialized here, so consecutive calls may reuse `sm`.
// SE <= S: only the leading SE slices of both images take part (diagonals
// t < SE: SE(SE+1)/2 of the S(S+1)/2 slice-pair MMAs, SE/S of the bytes) -- a
// product truncated to 8 SE - 2 bits, an opt-in experiment for the steering
// phases of an iteration (AERO_OZ_SE; the default runs every phase at SE = S).
template <int S, int SE = S>
__device__ inline void ozaki_tile(int M, int N, int nkb_all, int tile_m, int tile_n, int kb0, int nkb,
                                  const int8_t* __restrict__ As, const int8_t* __restrict__ Bs,
                                  const int* __restrict__ ea, const int* __restrict__ fb, double* __restrict__ o,
                                  int ldo, const int* __restrict__ colmask, int direct, uint8_t* sm, uint32_t tmem) {
    static_assert(SE >= 1 && SE <= S, "effective slices");
    using Cfg = OzCfg<S>;
    constexpr int NST = Cfg::NST;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * Cfg::STAGE);
    uint64_t* empty = full + NST;
    uint64_t* done = empty + NST;  // one commit after the last stage: accumulators final
    double* cscale = reinterpret_cast<double*>(done + 2);  // kOzBN per-column 2^(f - 12)
    int* clim = reinterpret_cast<int*>(cscale + kOzBN);    // kOzBN per-column row limits
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bm = tile_m * kOzBM, bn = tile_n * kOzBN;
    __syncthreads();  // previous item (if any) is done with sm and TMEM
    if (tid == 0) {
        for (int b = 0; b < NST; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < kOzBN) {
        const int n = bn + tid;
        // (G X)_ic = 2^(e_i + f_c - 2F) sum_pq d_p d'_q 256^(2(S-1) - p - q), F = 8S - 2:
        // 2^(e_i + f_c - 12) sum_t 2^(-8t) D_t
        cscale[tid] = (n < N) ? ldexp(1.0, fb[n] - 12) : 0.0;
        clim[tid] = (n >= N) ? 0 : ((direct && colmask) ? colmask[n] : M);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t sbase = smem_u32(sm);
    if (tid == 0 && nkb > 0) {  // producer + MMA issuer
        const int8_t* Ablk = As + ((int64_t)tile_m * nkb_all + kb0) * Cfg::A_BYTES;
        const int8_t* Bblk = Bs + ((int64_t)tile_n * nkb_all + kb0) * Cfg::B_BYTES;
        auto load = [&](int st, int kb) {
            const uint32_t dA = sbase + st * Cfg::STAGE;
            // slices are contiguous (p-major) inside a block: the leading SE of them
            constexpr unsigned aB = SE * kOzBM * kOzBK, bB = SE * kOzBN * kOzBK;
            mbar_expect_tx(&full[st], aB + bB);
            bulk_g2s(dA, Ablk + (int64_t)kb * Cfg::A_BYTES, aB, &full[st]);
            bulk_g2s(dA + Cfg::A_BYTES, Bblk + (int64_t)kb * Cfg::B_BYTES, bB, &full[st]);
        };
        for (int kb = 0; kb < NST - 1 && kb < nkb; ++kb) load(kb, kb);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % NST;
            mbar_wait(&full[st], (kb / NST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t aS = sbase + st * Cfg::STAGE, bS = aS + Cfg::A_BYTES;
#pragma unroll
            for (int ks = 0; ks < kOzBK / 32; ++ks) {
#pragma unroll
                for (int p = 0; p < SE; ++p) {
                    const uint64_t da = umma_desc(aS + p * kOzBM * kOzBK + ks * 32);
#pragma unroll
                    for (int q = 0; q < SE - p; ++q) {
                        const uint64_t db = umma_desc(bS + q * kOzBN * kOzBK + ks * 32);
                        mma_i8(tmem + (uint32_t)((p + q) * kOzBN), da, db, (kb > 0 || ks > 0 || p > 0) ? 1u : 0u);
                    }
                }
            }
            umma_commit(&empty[st]);
            // refill the stage the MMAs of kb-1 have drained (those of kb are
            // queued behind them, so the tensor pipe stays busy) with block
            // kb + NST - 1: NST - 1 loads stay in flight
            const int kn = kb + NST - 1;
            if (kn < nkb) {
                const int sn = kn % NST;  // == (kb - 1) % NST
                if (kb >= 1) mbar_wait(&empty[sn], ((kb - 1) / NST) & 1);
                load(sn, kn);
            }
        }
        umma_commit(done);
    }
    __syncwarp();

    // epilogue: warp w reads TMEM lanes 32 (w % 4) + lane = tile row, columns 32 (w / 4) ..
    const int qd = warp & 3, half = warp >> 2;
    const int m = bm + qd * 32 + lane;
    if (nkb > 0) {
        // (a parity wait on a stage barrier could pass on its not-yet-started
        // phase; the single-use barrier cannot)
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    const double rs = (m < M) ? ldexp(1.0, ea[m]) : 0.0;
#pragma unroll 1
    for (int c16 = 0; c16 < 2; ++c16) {
        const int c0 = half * 32 + c16 * 16;
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        if (nkb > 0) {
            uint32_t v[SE][16];
#pragma unroll
            for (int t = 0; t < SE; ++t)
                tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(t * kOzBN + c0), v[t]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int t = SE - 1; t >= 0; --t)  // Horner in 2^-8: sum_t 2^{-8t} D_t
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], 0x1.0p-8, (double)(int)v[t][j]);
        }
        if (m < M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = c0 + j;
                if (clim[c] == 0) break;
                o[m + (int64_t)(bn + c) * ldo] = (m < clim[c]) ? (acc[j] * rs) * cscale[c] : 0.0;
            }
        }
    }
}

}  // namespace aero_b200
