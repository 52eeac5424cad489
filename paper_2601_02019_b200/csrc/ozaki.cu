// fp64 power / subspace-iteration product Y = G X on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM), by exact
// integer slicing (Ozaki scheme).
//
// Why: the dominant contraction of the update path (reference
// linalg.cpp:109-118 and :141-143, Gram form: Y = G X with G the r x r Gram of
// the row buffer) must be fp64-accurate -- the gate, tail and xi decisions are
// threshold comparisons on its results -- and tcgen05 has no f64 kind; the
// fp64 DMMA pipe (k_product_mma, product.cu) peaks at ~35 TF/s on B200 while
// the int8 tensor pipe peaks at ~4.5 POP/s.
//
// Scheme: every row i of G (and column c of X) is scaled by a power of two so
// that its entries lie in (-1, 1) and is cut into S signed 7-bit slices:
//     G_ik = 2^{e_i} sum_p a_p[i,k] 2^{-7(p+1)},  a_p in [-127, 127]
// (exact: multiplications by powers of two and removals of integer parts).
// Then  (G X)_ic = 2^{e_i + f_c - 14} sum_t 2^{-7t} D_t[i,c],
//       D_t = sum_{p+q=t} A_p B_q   (int8 x int8 -> int32, exact),
// keeping the diagonals t < S. With S = 7 the dropped terms and the slice
// remainders are below 2^-46 of max|G_i| max|X_c| per product term -- fp64
// GEMM accuracy to within a small factor (tests/test_gpu_parity.py states the
// tolerance and checks it against numpy fp64).
//
// Kernel: CTA tile 128 (rows of G) x 64 (job columns), 256 threads. The
// slicing kernels write every (tile, 64-byte K block) of all S slices as one
// contiguous block that is already the shared-memory image (K-major, 64-byte
// swizzle), so a pipeline stage is two bulk copies (cp.async.bulk, mbarrier
// transaction count) issued by one thread; the same thread issues the
// S(S+1)/2 x 2 MMAs (M128 N64 K32) of a stage into S TMEM accumulators
// (S x 64 columns) and commits to the stage's "empty" mbarrier. Two stages.
// The eight warps then read the accumulators (tcgen05.ld; warp w: TMEM lanes
// 32 (w % 4).., columns 32 (w / 4)..) and combine the diagonals in fp64.
// Deterministic split-K (fixed-order sum).
#include <algorithm>
#include <cstdint>

#include "aero_common.cuh"
#include "kernels.cuh"
#include "ozaki.cuh"

namespace aero_b200 {

namespace {
constexpr int OZ_BM = kOzBM;  // rows of G per CTA (UMMA M)
constexpr int OZ_BN = kOzBN;  // job columns per CTA (UMMA N)
constexpr int OZ_BK = kOzBK;  // K bytes (int8 elements) per stage
constexpr int OZ_THREADS = 256;

template <int S>
struct OzCfg {
    static constexpr int A_BYTES = S * OZ_BM * OZ_BK;
    static constexpr int B_BYTES = S * OZ_BN * OZ_BK;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int SMEM = 2 * STAGE + 1024 + 128 + OZ_BN * 12;  // + alignment slack, barriers, column scales
    static constexpr int TMEM_COLS = (S * OZ_BN <= 256) ? 256 : 512;
};

// UMMA instruction descriptor: D s32, A/B signed int8, both K-major, M=128, N=64
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

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

// Slices of `nvec` fp64 vectors of length K (vector i at V + i*ldv; entries
// at k >= lim_i are zero, lim_i = min(mask[i], K) or K) into the tiled image
// (ozaki.cuh); vectors nvec.. of the last tile are zero. One CTA per vector.
constexpr int SL_THREADS = 256;
template <int S, int TR>
__global__ void __launch_bounds__(SL_THREADS) k_ozaki_slice(int nvec, int K, int Kp, const double* __restrict__ V,
                                                            int ldv, const int* __restrict__ mask,
                                                            int8_t* __restrict__ out, int* __restrict__ ex) {
    __shared__ double red[SL_THREADS / 32];
    const int i = blockIdx.x;
    int lim = 0;
    if (i < nvec) lim = mask ? min(mask[i], K) : K;
    ozaki_slice_vector<S, TR>(V + (int64_t)i * ldv, lim, Kp, i, out, ex, red);
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_product_i8(int M, int N, int Kp, int kb_per_split, const int8_t* __restrict__ As,
                 const int8_t* __restrict__ Bs, const int* __restrict__ ea, const int* __restrict__ fb,
                 double* __restrict__ out, int ldo, int64_t sstride, const int* __restrict__ colmask,
                 int direct, unsigned long long* __restrict__ dbg) {
    using Cfg = OzCfg<S>;
    unsigned long long t_0 = 0;
    if (dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_0));
#define OZ_MARK(slot_)                                                                         \
    if (dbg && threadIdx.x == 0) {                                                              \
        unsigned long long t_;                                                                  \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
        const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);        \
        dbg[cta_ * 8 + (slot_)] = t_;                                                           \
    }
    extern __shared__ __align__(1024) uint8_t smraw[];
    // swizzled tiles need 1024-byte aligned shared addresses
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * Cfg::STAGE);
    uint64_t* empty = full + 2;
    uint64_t* done = empty + 2;  // one commit after the last stage: accumulators final
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    double* cscale = reinterpret_cast<double*>(slot + 2);  // OZ_BN per-column 2^(f - 14)
    int* clim = reinterpret_cast<int*>(cscale + OZ_BN);    // OZ_BN per-column row limits
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bm = blockIdx.y * OZ_BM, bn = blockIdx.x * OZ_BN, z = blockIdx.z;
    const int nkb_all = Kp / OZ_BK;
    const int kb0 = z * kb_per_split;
    const int nkb = max(0, min(nkb_all - kb0, kb_per_split));

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < OZ_BN) {
        const int n = bn + tid;
        cscale[tid] = (n < N) ? ldexp(1.0, fb[n] - 14) : 0.0;
        clim[tid] = (n >= N) ? 0 : ((direct && colmask) ? colmask[n] : M);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                     "r"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    const uint32_t sbase = smem_u32(sm);
    if (dbg && tid == 0) dbg[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 8] = t_0;
    OZ_MARK(1);

    if (tid == 0 && nkb > 0) {  // producer + MMA issuer
        const int8_t* Ablk = As + ((int64_t)blockIdx.y * nkb_all + kb0) * Cfg::A_BYTES;
        const int8_t* Bblk = Bs + ((int64_t)blockIdx.x * nkb_all + kb0) * Cfg::B_BYTES;
        auto load = [&](int st, int kb) {
            const uint32_t dA = sbase + st * Cfg::STAGE;
            mbar_expect_tx(&full[st], Cfg::STAGE);
            bulk_g2s(dA, Ablk + (int64_t)kb * Cfg::A_BYTES, Cfg::A_BYTES, &full[st]);
            bulk_g2s(dA + Cfg::A_BYTES, Bblk + (int64_t)kb * Cfg::B_BYTES, Cfg::B_BYTES, &full[st]);
        };
        load(0, 0);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb & 1;
            mbar_wait(&full[st], (kb >> 1) & 1);
            if (kb == 0) OZ_MARK(2);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t aS = sbase + st * Cfg::STAGE, bS = aS + Cfg::A_BYTES;
#pragma unroll
            for (int ks = 0; ks < OZ_BK / 32; ++ks) {
#pragma unroll
                for (int p = 0; p < S; ++p) {
                    const uint64_t da = umma_desc(aS + p * OZ_BM * OZ_BK + ks * 32);
#pragma unroll
                    for (int q = 0; q < S - p; ++q) {
                        const uint64_t db = umma_desc(bS + q * OZ_BN * OZ_BK + ks * 32);
                        mma_i8(tmem + (uint32_t)((p + q) * OZ_BN), da, db, (kb > 0 || ks > 0 || p > 0) ? 1u : 0u);
                    }
                }
            }
            umma_commit(&empty[st]);
            // refill the other stage once the MMAs of kb-1 have drained it
            // (those of kb are queued behind them, so the tensor pipe stays busy)
            if (kb + 1 < nkb) {
                if (kb >= 1) mbar_wait(&empty[st ^ 1], ((kb - 1) >> 1) & 1);
                load(st ^ 1, kb + 1);
            }
        }
        umma_commit(done);
        OZ_MARK(3);
    }
    __syncwarp();

    // epilogue: warp w reads TMEM lanes 32 (w % 4) + lane = tile row, columns 32 (w / 4) ..
    const int qd = warp & 3, half = warp >> 2;
    const int m = bm + qd * 32 + lane;
    double* o = out + (direct ? 0 : (int64_t)z * sstride);
    if (nkb > 0) {
        // (a parity wait on a stage barrier could pass on its not-yet-started
        // phase; the single-use barrier cannot)
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    OZ_MARK(4);
    const double rs = (m < M) ? ldexp(1.0, ea[m]) : 0.0;
#pragma unroll 1
    for (int c16 = 0; c16 < 2; ++c16) {
        const int c0 = half * 32 + c16 * 16;
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        if (nkb > 0) {
            uint32_t v[S][16];
#pragma unroll
            for (int t = 0; t < S; ++t)
                tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(t * OZ_BN + c0), v[t]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int t = S - 1; t >= 0; --t)  // Horner in 2^-7: sum_t 2^{-7t} D_t
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], 0x1.0p-7, (double)(int)v[t][j]);
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
    OZ_MARK(5);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    OZ_MARK(6);
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
    }
}

__global__ void k_ozaki_reduce(int M, int N, int splits, const double* __restrict__ ws, int64_t sstride,
                               double* __restrict__ Y, int ldy, const int* __restrict__ colmask) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)M * N) return;
    const int i = (int)(e % M), j = (int)(e / M);
    double v = 0.0;
    for (int zz = 0; zz < splits; ++zz) v += __ldcg(ws + zz * sstride + e);
    if (colmask && i >= colmask[j]) v = 0.0;
    Y[i + (int64_t)j * ldy] = v;
}

constexpr int kSlices = kOzSlices;
}  // namespace

int ozaki_slices() { return kSlices; }

void OzakiGram::prepare(cudaStream_t st, int R_, const double* G, int ldg) {
    R = R_;
    Rp = (R + OZ_BM - 1) / OZ_BM * OZ_BM;
    Kp = (R + OZ_BK - 1) / OZ_BK * OZ_BK;
    const size_t need = (size_t)kSlices * Rp * Kp;
    if (a_bytes < need) {
        if (a) cudaFree(a);
        AERO_CUDA(cudaMalloc(&a, need));
        a_bytes = need;
    }
    if (ea_n < (size_t)Rp) {
        if (ea) cudaFree(ea);
        AERO_CUDA(cudaMalloc(&ea, sizeof(int) * Rp));
        ea_n = Rp;
    }
    k_ozaki_slice<kSlices, OZ_BM><<<Rp, SL_THREADS, 0, st>>>(R, R, Kp, G, ldg, nullptr, a, ea);
    AERO_LAUNCHED();
}

void OzakiGram::product(cudaStream_t st, int N, const double* X, int ldx, const int* colmask, double* Y,
                        int ldy, double* ws, size_t ws_doubles, unsigned long long* dbg) {
    using Cfg = OzCfg<kSlices>;
    if (N <= 0) return;
    const int Np = (N + OZ_BN - 1) / OZ_BN * OZ_BN;
    const size_t need = (size_t)kSlices * Np * Kp;
    if (b_bytes < need) {
        if (b) cudaFree(b);
        AERO_CUDA(cudaMalloc(&b, need));
        b_bytes = need;
    }
    if (fb_n < (size_t)Np) {
        if (fb) cudaFree(fb);
        AERO_CUDA(cudaMalloc(&fb, sizeof(int) * Np));
        fb_n = Np;
    }
    k_ozaki_slice<kSlices, OZ_BN><<<Np, SL_THREADS, 0, st>>>(N, R, Kp, X, ldx, colmask, b, fb);
    AERO_LAUNCHED();
    static bool attr = false;
    if (!attr) {
        AERO_CUDA(cudaFuncSetAttribute(k_product_i8<kSlices>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM));
        attr = true;
    }
    // split-K so tiles x splits fills the 148 SMs once (one CTA per SM: TMEM
    // and shared memory), each split >= 2 K stages
    const int tm = Rp / OZ_BM, tn = Np / OZ_BN, nkb = Kp / OZ_BK;
    int splits = std::max(1, std::min(148 / std::max(tm * tn, 1), nkb / 2));
    while (splits > 1 && (size_t)splits * R * N > ws_doubles) --splits;
    const int per = (nkb + splits - 1) / splits;
    splits = (nkb + per - 1) / per;
    const int direct = splits == 1;
    double* o = direct ? Y : ws;
    const int ldo = direct ? ldy : R;
    const int64_t sstride = (int64_t)R * N;
    k_product_i8<kSlices><<<dim3(tn, tm, splits), OZ_THREADS, Cfg::SMEM, st>>>(
        R, N, Kp, per, a, b, ea, fb, o, ldo, sstride, colmask, direct, dbg);
    AERO_LAUNCHED();
    if (!direct) {
        const int64_t tot = (int64_t)R * N;
        k_ozaki_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(R, N, splits, ws, sstride, Y, ldy, colmask);
        AERO_LAUNCHED();
    }
}

void OzakiGram::release() {
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (ea) cudaFree(ea);
    if (fb) cudaFree(fb);
    a = b = nullptr;
    ea = fb = nullptr;
    a_bytes = b_bytes = ea_n = fb_n = 0;
}

}  // namespace aero_b200
