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
// Scheme: every row i of G (and column c of X) gets a power-of-two bound
// 2^{e_i} > max|G_i|, is rounded to F = 8S - 2 fractional bits below it and
// written in S balanced signed base-256 digits (ozaki_slice.h):
//     G_ik ~ 2^{e_i - F} sum_p a_p[i,k] 256^{S-1-p},  a_p in [-128, 127].
// Then  (G X)_ic = 2^{e_i + f_c - 12} sum_t 2^{-8t} D_t[i,c],
//       D_t = sum_{p+q=t} A_p B_q   (int8 x int8 -> int32, exact),
// keeping the diagonals t < S: S(S+1)/2 = 21 slice-pair products at S = 6.
// Error per product term, relative to 2^{e_i + f_c}: the two roundings
// (2^-47 each) plus the dropped diagonals (t = 6: five pairs of at most
// 128^2 2^-60) -- below 6.1 x 2^-46, i.e. below 2^-41 max|G_i| max|X_c| per
// term in the worst case; the digits are balanced, so these terms carry random
// signs and the observed error is two to three orders of magnitude smaller
// (tests/test_gpu_parity.py states the bound and checks it against numpy
// fp64). (Round 1 used 7-bit sign-magnitude slices: S = 7, 28 products, every
// dropped term biased toward zero.)
//
// Kernel: CTA tile 128 (rows of G) x 64 (job columns), 256 threads. The
// slicing kernels write every (tile, 64-byte K block) of all S slices as one
// contiguous block that is already the shared-memory image (K-major, 64-byte
// swizzle), so a pipeline stage is two bulk copies (cp.async.bulk, mbarrier
// transaction count) issued by one thread; the same thread issues the
// S(S+1)/2 x 2 MMAs (M128 N64 K32) of a stage into S TMEM accumulators
// (S x 64 columns) and commits to the stage's "empty" mbarrier. Three 72 KiB
// stages at S = 6 (two bulk loads in flight behind the stage being read).
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
                 int direct) {
    using Cfg = OzCfg<S>;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);  // swizzled tiles: 1024-B aligned
    __shared__ uint32_t slot;
    const int z = blockIdx.z, nkb_all = Kp / OZ_BK, kb0 = z * kb_per_split;
    const int nkb = max(0, min(nkb_all - kb0, kb_per_split));
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&slot)),
                     "r"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = slot;
    ozaki_tile<S>(M, N, nkb_all, blockIdx.y, blockIdx.x, kb0, nkb, As, Bs, ea, fb,
                  out + (direct ? 0 : (int64_t)z * sstride), ldo, colmask, direct, sm, tmem);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
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

void OzakiGram::reserve(int Rmax, int Nmax) {
    const int Rp_ = (Rmax + OZ_BM - 1) / OZ_BM * OZ_BM, Kp_ = (Rmax + OZ_BK - 1) / OZ_BK * OZ_BK;
    const int Np = (Nmax + OZ_BN - 1) / OZ_BN * OZ_BN;
    const size_t na = (size_t)kSlices * Rp_ * Kp_, nb = (size_t)kSlices * Np * Kp_;
    if (a_bytes < na) {
        if (a) cudaFree(a);
        AERO_CUDA(cudaMalloc(&a, na));
        a_bytes = na;
    }
    if (ea_n < (size_t)Rp_) {
        if (ea) cudaFree(ea);
        AERO_CUDA(cudaMalloc(&ea, sizeof(int) * Rp_));
        ea_n = Rp_;
    }
    if (b_bytes < nb) {
        if (b) cudaFree(b);
        AERO_CUDA(cudaMalloc(&b, nb));
        b_bytes = nb;
    }
    if (fb_n < (size_t)Np) {
        if (fb) cudaFree(fb);
        AERO_CUDA(cudaMalloc(&fb, sizeof(int) * Np));
        fb_n = Np;
    }
}

void OzakiGram::reserve_x(int N) {
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
}

void OzakiGram::product(cudaStream_t st, int N, const double* X, int ldx, const int* colmask, double* Y,
                        int ldy, double* ws, size_t ws_doubles) {
    using Cfg = OzCfg<kSlices>;
    if (N <= 0) return;
    const int Np = (N + OZ_BN - 1) / OZ_BN * OZ_BN;
    reserve_x(N);
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
        R, N, Kp, per, a, b, ea, fb, o, ldo, sstride, colmask, direct);
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
