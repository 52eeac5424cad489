// Device side of the exact int8 slicing (Ozaki scheme) shared by the slicing
// kernel (ozaki.cu) and the iteration normalization (kernels.cu), which
// slices each new iterate column as it writes it.
#pragma once

#include <cstdint>

namespace aero_b200 {

constexpr int kOzSlices = 7;  // 7-bit slices per fp64 value (49 bits)
constexpr int kOzBK = 64;     // K bytes per tiled block (one pipeline stage)
constexpr int kOzBM = 128;    // G-tile rows (UMMA M)
constexpr int kOzBN = 64;     // X-tile columns (UMMA N)

// Slice vector i (v[0..lim), zero beyond; padded to Kp) into the product
// kernel's tiled image: tiles of TR vectors; block (tile t, K block b) at
// out + (t * nkb + b) * S * TR * 64 holds slice p at p * TR * 64, vector row r
// at 64 r, its 16-byte chunk c at chunk c ^ ((r >> 1) & 3) (64-byte swizzle).
// ex[i] = e with max|v| < 2^e. Whole CTA; red: blockDim.x / 32 doubles.
template <int S>
__device__ __forceinline__ void ozaki_slice8(double (&x)[8], int e, uint64_t (&pk)[S]) {
#pragma unroll
    for (int p = 0; p < S; ++p) pk[p] = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        double y = scalbn(x[u], 7 - e);  // |y| < 128
#pragma unroll
        for (int p = 0; p < S; ++p) {
            const double sv = trunc(y);
            y = (y - sv) * 128.0;
            pk[p] |= (uint64_t)(uint8_t)(int8_t)(int)sv << (8 * u);
        }
    }
}

// Slice vector i (v[0..lim), zero beyond; padded to Kp) into the product
// kernel's tiled image: tiles of TR vectors; block (tile t, K block b) at
// out + (t * nkb + b) * S * TR * 64 holds slice p at p * TR * 64, vector row r
// at 64 r, its 16-byte chunk c at chunk c ^ ((r >> 1) & 3) (64-byte swizzle).
// ex[i] = e with max|v| < 2^e. Whole CTA; red: blockDim.x / 32 doubles. Each
// thread owns 8 consecutive entries per 8 * blockDim.x: for Kp <= that span
// the vector is read once (registers), max-reduced, sliced and stored.
template <int S, int TR>
__device__ inline void ozaki_slice_vector(const double* __restrict__ v, int lim, int Kp, int i,
                                          int8_t* __restrict__ out, int* __restrict__ ex, double* red) {
    const int tid = threadIdx.x, nt = blockDim.x, span = 8 * nt;
    const int nkb = Kp / kOzBK, t = i / TR, r = i % TR;
    auto load8 = [&](int k0, double (&x)[8]) {
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = (k0 + u < lim) ? v[k0 + u] : 0.0;
    };
    auto store8 = [&](int k0, const uint64_t (&pk)[S]) {
        const int b = k0 / kOzBK, kk = k0 % kOzBK, kc = kk >> 4;
        int8_t* blk = out + ((int64_t)t * nkb + b) * S * TR * kOzBK + r * kOzBK + ((kc ^ ((r >> 1) & 3)) << 4) +
                      (kk & 15);
#pragma unroll
        for (int p = 0; p < S; ++p) *reinterpret_cast<uint64_t*>(blk + p * TR * kOzBK) = pk[p];
    };
    double x0[8];
    const int k00 = tid * 8;
    load8(k00, x0);
    double m = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) m = fmax(m, fabs(x0[u]));
    for (int k0 = k00 + span; k0 < lim; k0 += span) {  // long vectors (Kp > span): extra chunks
        double x[8];
        load8(k0, x);
#pragma unroll
        for (int u = 0; u < 8; ++u) m = fmax(m, fabs(x[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    m = 0.0;
    for (int w = 0; w < nt / 32; ++w) m = fmax(m, red[w]);
    const int e = (m > 0.0) ? ilogb(m) + 1 : 0;  // |v| < 2^e
    if (tid == 0) ex[i] = e;
    uint64_t pk[S];
    if (k00 < Kp) {
        ozaki_slice8<S>(x0, e, pk);
        store8(k00, pk);
    }
    for (int k0 = k00 + span; k0 < Kp; k0 += span) {
        double x[8];
        load8(k0, x);
        ozaki_slice8<S>(x, e, pk);
        store8(k0, pk);
    }
}

}  // namespace aero_b200
