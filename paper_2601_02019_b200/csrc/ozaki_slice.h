// Slicing of fp64 values into signed 8-bit digits (the digit step of the
// Ozaki scheme, ozaki.cuh) in integer arithmetic. A value x with |x| < 2^e is
// rounded to F = 8S - 2 fractional bits below 2^e,
//     Y = round(x 2^(F - e)),  |Y| <= 2^F            (half away from zero)
// and Y is written in BALANCED base-256 digits d_0 .. d_{S-1} in [-128, 127]:
//     Y = sum_p d_p 256^(S-1-p).
// Balanced digits are the bytes of Y + 0x80 80 .. 80 (0x80 added at each of
// the S-1 lower byte positions, carries propagating naturally) with the top
// bit of every lower byte flipped: byte - 128 at a lower position undoes the
// added 0x80. |Y| <= 2^(8S-2) leaves the top digit in [-65, 65], so the carry
// never overflows it. All digits are signed (one MMA descriptor, s8 x s8), the
// terms dropped by the truncated product (ozaki.cuh) have random signs instead
// of the sign of the value (a sign-magnitude split biases every dropped term
// toward zero), and a slice carries 8 bits instead of 7: S = 6 gives 46 bits +
// sign with 21 slice-pair products where 7-bit sign-magnitude slices needed
// S = 7 (49 bits, 28 products).
// The mantissa shift replaces an fp64 trunc / subtract / multiply / convert
// chain per digit. Plain C++: the same header compiles under g++ for
// tests/cpp/test_ozaki_slice.cpp, which checks it against an independent
// restatement (ozaki_slice8_ref: std::round + sequential carry).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define AERO_OZ_HD __host__ __device__ __forceinline__
#else
#define AERO_OZ_HD inline
#endif
#if defined(__CUDA_ARCH__)
#define AERO_OZ_UNROLL _Pragma("unroll")
#else
#define AERO_OZ_UNROLL
#endif

namespace aero_b200 {

AERO_OZ_HD uint64_t oz_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t b;
    std::memcpy(&b, &x, sizeof(b));
    return b;
#endif
}

// fractional bits kept below 2^e
template <int S>
constexpr int oz_frac_bits() {
    return 8 * S - 2;
}

// 0x80 at each of the S-1 lower byte positions
template <int S>
constexpr uint64_t oz_low_bias() {
    uint64_t b = 0;
    for (int p = 1; p < S; ++p) b |= (uint64_t)0x80 << (8 * (S - 1 - p));
    return b;
}

// the balanced digits of round(x 2^(F-e)) for a finite |x| < 2^e, as the bytes
// of the returned word: digit p = byte S-1-p (signed)
template <int S>
AERO_OZ_HD uint64_t oz_digits(uint64_t bits, int e) {
    const int ex = (int)((bits >> 52) & 0x7ffu);
    const uint64_t mant = (bits & 0x000FFFFFFFFFFFFFull) | (ex ? (1ull << 52) : 0ull);
    const int sh = 1075 - (ex ? ex : 1) + e - oz_frac_bits<S>();  // >= 55 - 8S > 0 for a normal |x| < 2^e
    uint64_t ya;
    if (sh <= 0) ya = mant << ((-sh) & 63);  // subnormal-scale vectors (exact)
    else if (sh >= 64) ya = 0ull;
    else ya = (mant + (1ull << (sh - 1))) >> sh;  // round half away from zero
    const uint64_t y = (bits >> 63) ? (0ull - ya) : ya;  // two's complement
    return (y + oz_low_bias<S>()) ^ oz_low_bias<S>();
}

// cut 8 values (|x| < 2^e) into S signed 8-bit slices, packed 8 per uint64
// (byte u of pk[p] = slice p of x[u])
template <int S>
AERO_OZ_HD void ozaki_slice8_int(const double (&x)[8], int e, uint64_t (&pk)[S]) {
    uint32_t lo[S], hi[S];
    AERO_OZ_UNROLL
    for (int p = 0; p < S; ++p) lo[p] = hi[p] = 0u;
    AERO_OZ_UNROLL
    for (int u = 0; u < 8; ++u) {
        const uint64_t z = oz_digits<S>(oz_bits(x[u]), e);
        AERO_OZ_UNROLL
        for (int p = 0; p < S; ++p) {
            const uint32_t d = (uint32_t)(z >> (8 * (S - 1 - p))) & 255u;
            if (u < 4) lo[p] |= d << (8 * u);
            else hi[p] |= d << (8 * (u - 4));
        }
    }
    AERO_OZ_UNROLL
    for (int p = 0; p < S; ++p) pk[p] = (uint64_t)lo[p] | ((uint64_t)hi[p] << 32);
}

// the S slices of one value as int8 digits
template <int S>
AERO_OZ_HD void ozaki_slice1_int(double x, int e, int8_t (&dg)[S]) {
    const uint64_t z = oz_digits<S>(oz_bits(x), e);
    AERO_OZ_UNROLL
    for (int p = 0; p < S; ++p) dg[p] = (int8_t)(uint8_t)(z >> (8 * (S - 1 - p)));
}

// independent restatement for the CPU test: fp64 rounding, sequential carry
template <int S>
inline void ozaki_slice8_ref(const double (&x)[8], int e, uint64_t (&pk)[S]) {
    for (int p = 0; p < S; ++p) pk[p] = 0;
    for (int u = 0; u < 8; ++u) {
        long long y = (long long)std::round(std::ldexp(x[u], oz_frac_bits<S>() - e));  // exact: |y| <= 2^(8S-2)
        int d[S];
        for (int p = S - 1; p >= 1; --p) {  // least significant digit first
            long long r = ((y % 256) + 256) % 256;
            if (r >= 128) r -= 256;
            d[p] = (int)r;
            y = (y - r) / 256;
        }
        d[0] = (int)y;
        for (int p = 0; p < S; ++p) pk[p] |= (uint64_t)(uint8_t)(int8_t)d[p] << (8 * u);
    }
}

// the value the digits represent, in units of 2^(e - F) (test helper)
template <int S>
inline long long ozaki_digits_value(const uint64_t (&pk)[S], int u) {
    long long y = 0;
    for (int p = 0; p < S; ++p) y = y * 256 + (long long)(int8_t)(uint8_t)(pk[p] >> (8 * u));
    return y;
}

}  // namespace aero_b200
