// CPU check of the integer balanced-digit slicing (csrc/ozaki_slice.h) against
// an independent restatement (fp64 rounding + sequential carry): identical
// bytes on random and edge-case inputs, and the digits sum back to
// round(x 2^(F-e)).
#include <cstdio>
#include <cstdlib>
#include <random>

#include "ozaki_slice.h"

using namespace aero_b200;

template <int S>
static long check(const double (&x)[8], int e) {
    uint64_t a[S], b[S];
    ozaki_slice8_ref<S>(x, e, a);
    ozaki_slice8_int<S>(x, e, b);
    long bad = 0;
    for (int p = 0; p < S; ++p) bad += a[p] != b[p];
    for (int u = 0; u < 8; ++u)
        bad += ozaki_digits_value<S>(b, u) != (long long)std::round(std::ldexp(x[u], oz_frac_bits<S>() - e));
    if (bad && std::getenv("OZ_VERBOSE"))
        for (int u = 0; u < 8; ++u) std::printf("S=%d e=%d x[%d]=%a\n", S, e, u, x[u]);
    for (int u = 0; u < 8; ++u) {
        int8_t dg[S];
        ozaki_slice1_int<S>(x[u], e, dg);
        for (int p = 0; p < S; ++p) bad += (uint8_t)dg[p] != (uint8_t)(a[p] >> (8 * u));
    }
    return bad;
}

int main() {
    std::mt19937_64 g(12345);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::uniform_int_distribution<int> E(-1000, 1000), D(0, 60);
    long bad = 0, n = 0;
    for (int it = 0; it < 400000; ++it) {
        const int e = (it % 5 == 0) ? E(g) : (int)(E(g) % 40);
        double x[8];
        for (int u = 0; u < 8; ++u) {
            double v = U(g);                             // |v| < 1
            if (it % 3 == 1) v = std::ldexp(v, -D(g));  // wide dynamic range inside a vector
            x[u] = std::ldexp(v, e);                    // |x| < 2^e
        }
        if (it % 7 == 0) x[it % 8] = 0.0;
        if (it % 11 == 0) x[(it + 3) % 8] = -0.0;
        if (it % 13 == 0) x[(it + 5) % 8] = std::nextafter(std::ldexp(1.0, e), 0.0);    // just below 2^e
        if (it % 17 == 0) x[(it + 1) % 8] = -std::nextafter(std::ldexp(1.0, e), 0.0);
        if (it % 19 == 0) x[(it + 2) % 8] = std::ldexp(1.0, e - 1);                     // exact powers of two
        if (it % 23 == 0) x[(it + 6) % 8] = -std::ldexp(1.0, e - 47);               // half an ulp: tie
        if (it % 29 == 0 && e > -1020) x[(it + 4) % 8] = 4.9406564584124654e-324 * (double)(1 + it % 5);  // subnormals
        bad += check<7>(x, e) + check<6>(x, e) + check<5>(x, e);
        n += 3;
    }
    // subnormal-only vector with its own exponent bound
    {
        double x[8];
        for (int u = 0; u < 8; ++u) x[u] = std::ldexp((double)(u * 37 + 1), -1074) * (u % 2 ? -1.0 : 1.0);
        for (int e = -1065; e < -1040; ++e) bad += check<6>(x, e), ++n;
    }
    std::printf("%ld cases, %ld mismatches\n", n, bad);
    return bad != 0;
}
