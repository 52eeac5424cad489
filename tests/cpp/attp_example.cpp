// C++ host using the drop-in shim (include/aero_b200.hpp) the way the
// reference's bench.cpp:148-160 drives aero::AttpState: per-row updates,
// then a prefix query. Prints "rows clock ell fro_mass sketch_fro2".
#include <cmath>
#include <cstdio>
#include <vector>

#include "aero_b200.hpp"

int main(int argc, char** argv) {
    const int d = 64, n = argc > 1 ? std::atoi(argv[1]) : 500;
    aero::b200::AttpState s(d, 0.25, 1, 1000);
    std::vector<double> a(d);
    unsigned long long x = 12345;
    for (int i = 1; i <= n; ++i) {
        for (int j = 0; j < d; ++j) {  // xorshift uniforms in (0, 1]
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            a[j] = ((x >> 11) + 1) * 0x1.0p-53;
        }
        s.update(a, i);
    }
    const std::vector<double> b = s.query(n);
    double f2 = 0.0;
    for (double v : b) f2 += v * v;
    std::printf("%d %lld %d %.6f %.6f\n", n, (long long)s.clock(), s.ell(), s.fro_mass(), f2);
    try {
        s.update(a, 1);  // timestamp regression -> aero::b200::InvalidInput
    } catch (const aero::b200::InvalidInput& e) {
        std::printf("InvalidInput: %s\n", e.what());
    }
    return 0;
}
