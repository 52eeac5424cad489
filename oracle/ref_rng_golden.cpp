// Golden-vector generator compiled directly against the REFERENCE's own
// rng.hpp (/root/reference/proj/include/aero/rng.hpp; the one reference header
// that builds without Eigen). Built by oracle/Makefile into oracle/_ref/ and
// run by oracle/make_golden.sh to produce tests/golden/rng_golden.json, which
// pins the oracle's (and the product's) RngState restatement bit-for-bit.
#include <cstdio>
#include <cstdint>
#include <cstring>

#include "aero/rng.hpp"

static void hex(double x) {
    std::uint64_t b;
    std::memcpy(&b, &x, 8);
    std::printf("\"%016llx\"", (unsigned long long)b);
}

int main() {
    struct Case { std::uint64_t seed, stream; int fork; int n; int kind; };
    // kind 0: gaussian(), 1: uniform(); fork = number of fork() calls on the
    // root before drawing from the last child (0 = draw from the root)
    const Case cases[] = {
        {1, 1000, 1, 9, 0}, {1, 1000, 2, 7, 0}, {1, 1000, 0, 5, 1}, {0, 0, 0, 6, 1},
        {0, 0, 0, 6, 0},    {7, 0, 1, 5, 0},    {13, 4, 3, 4, 0},   {42, 7, 1, 3, 1},
        {5, 1003, 17, 5, 0}, {123456789, 987654321, 1000, 4, 0},
        {0xffffffffffffffffULL, 0x8000000000000000ULL, 2, 4, 0},
    };
    std::printf("{\n  \"source\": \"/root/reference/proj/include/aero/rng.hpp\",\n  \"cases\": [\n");
    bool first = true;
    for (const Case& c : cases) {
        aero::RngState root(c.seed, c.stream);
        aero::RngState r = root;
        for (int f = 0; f < c.fork; ++f) r = root.fork();
        std::printf("%s    {\"seed\": \"%llu\", \"stream\": \"%llu\", \"fork\": %d, \"kind\": %d, \"bits\": [",
                    first ? "" : ",\n", (unsigned long long)c.seed,
                    (unsigned long long)c.stream, c.fork, c.kind);
        for (int i = 0; i < c.n; ++i) {
            if (i) std::printf(", ");
            hex(c.kind == 0 ? r.gaussian() : r.uniform());
        }
        std::printf("]}");
        first = false;
    }
    // mixed sequence: gaussian, uniform, gaussian (spare interplay)
    {
        aero::RngState r(3, 9);
        std::printf(",\n    {\"seed\": \"3\", \"stream\": \"9\", \"fork\": 0, \"kind\": 2, \"bits\": [");
        hex(r.gaussian()); std::printf(", "); hex(r.uniform()); std::printf(", ");
        hex(r.gaussian()); std::printf(", "); hex(r.gaussian()); std::printf("]}");
    }
    std::printf("\n  ]\n}\n");
    return 0;
}
