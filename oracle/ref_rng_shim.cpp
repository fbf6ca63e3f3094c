// ref_rng_shim.cpp — prints the reference's seed derivation (proj/src/rng.hpp:10-25)
// for the inputs our synthetic library uses, as JSON. Compiled against the
// reference header by oracle/build_ref.sh; output pins oracle/omc_oracle.c's
// orc_derive_seed and the product's derive_seed (tests/golden/ref_derive_seed.json).
#include <cstdio>
#include <cstdint>

#include "rng.hpp"

int main() {
    const std::uint64_t bases[] = {0ULL, 1ULL, 42ULL, 1234ULL, 0xdeadbeefULL, 0xffffffffffffffffULL};
    const std::uint64_t streams[] = {0ULL, 1ULL, 2ULL, 13ULL, 271ULL, 0xF00DULL, 1000000ULL};
    std::printf("{\"derive_seed\": [");
    bool first = true;
    for (auto b : bases)
        for (auto s : streams) {
            std::printf("%s[\"%llu\", \"%llu\", \"%llu\"]", first ? "" : ", ", (unsigned long long)b,
                        (unsigned long long)s, (unsigned long long)autotune::derive_seed(b, s));
            first = false;
        }
    std::printf("], \"splitmix64_from_1234\": [");
    std::uint64_t st = 1234;
    for (int i = 0; i < 8; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)autotune::splitmix64(st));
    std::printf("]}\n");
    return 0;
}
