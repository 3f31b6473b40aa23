// Driver for the reference's own rng.hpp (compiled verbatim from
// /root/reference/proj/include/nrrs/rng.hpp; it is Eigen-free).
// Prints RNG known-answer values as JSON so tests/golden/rng_kat.json can be
// regenerated: python tests/golden/make_rng_kat.py
#include "nrrs/rng.hpp"
#include <cinttypes>
#include <cstdio>
using namespace nrrs;
int main() {
    std::printf("{\n  \"pixels\": [\n");
    for (uint32_t px = 0; px < 64; ++px) {
        const uint64_t key = root_path_key(px, px % 3);
        const float u1 = path_stream(0, key, 1, Draw::RrsRound).next_float();
        const float u2 = path_stream(7, key, 2, Draw::RrsRound).next_float();
        const float u5 = path_stream(0x9e3779b97f4a7c15ull, key, 5, Draw::RrsRound).next_float();
        const uint64_t ck0 = child_path_key(key, 0), ck3 = child_path_key(key, 3);
        std::printf("    {\"pixel\": %u, \"frame\": %u, \"key\": \"%016" PRIx64 "\", \"u_seed0_d1\": %.9g, "
                    "\"u_seed7_d2\": %.9g, \"u_seedphi_d5\": %.9g, \"child0\": \"%016" PRIx64 "\", "
                    "\"child3\": \"%016" PRIx64 "\"}%s\n",
                    px, px % 3, key, u1, u2, u5, ck0, ck3, px + 1 < 64 ? "," : "");
    }
    std::printf("  ],\n  \"streams\": [\n");
    const uint64_t seeds[4] = {0, 3, 0xC0FFEE, 0xACC02};
    for (int s = 0; s < 4; ++s) {
        RngStream r(seeds[s], (uint64_t)s * 7 + 3);
        std::printf("    {\"seed\": %" PRIu64 ", \"seq\": %d, \"u32\": [", seeds[s], s * 7 + 3);
        for (int i = 0; i < 16; ++i)
            std::printf("%u%s", r.next_u32(), i + 1 < 16 ? ", " : "");
        std::printf("]}%s\n", s + 1 < 4 ? "," : "");
    }
    std::printf("  ],\n  \"mix_bits\": [");
    for (uint64_t x = 0; x < 8; ++x)
        std::printf("\"%016" PRIx64 "\"%s", mix_bits(x * 0x1234567ull), x + 1 < 8 ? ", " : "");
    std::printf("]\n}\n");
    return 0;
}
