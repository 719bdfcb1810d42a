// Shadow of the reference's tests/support/oracles.hpp for the bf16-input runs
// (test infrastructure): includes the reference header unchanged, renaming
// its random_block, and provides random_block returning the same draws
// rounded to the nearest bf16 (RNE).  Only on the include path of the
// *_bf16 binaries (tests/ref_suite/Makefile).
#pragma once
#include <cstring>
#define random_block random_block_f32
#include_next "oracles.hpp"
#undef random_block

namespace oracles {
inline saap::TensorBlock random_block(saap::Rng& rng, std::size_t rows, std::size_t dim,
                                      double scale = 1.0) {
    saap::TensorBlock t = random_block_f32(rng, rows, dim, scale);
    for (float& x : t.data) {
        uint32_t u;
        std::memcpy(&u, &x, 4);
        if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
        std::memcpy(&x, &u, 4);
    }
    return t;
}
}  // namespace oracles
