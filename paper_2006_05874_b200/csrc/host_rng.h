#pragma once
#include <cstdint>

namespace ihs_b200 {
uint64_t splitmix64(uint64_t& state);
uint64_t derive_seed(uint64_t seed, uint64_t tag);
// sample_without_replacement(n, m, std::mt19937_64(stream_seed)) of rng.hpp:56-66
void sample_without_replacement(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out);
}  // namespace ihs_b200
