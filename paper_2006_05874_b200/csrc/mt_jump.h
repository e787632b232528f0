// mt_jump.h — F2-linear jump-ahead for std::mt19937_64 substreams.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace ihs_b200 {

// Draws per substream of a long Gaussian stream (one CTA each).
constexpr int64_t kJumpStride = int64_t{1} << 18;
// Draws per substream of an SRHT sign vector (a multiple of 32 for whole bit words).
constexpr int64_t kSignStride = int64_t{1} << 15;

// Characteristic polynomial of the MT19937-64 transition (degree 19937),
// found once per process by Berlekamp-Massey over GF(2); bit i = coeff of x^i.
const std::vector<uint64_t>& mt_charpoly();
// x^(q*stride) mod charpoly for q = 0..nsub-1 (cached per stride), packed
// nsub x 312 words.
const std::vector<uint64_t>& mt_jump_polys(int64_t stride, int64_t nsub);
// Words of device scratch mt_jump_starts needs for the seeded word sequence.
constexpr int64_t kJumpSeqWords = 19937 + 312 - 1;
// Device: write the 312-word start window of substream q (state after
// q*stride draws of mt19937_64(seed)) to d_starts[q*312 ...]; d_X is
// kJumpSeqWords words of scratch.
// q0 > 0: substreams q0 .. q0+nsub-1 (start windows still written from d_starts[0]).
void mt_jump_starts(uint64_t seed, int64_t stride, int64_t nsub, uint64_t* d_starts, uint64_t* d_X, cudaStream_t st,
                    int64_t q0 = 0);
// Draws per substream of the streamed (block-by-block) Gaussian generation.
constexpr int64_t kStreamStride = int64_t{1} << 22;

}  // namespace ihs_b200
