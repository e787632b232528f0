// mt19937.cu — the reference's random streams, generated on the device.
//
// The reference draws every random quantity of the hot path from
// std::mt19937_64 seeded through derive_seed (rng.hpp:23-32):
//   * SRHT signs   rademacher(n_pad, make_stream(seed,1))   (rng.hpp:48-52, sketch.hpp:85-87)
//   * Gaussian S   fill_gaussian(S, make_stream(seed,0), 1/sqrt(m))  (rng.hpp:35-40, sketch.hpp:62-64)
// This file reproduces those streams bit-for-bit: the MT19937-64 recurrence
// and tempering, libstdc++'s generate_canonical<double,53> (one draw,
// double(raw) * 2^-64, clamped below 1) and its Marsaglia polar
// normal_distribution with the cached second value. All double arithmetic
// uses explicit _rn intrinsics (no FMA contraction) so it rounds exactly like
// the reference's x86-64 build; only log() may differ from glibc in the last
// ulp, which leaves acceptance (and hence every stream position) exact.
//
// Generation is block-sequential: one twist produces 312 words from the
// previous 312 (two data-parallel half-steps). A single-stream sequence is
// produced by one CTA; long Gaussian streams are split into substreams whose
// start states are obtained by F2-linear jump-ahead (mt_jump.cpp) and run one
// CTA per substream.
#include "common.cuh"

#include <functional>
#include "mt_core.cuh"
#include "mt_jump.h"


namespace ihs_b200 {

namespace {
using mt::NN;
using mt::temper;

// Single-stream raw generator: draws [0, count) of mt19937_64(seed).
__global__ void __launch_bounds__(mt::THREADS) mt_raw_kernel(uint64_t seed, int64_t count, uint64_t* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    mt::seed_array(buf, seed);
    __syncthreads();
    mt::Twister tw{buf, 0};
    const int k = threadIdx.x;
    for (int64_t base = 0; base < count; base += NN) {
        uint64_t lo, hi;
        tw.next(lo, hi);
        if (tw.worker()) {
            if (base + k < count) out[base + k] = temper(lo);
            if (base + mt::MM + k < count) out[base + mt::MM + k] = temper(hi);
        }
    }
}


// Sign bits of draws [beg, end) into a shared bit buffer (bit g - beg).
__device__ __forceinline__ void or_bits32(uint32_t* accw, int64_t o, uint32_t v) {
    // bits [o, o + 32) |= v (o need not be word aligned)
    if (!v) return;
    const int sh = (int)(o & 31);
    atomicOr(&accw[o >> 5], v << sh);
    if (sh && (v >> (32 - sh))) atomicOr(&accw[(o >> 5) + 1], v >> (32 - sh));  // only bits inside the range
}
// one warp ballot per 32 draws instead of one atomic per set bit
__device__ __forceinline__ void sign_bits_range(mt::Twister& tw, int64_t beg, int64_t end, uint32_t* accw) {
    const int k = threadIdx.x, lane = k & 31;
    for (int64_t base = beg; base < end; base += NN) {
        uint64_t lo = 0, hi = 0;
        tw.next(lo, hi);
        const bool w = tw.worker();
        const int64_t g0 = base + k, g1 = base + mt::MM + k;
        const uint32_t b0 = __ballot_sync(0xffffffffu, w && g0 < end && (temper(lo) & 1ULL));
        const uint32_t b1 = __ballot_sync(0xffffffffu, w && g1 < end && (temper(hi) & 1ULL));
        if (lane == 0) {
            or_bits32(accw, g0 - beg, b0);  // lane 0's draw is bit 0 of the ballot
            or_bits32(accw, g1 - beg, b1);
        }
    }
}

// Sign bits, single stream: chunks of 32 blocks (9984 draws = 312 words).
__global__ void __launch_bounds__(mt::THREADS) mt_signbits_kernel(uint64_t seed, int64_t n, uint32_t* __restrict__ bits) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    __shared__ uint32_t acc[NN];
    mt::seed_array(buf, seed);
    __syncthreads();
    mt::Twister tw{buf, 0};
    const int64_t nwords = (n + 31) / 32;
    for (int64_t beg = 0; beg < n; beg += 32 * NN) {
        for (int i = threadIdx.x; i < NN; i += blockDim.x) acc[i] = 0u;
        __syncthreads();
        sign_bits_range(tw, beg, min(n, beg + 32 * NN), acc);
        __syncthreads();
        for (int i = threadIdx.x; i < NN; i += blockDim.x) {
            const int64_t w = beg / 32 + i;
            if (w < nwords) bits[w] = acc[i];
        }
        __syncthreads();
    }
}

// Sign bits from jump-ahead substreams: CTA q produces draws
// [q*stride, min(n, (q+1)*stride)) (stride a multiple of 32) into a shared
// bit buffer, then writes its whole words.
__global__ void __launch_bounds__(mt::THREADS) mt_signbits_sub_kernel(const uint64_t* __restrict__ starts,
                                                                      int64_t stride, int64_t n,
                                                                      uint32_t* __restrict__ bits) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ uint32_t accw[];
    __shared__ uint64_t buf[2 * NN];
    const int64_t q = blockIdx.x;
    const int nw = (int)(stride / 32);
    for (int i = threadIdx.x; i < NN; i += blockDim.x) buf[i] = starts[q * NN + i];
    for (int i = threadIdx.x; i < nw; i += blockDim.x) accw[i] = 0u;
    __syncthreads();
    mt::Twister tw{buf, 0};
    const int64_t beg = q * stride;
    const int64_t end = min(n, beg + stride);
    sign_bits_range(tw, beg, end, accw);
    __syncthreads();
    const int64_t w_end = (end + 31) / 32;
    for (int64_t w = beg / 32 + threadIdx.x; w < w_end; w += blockDim.x) bits[w] = accw[w - beg / 32];
}

}  // namespace

void mt_seed_host(uint64_t seed, MTState& s) {
    s.mt[0] = seed;
    for (int i = 1; i < NN; ++i) s.mt[i] = 6364136223846793005ULL * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + (uint64_t)i;
}

void mt_generate_raw(uint64_t seed, int64_t count, uint64_t* d_out, cudaStream_t st) {
    if (count <= 0) return;
    LAUNCH_PDL(mt_raw_kernel, 1, 160, 0, st, seed, count, d_out);
}

size_t rademacher_scratch_bytes(int64_t n) {
    const int64_t nsub = ceil_div(std::max<int64_t>(n, 1), kSignStride);
    return (size_t)nsub * NN * 8 + (size_t)kJumpSeqWords * 8 + 256;
}

void mt_rademacher_bits(uint64_t seed, int64_t n, uint32_t* d_bits, void* d_scratch, cudaStream_t st) {
    if (n <= 0) return;
    if (n <= 2 * kSignStride || d_scratch == nullptr) {
        LAUNCH_PDL(mt_signbits_kernel, 1, 160, 0, st, seed, n, d_bits);
        return;
    }
    const int64_t nsub = ceil_div(n, kSignStride);
    uint64_t* starts = static_cast<uint64_t*>(d_scratch);
    uint64_t* xseq = starts + nsub * NN;
    mt_jump_starts(seed, kSignStride, nsub, starts, xseq, st);
    LAUNCH_PDL(mt_signbits_sub_kernel, (unsigned)nsub, 160, (size_t)(kSignStride / 32) * 4, st, starts,
           (int64_t)kSignStride, n, d_bits);
}

}  // namespace ihs_b200
