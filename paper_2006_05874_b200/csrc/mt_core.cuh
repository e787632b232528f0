// mt_core.cuh — the MT19937-64 block recurrence on the device.
//
// std::mt19937_64 regenerates its 312-word state in one twist:
//   new[k]       = old[k+156] ^ f(old[k], old[k+1])          k = 0..155
//   new[k+156]   = new[k]     ^ f(old[k+156], old[k+157])   k = 0..154
//   new[311]     = new[155]   ^ f(old[311], new[0])
// with f(a, b) = (y >> 1) ^ (y & 1 ? MATRIX_A : 0), y = (a & UM) | (b & LM).
// Thread k (< 156) owns words k and k+156 of every block and reads only the
// previous block (thread 155 recomputes new[0] locally), so a block costs a
// single barrier with the state ping-ponged between two shared buffers.
#pragma once
#include <cstdint>

namespace ihs_b200 {
namespace mt {

constexpr int NN = 312;
constexpr int MM = 156;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL;  // upper 33 bits
constexpr uint64_t LM = 0x7FFFFFFFULL;          // lower 31 bits
constexpr int THREADS = 160;                    // 156 workers, rounded to whole warps

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

__device__ __forceinline__ uint64_t mix(uint64_t a, uint64_t b) {
    const uint64_t y = (a & UM) | (b & LM);
    return (y >> 1) ^ ((y & 1ULL) ? MATRIX_A : 0ULL);
}

// Seeded initial array of std::mt19937_64(seed) into st[0..312) (one thread).
__device__ __forceinline__ void seed_array(uint64_t* st, uint64_t seed) {
    if (threadIdx.x == 0) {
        st[0] = seed;
        for (int i = 1; i < NN; ++i) st[i] = 6364136223846793005ULL * (st[i - 1] ^ (st[i - 1] >> 62)) + (uint64_t)i;
    }
}

// Ping-pong state: buf holds 2 x 312 words in shared memory; the current
// block lives in buf + cur * 312. next() must be called by all threads of
// the CTA; threads k < 156 receive the new words k (lo) and k + 156 (hi).
struct Twister {
    uint64_t* buf;
    int cur;
    __device__ __forceinline__ bool worker() const { return threadIdx.x < MM; }
    __device__ __forceinline__ void next(uint64_t& lo, uint64_t& hi) {
        const uint64_t* o = buf + cur * NN;
        uint64_t* nw = buf + (cur ^ 1) * NN;
        const int k = threadIdx.x;
        if (k < MM) {
            lo = o[k + MM] ^ mix(o[k], o[k + 1]);
            if (k < MM - 1) {
                hi = lo ^ mix(o[k + MM], o[k + MM + 1]);
            } else {
                const uint64_t n0 = o[MM] ^ mix(o[0], o[1]);
                hi = lo ^ mix(o[NN - 1], n0);
            }
            nw[k] = lo;
            nw[k + MM] = hi;
        }
        __syncthreads();
        cur ^= 1;
    }
};

}  // namespace mt
}  // namespace ihs_b200
