// host_rng.cpp — host side of the reference RNG (rng.hpp:13-66).
//
// derive_seed/splitmix64 are pure integer functions. The row sample P of the
// SRHT (sample_without_replacement, rng.hpp:56-66) is a partial Fisher-Yates
// driven by std::uniform_int_distribution<Index>(k, n-1) on std::mt19937_64;
// we draw with exactly those libstdc++ types (so every index matches the
// reference) but keep the pool sparse: only positions touched by a swap are
// stored, so the cost is O(m) instead of the reference's O(n_pad) iota.
#include "host_rng.h"

#include <random>
#include <vector>

namespace ihs_b200 {

uint64_t splitmix64(uint64_t& state) {  // rng.hpp:13-18
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t derive_seed(uint64_t seed, uint64_t tag) {  // rng.hpp:23-28
    uint64_t s = seed + 0x632be59bd9b4e019ULL * (tag + 1);
    const uint64_t a = splitmix64(s);
    const uint64_t b = splitmix64(s);
    return a ^ (b << 1);
}

namespace {
// open-addressing map position -> value for the sparse Fisher-Yates pool
struct SparsePool {
    std::vector<int64_t> keys, vals;
    uint64_t mask;
    explicit SparsePool(int64_t m) {
        uint64_t cap = 16;
        while (cap < (uint64_t)(4 * m + 16)) cap <<= 1;
        keys.assign(cap, -1);
        vals.assign(cap, 0);
        mask = cap - 1;
    }
    static uint64_t hash(int64_t k) {
        uint64_t x = (uint64_t)k * 0x9E3779B97F4A7C15ULL;
        return x ^ (x >> 29);
    }
    int64_t get(int64_t k) const {
        for (uint64_t h = hash(k) & mask;; h = (h + 1) & mask) {
            if (keys[h] == k) return vals[h];
            if (keys[h] < 0) return k;  // untouched position holds its own index
        }
    }
    void set(int64_t k, int64_t v) {
        for (uint64_t h = hash(k) & mask;; h = (h + 1) & mask) {
            if (keys[h] == k || keys[h] < 0) {
                keys[h] = k;
                vals[h] = v;
                return;
            }
        }
    }
};
}  // namespace

void sample_without_replacement(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out) {
    std::mt19937_64 gen(stream_seed);
    using Index = long;  // Eigen::Index on LP64, the reference's distribution type
    if (m * 8 >= n) {
        // dense pool (the reference's own layout) when m is a sizable fraction of n
        std::vector<int64_t> pool((size_t)n);
        for (int64_t i = 0; i < n; ++i) pool[(size_t)i] = i;
        for (int64_t k = 0; k < m; ++k) {
            std::uniform_int_distribution<Index> pick((Index)k, (Index)(n - 1));
            const int64_t j = (int64_t)pick(gen);
            std::swap(pool[(size_t)k], pool[(size_t)j]);
            out[k] = pool[(size_t)k];
        }
        return;
    }
    SparsePool pool(m);
    for (int64_t k = 0; k < m; ++k) {
        std::uniform_int_distribution<Index> pick((Index)k, (Index)(n - 1));
        const int64_t j = (int64_t)pick(gen);
        const int64_t vk = pool.get(k);
        const int64_t vj = pool.get(j);
        pool.set(k, vj);
        pool.set(j, vk);
        out[k] = vj;
    }
}

}  // namespace ihs_b200
