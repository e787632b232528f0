// srht.cu — SRHT sketch SA = sqrt(n_pad/m) * R * H * D * A on sm_100a.
//
// Reference: srht_sketch (sketch.hpp:77-108) with fwht_inplace
// (sketch.hpp:33-49). The reference materializes a zero-padded n_pad x d copy
// B, multiplies row i by eps_i, runs radix-2 butterflies per column for
// h = 1, 2, ..., n_pad/2 (bit 0 first), scales by 1/sqrt(n_pad), and gathers
// the m sampled rows scaled by sqrt(n_pad/m).
//
// B200 design (bit-exact with the reference):
//   * no padded copy: rows >= n are virtual +0.0, the sign flip is fused into
//     the load as a real multiply by +-1.0 (like :91);
//   * phase 1 (n_pad >= 2^11): one warp per 1024-row chunk of a column —
//     coalesced 256 B loads, two padded shared-memory transposes, all ten
//     low-bit stages in registers, coalesced store of the chunk to T;
//   * phase 2: the remaining high bits in passes of <= 10 bits over tiles of
//     W consecutive low indices x 2^hb combinations of the pass bits, loaded
//     straight into registers (the pass bits are register bits, the low bits
//     are lane bits, so every load is coalesced), one shared-memory exchange
//     between the two 5-bit register rounds; the last pass runs only for tiles
//     that hold a sampled row and emits just those rows;
//   * n_pad <= 2^10: one CTA per column does everything on chip;
//   * every butterfly is v[j] = s + t, v[j+h] = s - t in increasing bit order,
//     and the two scalings (1/sqrt(n_pad) at :47-48, sqrt(n_pad/m) at
//     :95-97) are separate rounded multiplies of host-computed constants.
#include "common.cuh"
#include "tma.cuh"

#include <cstring>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <vector>

namespace ihs_b200 {

namespace {
constexpr int kSmallL = 10;  // n_pad <= 2^10: single on-chip kernel
constexpr int kChunkL = 10;  // phase-1 chunk: 1024 rows per warp

constexpr int kP2Threads = 256;

__host__ __device__ constexpr int padded(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int pad32(int i) { return i + (i >> 5); }

__device__ __forceinline__ void bfly(double& a, double& b) {
    const double s = a, t = b;
    a = __dadd_rn(s, t);
    b = __dsub_rn(s, t);
}

__device__ __forceinline__ double eps_mul(const uint32_t* __restrict__ signbits, int64_t r, double a) {
    const uint32_t w = __ldg(signbits + (r >> 5));
    return __dmul_rn(((w >> (r & 31)) & 1u) ? 1.0 : -1.0, a);
}

// ------------------------------------------------------------ small n_pad
// One CTA per column: the whole transform and the gather on chip.
template <int L>
__global__ void __launch_bounds__((1 << L) / 16 > 0 ? (1 << L) / 16 : 1)
srht_small_kernel(const double* __restrict__ A, int64_t n, int64_t lda, const uint32_t* __restrict__ signbits,
                  const int2* __restrict__ entries, int n_entries, double s1, double s2, double* __restrict__ SA,
                  int64_t m) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    constexpr int N = 1 << L;
    constexpr int THREADS = N / 16 > 0 ? N / 16 : 1;
    constexpr int E = N / THREADS;
    extern __shared__ double xs[];
    const int64_t j = blockIdx.x;
    const double* Acol = A + j * lda;
    const int t = threadIdx.x;
    for (int e = t; e < N; e += THREADS) xs[padded(e)] = (e < n) ? eps_mul(signbits, e, __ldg(Acol + e)) : 0.0;
    __syncthreads();
    if constexpr (L < 4) {
        double v[E];
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = xs[padded(c)];
#pragma unroll
        for (int s = 0; s < L; ++s)
#pragma unroll
            for (int c = 0; c < E; ++c)
                if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
        for (int c = 0; c < E; ++c) xs[padded(c)] = v[c];
        __syncthreads();
    } else {
        int done = 0;
        while (done < L) {  // 4-bit register rounds (the last one shifted down)
            const int b0 = (done + 4 <= L) ? done : L - 4;
            const int lo_stage = done - b0;
            const int base = ((t >> b0) << (b0 + 4)) | (t & ((1 << b0) - 1));
            double v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = xs[padded(base | (c << b0))];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                if (s < lo_stage) continue;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) xs[padded(base | (c << b0))] = v[c];
            __syncthreads();
            done = b0 + 4;
        }
    }
    for (int q = t; q < n_entries; q += THREADS) {
        const int2 rk = entries[q];
        SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(xs[padded(rk.x)], s1), s2);
    }
}

// ------------------------------------------------------------ phase 1
// 8-byte async copy global -> shared with an L2 evict-first policy (A is
// read exactly once); src_valid == false zero-fills (+0.0).
__device__ __forceinline__ void cp_async8_zfill(double* dst, const double* src, bool src_valid, uint64_t pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;\n" ::"r"(s), "l"(src),
                 "r"(src_valid ? 8 : 0), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Phase-1 chunk pipeline of one warp. A chunk (1024 rows of one column) is
// staged by cp.async into a padded shared buffer (lane = row bits 0-4), then
// transformed: the sign is applied on the first transposed read (lane holds
// rows 32*lane .. 32*lane+31: one sign word per lane), bits 0-4 and 5-9 run
// in registers around one in-place shared-memory transpose.
constexpr int kP1Buf = 1024 + 32;
__device__ __forceinline__ void cp_async8(double* dst, const double* src, uint64_t pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, 8, %2;\n" ::"r"(s), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void p1_issue(double* buf, const double* col, int64_t n, int64_t r0, uint64_t pol) {
    const int lane = threadIdx.x & 31;
    if (r0 + 1024 <= n) {  // full chunk: constant offsets, no predicates
        const double* src = col + r0 + lane;
        double* dst = buf + lane;
#pragma unroll
        for (int c = 0; c < 32; ++c) cp_async8(dst + 33 * c, src + 32 * c, pol);
        return;
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        const int64_t r = r0 + (c << 5) + lane;
        cp_async8_zfill(buf + pad32((c << 5) | lane), r < n ? col + r : col, r < n, pol);
    }
}

// Per-lane store predicate of the masked phase-1 store: bit c set when
// element (c << 5) + lane belongs to a low-index group (of 2^logw indices)
// that a sampled row reads in the emitting pass; all ones when unmasked.
__device__ __forceinline__ uint32_t p1_store_bits(const uint32_t* __restrict__ mask, int logw) {
    if (mask == nullptr) return 0xffffffffu;
    const int lane = threadIdx.x & 31;
    uint32_t bits = 0u;
    for (int c = 0; c < 32; ++c) {
        const int g = ((c << 5) + lane) >> logw;
        bits |= ((__ldg(mask + (g >> 5)) >> (g & 31)) & 1u) << c;
    }
    return bits;
}

// x * (+-1.0) done as a sign-bit flip (exact: IEEE multiplication by -1 only
// flips the sign, so this equals the reference's rounded product bit for bit).
__device__ __forceinline__ double flip_sign(double a, uint32_t flip_bit31) {
    return __hiloint2double(__double2hiint(a) ^ (int)flip_bit31, __double2loint(a));
}

// Store a transformed chunk (lane holds element 32c + lane in v[c]): masked, the kept low-index groups
// to dst[element]; compact (lmap), element l to dst[lmap[l] * cstride] when some sampled row has low
// index l (lmap[l] = its rank u among the distinct low indices, else -1).
__device__ __forceinline__ void p1_store(const double (&v)[32], double* __restrict__ dst, uint32_t store_bits,
                                         const short* __restrict__ lmap, int64_t cstride) {
    const int lane = threadIdx.x & 31;
    if (lmap) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const int u = __ldg(lmap + ((c << 5) | lane));
            if (u >= 0) dst[(int64_t)u * cstride] = v[c];
        }
        return;
    }
    double* out = dst + lane;
#pragma unroll
    for (int c = 0; c < 32; ++c)
        if ((store_bits >> c) & 1u) out[c << 5] = v[c];
}

// Transform the chunk staged in buf and store the kept elements to dst.
__device__ __forceinline__ void p1_transform_store(double* buf, const uint32_t* __restrict__ signbits, int64_t n,
                                                   int64_t r0, double* __restrict__ dst, uint32_t store_bits,
                                                   const short* __restrict__ lmap = nullptr, int64_t cstride = 0) {
    const int lane = threadIdx.x & 31;
    const int64_t rl = r0 + (lane << 5);
    // flip bit c = row rl + c gets -1 (sign bit 0); padded rows stay +0.0
    uint32_t flip = 0u;
    if (rl < n) {
        flip = ~__ldg(signbits + (rl >> 5));
        if (rl + 32 > n) flip &= (1u << (n - rl)) - 1u;
    }
    double v[32];
    const double* row = buf + 33 * lane;  // pad32((lane << 5) | c) = 33 * lane + c
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = flip_sign(row[c], (flip << (31 - c)) & 0x80000000u);
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
    for (int c = 0; c < 32; ++c) buf[33 * lane + c] = v[c];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = buf[33 * c + lane];  // pad32((c << 5) | lane)
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    p1_store(v, dst, store_bits, lmap, cstride);
    __syncwarp();  // the buffer is refilled by the next issue
}

// ---- phase 1 fed by TMA (default)
// A full chunk (1024 rows of one column, 8 KiB) arrives by two 3-level TMA
// boxes of 32 x 128 B rows under SWIZZLE_128B: the even 128-byte rows of the
// chunk (rows 32l .. 32l+15 of lane l's block) to shared rows 0..31 and the
// odd ones to rows 32..63. Element e of the chunk (global row rg = e >> 4,
// k = e & 15) sits at shared row r' = 32 (rg & 1) + (rg >> 1), 16-byte unit
// (k >> 1) ^ (r' & 7), half k & 1. Both transposed reads are then free of
// bank conflicts: lane l owns shared rows l and 32 + l (its 32 elements, as
// 16-byte pairs), and the second read (lane = element bits 0-4) hits 16
// distinct 8-byte slots of one 128-byte row per half-warp. Only one elected
// lane issues the copies; the LSU/MIO queue carries just the shared accesses.
constexpr int kChunkDoubles = 1024;
__device__ __forceinline__ int p1_swz(int e) {
    const int rg = e >> 4, k = e & 15;
    const int rp = ((rg & 1) << 5) | (rg >> 1);
    return (rp << 4) | (((k >> 1) ^ (rp & 7)) << 1) | (k & 1);
}

struct ChunkMaps {
    CUtensorMap even, odd;  // (16 doubles, 32 rows of stride 256 B, chunk, column)
};

// rows >= n read as +0.0 (partial / padded chunks: synchronous, swizzled)
__device__ __forceinline__ void p1_sync_load(double* buf, const double* __restrict__ col, int64_t n, int64_t r0) {
    const int lane = threadIdx.x & 31;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
        const int e = (c << 5) | lane;
        const int64_t r = r0 + e;
        buf[p1_swz(e)] = r < n ? col[r] : 0.0;
    }
    __syncwarp();
}

// A is read exactly once: evict-first, so the T columns the emitting pass reads next stay in L2
__device__ __forceinline__ void p1_tma_issue(double* buf, const ChunkMaps* maps, int q, int j, uint64_t* bar,
                                             uint64_t pol) {
    tma::fence_proxy_async();
    tma::mbar_expect_tx(bar, kChunkDoubles * sizeof(double));
    tma::load_4d_hint(buf, &maps->even, 0, 0, q, j, bar, pol);
    tma::load_4d_hint(buf + kChunkDoubles / 2, &maps->odd, 0, 0, q, j, bar, pol);
}

__device__ __forceinline__ void p1_transform_store_swz(double* buf, const uint32_t* __restrict__ signbits, int64_t n,
                                                       int64_t r0, double* __restrict__ dst, uint32_t store_bits,
                                                       const short* __restrict__ lmap = nullptr,
                                                       int64_t cstride = 0) {
    const int lane = threadIdx.x & 31;
    const int64_t rl = r0 + (lane << 5);
    uint32_t flip = 0u;
    if (rl < n) {
        flip = ~__ldg(signbits + (rl >> 5));
        if (rl + 32 > n) flip &= (1u << (n - rl)) - 1u;
    }
    double v[32];
    double* row0 = buf + (lane << 4);         // shared row lane: elements 32 lane + 0..15
    double* row1 = buf + ((32 + lane) << 4);  // shared row 32 + lane: elements 32 lane + 16..31
    const int x = lane & 7;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const double2 a = *reinterpret_cast<const double2*>(row0 + ((u ^ x) << 1));
        const double2 b = *reinterpret_cast<const double2*>(row1 + ((u ^ x) << 1));
        v[2 * u] = a.x;
        v[2 * u + 1] = a.y;
        v[16 + 2 * u] = b.x;
        v[17 + 2 * u] = b.y;
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = flip_sign(v[c], (flip << (31 - c)) & 0x80000000u);
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        *reinterpret_cast<double2*>(row0 + ((u ^ x) << 1)) = make_double2(v[2 * u], v[2 * u + 1]);
        *reinterpret_cast<double2*>(row1 + ((u ^ x) << 1)) = make_double2(v[16 + 2 * u], v[17 + 2 * u]);
    }
    __syncwarp();
    // lane = element bits 0-4: element 32c + lane at shared row 32 (lane >> 4) + c
    const double* col = buf + ((lane >> 4) << 9) + (lane & 1);
    const int lu = (lane & 15) >> 1;
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = col[(c << 4) + ((lu ^ (c & 7)) << 1)];
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    p1_store(v, dst, store_bits, lmap, cstride);
    __syncwarp();  // the buffer is refilled by the next issue
}

__device__ __forceinline__ double* align1024(void* p) {
    const uint32_t a = tma::smem_u32(p);
    return reinterpret_cast<double*>(static_cast<unsigned char*>(p) + ((1024u - (a & 1023u)) & 1023u));
}

// Persistent phase 1 over TMA-fed two-slot rings (one per warp).
constexpr int kP1TWarps = 12;
constexpr size_t kP1TSmem = (size_t)kP1TWarps * 2 * kChunkDoubles * sizeof(double) + kP1TWarps * 2 * 8 + 1024;
__global__ void __launch_bounds__(32 * kP1TWarps, 1)
srht_phase1_tma_kernel(const __grid_constant__ ChunkMaps maps, const double* __restrict__ A, int64_t n, int64_t lda,
                       const uint32_t* __restrict__ signbits, double* __restrict__ T, int64_t n_pad, int lcpc,
                       int64_t nfull, int64_t total_chunks, const uint32_t* __restrict__ mask, int logw,
                       const short* __restrict__ lmap, int64_t U) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ unsigned char p1t_raw[];
    double* base = align1024(p1t_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* ring = base + warp * (2 * kChunkDoubles);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + kP1TWarps * 2 * kChunkDoubles) + 2 * warp;
    if (lane == 0) {
        tma::mbar_init(&bars[0], 1);
        tma::mbar_init(&bars[1], 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    const int64_t cmask = (int64_t{1} << lcpc) - 1;
    const int64_t nw = (int64_t)gridDim.x * kP1TWarps;
    const uint32_t store_bits = p1_store_bits(mask, logw);
    auto issue = [&](int64_t chunk, int slot) {
        if (lane == 0 && chunk < total_chunks && (chunk & cmask) < nfull)
            p1_tma_issue(ring + slot * kChunkDoubles, &maps, (int)(chunk & cmask), (int)(chunk >> lcpc), &bars[slot],
                         policy_evict_first());
    };
    uint32_t parity = 0u;
    int slot = 0;
    int64_t chunk = (int64_t)blockIdx.x * kP1TWarps + warp;
    issue(chunk, 0);
    for (; chunk < total_chunks; chunk += nw) {
        issue(chunk + nw, slot ^ 1);
        const int64_t q = chunk & cmask, j = chunk >> lcpc;
        const int64_t r0 = q << kChunkL;
        double* buf = ring + slot * kChunkDoubles;
        if (q < nfull) {
            tma::mbar_wait(&bars[slot], (parity >> slot) & 1u);
            parity ^= 1u << slot;
        } else {
            p1_sync_load(buf, A + j * lda, n, r0);
        }
        if (lmap)  // compact T[j][q][u]: this chunk's U kept values are one contiguous run
            p1_transform_store_swz(buf, signbits, n, r0, T + (j * (cmask + 1) + q) * ((U + 7) & ~int64_t{7}), 0u,
                                   lmap, 1);
        else
            p1_transform_store_swz(buf, signbits, n, r0, T + j * n_pad + r0, store_bits);
        slot ^= 1;
    }
}

// Persistent warp-per-chunk phase 1: bits 0..9 of every 1024-row chunk of
// every column -> T. Each warp streams its chunks through a two-slot ring
// (the next chunk is in flight while the current one is transformed), so HBM
// sees ~kP1AWarps x 8 KiB of reads in flight per SM at all times.
constexpr int kP1AWarps = 12;
__global__ void __launch_bounds__(32 * kP1AWarps, 1)
srht_phase1_kernel(const double* __restrict__ A, int64_t n, int64_t lda, const uint32_t* __restrict__ signbits,
                   double* __restrict__ T, int64_t n_pad, int lcpc, int64_t total_chunks,
                   const uint32_t* __restrict__ mask, int logw, const short* __restrict__ lmap, int64_t U) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double p1_smem[];  // kP1AWarps x 2 x kP1Buf doubles
    const int64_t cmask = (int64_t{1} << lcpc) - 1;  // chunks per column = 2^lcpc
    const int warp = threadIdx.x >> 5;
    double* ring = p1_smem + warp * (2 * kP1Buf);
    const uint64_t pol = policy_evict_first();
    const int64_t nw = (int64_t)gridDim.x * kP1AWarps;
    auto issue = [&](int64_t chunk, int slot) {
        if (chunk < total_chunks)
            p1_issue(ring + slot * kP1Buf, A + (chunk >> lcpc) * lda, n, (chunk & cmask) << kChunkL, pol);
        cp_async_commit();
    };
    const uint32_t store_bits = p1_store_bits(mask, logw);
    int slot = 0;
    int64_t chunk = (int64_t)blockIdx.x * kP1AWarps + warp;
    issue(chunk, 0);
    for (; chunk < total_chunks; chunk += nw) {
        issue(chunk + nw, slot ^ 1);
        cp_async_wait1();
        __syncwarp();
        const int64_t j = chunk >> lcpc;
        const int64_t r0 = (chunk & cmask) << kChunkL;
        if (lmap)
            p1_transform_store(ring + slot * kP1Buf, signbits, n, r0,
                               T + (j * (cmask + 1) + (chunk & cmask)) * ((U + 7) & ~int64_t{7}), 0u, lmap, 1);
        else
            p1_transform_store(ring + slot * kP1Buf, signbits, n, r0, T + j * n_pad + r0, store_bits);
        slot ^= 1;
    }
    cp_async_wait0();
}


// ------------------------------------------------------------ phase 2
// One CTA per (tile, column): bits [lo, lo+HB) of kTileElems elements = W
// consecutive low indices x 2^HB pass combinations. Round 1: register bits =
// pass bits [0, RB1); round 2 (RB2 = HB - RB1 > 0): register bits = pass bits
// [RB1, HB) after one shared-memory exchange. emit: write the tile's sampled
// rows (entries) instead of the tile.
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
template <int HB, int TH = kP2Threads>
struct P2Geom {
    static constexpr int RB1 = HB < 5 ? HB : 5;
    static constexpr int E = 1 << RB1;             // registers per thread
    static constexpr int W = TH * E / (1 << HB);   // consecutive low indices per tile
    static constexpr int LOGW = ilog2c(W);
    static_assert(W >= 1 && (1 << LOGW) == W, "tile width");
};

// One CTA: bits [lo, lo+HB) of the tile whose element (b, w) sits at
// Tcol[(b << lo) + w]; emit -> the tile's sampled rows go to SA, else the
// tile is written back in place. CG: T loads bypass L1 (written by other
// CTAs of the same fused launch).
struct CtaBar {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// barrier over the `count` threads of a warp group (named barrier `id`)
struct GroupBar {
    int id, count;
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
    }
};

// CMAJOR: the tile is stored c-major (element (b, w) at (b & 31) TH + (b >> 5) W + w, the layout the L2-resident
// kernel writes), so round 1's load of register c is one contiguous TH-double run across the threads
template <int HB, bool CG, class Bar = CtaBar, int TH = kP2Threads, bool CMAJOR = false>
__device__ __forceinline__ void p2_tile(double* __restrict__ xs, double* __restrict__ Tcol, int lo, bool emit,
                                        int4 tile, const int2* __restrict__ entries, int64_t j, double s1, double s2,
                                        double* __restrict__ SA, int64_t m, int t = threadIdx.x, Bar bar = Bar(),
                                        int row_lo = -1) {
    constexpr int RB1 = P2Geom<HB, TH>::RB1;
    constexpr int RB2 = HB - RB1;
    constexpr int E = P2Geom<HB, TH>::E;
    constexpr int W = P2Geom<HB, TH>::W;
    const int w = t % W;
    const int g = t / W;  // 2^RB2 groups
    double v[E];
    // round 1: register c = pass bits [0, RB1), g = pass bits [RB1, HB)
#pragma unroll
    for (int c = 0; c < E; ++c) {
        const double* src = CMAJOR ? Tcol + c * TH + t : Tcol + ((int64_t)((g << RB1) | c) << lo) + w;
        v[c] = CG ? __ldcg(src) : *src;
    }
#pragma unroll
    for (int s = 0; s < RB1; ++s)
#pragma unroll
        for (int c = 0; c < E; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    if constexpr (HB > 10) {
        // three rounds (pass bits [0,5), [5,10), [10,HB)), in the reference's bit order; thread group g
        // (NG = 2^(HB-5) of them) covers the bits a round does not hold in registers
        constexpr int NG = 1 << (HB - RB1);
        constexpr int RB3 = HB - 10, G3 = 1 << RB3, GRPS3 = E / G3;
        static_assert(E == 32 && NG * E == (1 << HB), "three-round tile geometry");
#pragma unroll
        for (int c = 0; c < E; ++c) xs[pad32(((g << RB1) | c) * W + w)] = v[c];
        bar();
        // round 2: registers = bits [5,10); g = bits [0,5) | bits [10,HB) << 5
#pragma unroll
        for (int c2 = 0; c2 < E; ++c2) {
            const int b = (g & 31) | (c2 << 5) | ((g >> 5) << 10);
            v[c2] = xs[pad32(b * W + w)];
        }
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
            for (int c = 0; c < E; ++c)
                if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
        bar();  // every round-2 read is done before the buffer is rewritten
#pragma unroll
        for (int c2 = 0; c2 < E; ++c2) {
            const int b = (g & 31) | (c2 << 5) | ((g >> 5) << 10);
            xs[pad32(b * W + w)] = v[c2];
        }
        bar();
        // round 3: registers (grp, c3) = bits [10,HB) = c3, bits [0,10) = g + grp * NG
#pragma unroll
        for (int grp = 0; grp < GRPS3; ++grp)
#pragma unroll
            for (int c3 = 0; c3 < G3; ++c3) {
                const int b = (g + grp * NG) | (c3 << 10);
                v[grp * G3 + c3] = xs[pad32(b * W + w)];
            }
#pragma unroll
        for (int s = 0; s < RB3; ++s)
#pragma unroll
            for (int grp = 0; grp < GRPS3; ++grp)
#pragma unroll
                for (int c3 = 0; c3 < G3; ++c3)
                    if (!(c3 & (1 << s))) bfly(v[grp * G3 + c3], v[grp * G3 + (c3 | (1 << s))]);
        if (!emit) {
#pragma unroll
            for (int grp = 0; grp < GRPS3; ++grp)
#pragma unroll
                for (int c3 = 0; c3 < G3; ++c3) {
                    const int b = (g + grp * NG) | (c3 << 10);
                    Tcol[((int64_t)b << lo) + w] = v[grp * G3 + c3];
                }
            return;
        }
        bar();
#pragma unroll
        for (int grp = 0; grp < GRPS3; ++grp)
#pragma unroll
            for (int c3 = 0; c3 < G3; ++c3) {
                const int b = (g + grp * NG) | (c3 << 10);
                xs[pad32(b * W + w)] = v[grp * G3 + c3];
            }
    } else if constexpr (RB2 > 0) {
        // exchange: element (b, w) at xs[pad32(b*W + w)]
#pragma unroll
        for (int c = 0; c < E; ++c) xs[pad32(((g << RB1) | c) * W + w)] = v[c];
        bar();
        // round 2: thread (w, g2) with g2 in [0, 2^RB2), register (grp, c2):
        // pass bits [0, RB1) = g2 + grp * 2^RB2, pass bits [RB1, HB) = c2
        constexpr int G2 = 1 << RB2;
        constexpr int GRPS = E / G2;
        const int g2 = g;
#pragma unroll
        for (int grp = 0; grp < GRPS; ++grp)
#pragma unroll
            for (int c2 = 0; c2 < G2; ++c2) {
                const int b = (g2 + grp * G2) | (c2 << RB1);
                v[grp * G2 + c2] = xs[pad32(b * W + w)];
            }
#pragma unroll
        for (int s = 0; s < RB2; ++s)
#pragma unroll
            for (int grp = 0; grp < GRPS; ++grp)
#pragma unroll
                for (int c2 = 0; c2 < G2; ++c2)
                    if (!(c2 & (1 << s))) bfly(v[grp * G2 + c2], v[grp * G2 + (c2 | (1 << s))]);
        if (!emit) {
#pragma unroll
            for (int grp = 0; grp < GRPS; ++grp)
#pragma unroll
                for (int c2 = 0; c2 < G2; ++c2) {
                    const int b = (g2 + grp * G2) | (c2 << RB1);
                    Tcol[((int64_t)b << lo) + w] = v[grp * G2 + c2];
                }
            return;
        }
        bar();
#pragma unroll
        for (int grp = 0; grp < GRPS; ++grp)
#pragma unroll
            for (int c2 = 0; c2 < G2; ++c2) {
                const int b = (g2 + grp * G2) | (c2 << RB1);
                xs[pad32(b * W + w)] = v[grp * G2 + c2];
            }
    } else {
        if (!emit) {
#pragma unroll
            for (int c = 0; c < E; ++c) Tcol[((int64_t)((g << RB1) | c) << lo) + w] = v[c];
            return;
        }
#pragma unroll
        for (int c = 0; c < E; ++c) xs[pad32(((g << RB1) | c) * W + w)] = v[c];
    }
    bar();
    const int64_t bmask = (int64_t{1} << HB) - 1;
    const int rlo = row_lo >= 0 ? row_lo : lo;  // row bit where the pass bits start (tile-major T: 10)
    for (int q = tile.y + t; q < tile.z; q += TH) {
        const int2 rk = entries[q];
        const int64_t r = rk.x;
        const int b = (int)((r >> rlo) & bmask);
        const int ww = (int)(r & (W - 1));
        SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(xs[pad32(b * W + ww)], s1), s2);
    }
}

// One CTA per (tile, column) of a phase-2 pass.
template <int HB, int TH>
__global__ void __launch_bounds__(TH)
srht_phase2_kernel(double* __restrict__ T, int64_t n_pad, int lo, const int4* __restrict__ tiles, int emit,
                   const int2* __restrict__ entries, double s1, double s2, double* __restrict__ SA, int64_t m) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double xs[];
    constexpr int LOGW = P2Geom<HB, TH>::LOGW;
    const int64_t j = blockIdx.y;
    int64_t base;
    int4 tile = make_int4(0, 0, 0, 0);
    if (emit) {
        tile = tiles[blockIdx.x];
        base = tile.x;
    } else {
        // enumerate tiles: low part (bits LOGW .. lo-1) and high part (bits >= lo+HB)
        const int64_t low_tiles = (int64_t{1} << lo) >> LOGW;
        const int64_t tid = blockIdx.x;
        base = ((tid % low_tiles) << LOGW) | ((tid / low_tiles) << (lo + HB));
    }
    p2_tile<HB, false, CtaBar, TH>(xs, T + j * n_pad + base, lo, emit != 0, tile, entries, j, s1, s2, SA, m);
}

// Two-round emitting pass for 11-12 high bits (n_pad = 2^21, 2^22): 256 threads x 64 registers hold the same
// 16384-element tile as the 512-thread three-round pass (W = 8 / 4 low indices, so the host's tiles and entries
// are shared), but cover 6 pass bits per round: round 1 = pass bits [0, 6) straight from T, one shared-memory
// exchange, round 2 = pass bits [6, HB), then the tile is staged once for the emission. One exchange instead of
// two (three shared-memory passes over the tile instead of five, three barriers instead of five); the padding
// (4 doubles per 256) keeps every exchange access conflict-free for both thread mappings.
// threads per two-round tile: 128 for 12 high bits (W = 2; 64 KiB tiles, two CTAs per SM so one CTA's copy
// overlaps the other's butterflies), 256 for 11 (W = 8)
template <int HB>
constexpr int r2_threads() { return HB == 12 ? 128 : 256; }
// padding of the exchange buffer: W doubles per TH (both thread mappings then hit distinct banks)
template <int TH, int W>
__host__ __device__ constexpr int pad_r2(int i) { return i + ((i >> ilog2c(TH)) << ilog2c(W)); }
template <int HB>
constexpr size_t r2_smem() {
    constexpr int TH = r2_threads<HB>();
    return (size_t)pad_r2<TH, (TH * 64 >> HB)>(TH * 64) * sizeof(double) + 128;
}

// TMA (tmap != nullptr): the tile arrives by ONE 4-D tensor copy (low index w, pass bits [6, HB), pass bits
// [0, 6), column) into xs as w + W g + 256 c, so round 1 reads register c of all threads as one conflict-free run
// and no thread issues global loads; the exchange then rewrites the buffer in the padded layout.
template <int HB, bool TMAP, int kR2Threads = r2_threads<HB>()>
__global__ void __launch_bounds__(kR2Threads, kR2Threads == 128 ? 2 : 1)
srht_phase2_r2_kernel(const __grid_constant__ CUtensorMap tmap, const double* __restrict__ T, int64_t n_pad,
                      const int4* __restrict__ tiles, const int2* __restrict__ entries, double s1, double s2,
                      double* __restrict__ SA, int64_t m) {
    static_assert(HB >= 8 && HB <= 12, "two-round tile geometry");
    constexpr int E = 64;
    constexpr int R2 = HB - 6;                     // bits of round 2 (5 or 6)
    constexpr int W = kR2Threads * E >> HB;        // low indices per tile
    constexpr int NG = kR2Threads / W;             // thread groups of round 1 (= 2^(HB - 6))
    auto pad_r2 = [](int i) { return ihs_b200::pad_r2<kR2Threads, W>(i); };
    constexpr int GR = E >> R2;                    // round-2 columns per thread (2 or 1)
    constexpr int lo = kChunkL;
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ unsigned char r2_raw[];
    double* xs = reinterpret_cast<double*>(r2_raw + ((128u - (tma::smem_u32(r2_raw) & 127u)) & 127u));
    const int t = threadIdx.x;
    const int w = t % W, g = t / W;
    const int64_t j = blockIdx.y;
    const int4 tile = tiles[blockIdx.x];
    double v[E];
    // round 1: register c = pass bits [0, 6), g = pass bits [6, HB)
    if constexpr (TMAP) {
        __shared__ alignas(8) uint64_t bar;
        if (t == 0) {
            tma::mbar_init(&bar, 1);
            tma::fence_mbar_init();
        }
        __syncthreads();
        if (t == 0) {
            tma::mbar_expect_tx(&bar, kR2Threads * E * sizeof(double));
            tma::load_4d(xs, &tmap, tile.x, 0, 0, (int)j, &bar);
        }
        tma::mbar_wait(&bar, 0);
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = xs[c * kR2Threads + t];
        __syncthreads();  // the copy's layout is read once; the exchange below rewrites the buffer
    } else {
        const double* Tcol = T + j * n_pad + tile.x;
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = Tcol[((int64_t)((g << 6) | c) << lo) + w];
    }
#pragma unroll
    for (int s_ = 0; s_ < 6; ++s_)
#pragma unroll
        for (int c = 0; c < E; ++c)
            if (!(c & (1 << s_))) bfly(v[c], v[c | (1 << s_)]);
#pragma unroll
    for (int c = 0; c < E; ++c) xs[pad_r2((((g << 6) | c) * W) + w)] = v[c];
    __syncthreads();
    // round 2: register (grp, c2) = pass bits [6, HB) = c2, pass bits [0, 6) = g + grp NG
#pragma unroll
    for (int grp = 0; grp < GR; ++grp)
#pragma unroll
        for (int c2 = 0; c2 < (1 << R2); ++c2)
            v[grp * (1 << R2) + c2] = xs[pad_r2(((c2 << 6) | (g + grp * NG)) * W + w)];
#pragma unroll
    for (int s_ = 0; s_ < R2; ++s_)
#pragma unroll
        for (int grp = 0; grp < GR; ++grp)
#pragma unroll
            for (int c2 = 0; c2 < (1 << R2); ++c2)
                if (!(c2 & (1 << s_))) bfly(v[grp * (1 << R2) + c2], v[grp * (1 << R2) + (c2 | (1 << s_))]);
    __syncthreads();  // every round-2 read is done before the buffer is rewritten
#pragma unroll
    for (int grp = 0; grp < GR; ++grp)
#pragma unroll
        for (int c2 = 0; c2 < (1 << R2); ++c2)
            xs[pad_r2(((c2 << 6) | (g + grp * NG)) * W + w)] = v[grp * (1 << R2) + c2];
    __syncthreads();
    constexpr int64_t bmask = (int64_t{1} << HB) - 1;
    for (int q = tile.y + t; q < tile.z; q += kR2Threads) {
        const int2 rk = entries[q];
        const int64_t r = rk.x;
        const int b = (int)((r >> lo) & bmask);
        const int ww = (int)(r & (W - 1));
        SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(xs[pad_r2(b * W + ww)], s1), s2);
    }
}

// Compact emitting pass (n_pad = 2^20, compact T[j][h][u] with u padded to 8, h = row bits 10..19): a CTA
// stages 8 consecutive ranks of column j with coalesced 64-byte reads into per-rank shared rows (element h
// at the XOR swizzle row h>>5, column (h ^ (h>>5)) & 31, so both orientations below are conflict-free);
// warp w then runs the ten high butterflies of rank u0 + w in the reference's order entirely in
// registers — bits 0-4 with the register index = h bits 0-4, a write-back, bits 5-9 with the register
// index = h bits 5-9 — and emits the sampled rows with that low index, scaled twice.
constexpr int kCmpU = 8;      // ranks (warps) per CTA
constexpr int kCmpRow = 1025;  // shared row per rank (odd: ranks start on different banks)
__device__ __forceinline__ int cmp_swz(int row, int col) { return (row << 5) | (col ^ row); }
__global__ void __launch_bounds__(32 * kCmpU) srht_phase2_compact_kernel(const double* __restrict__ Tc, int64_t U,
                                                                         const int4* __restrict__ ranges,
                                                                         const int2* __restrict__ entries,
                                                                         double s1, double s2,
                                                                         double* __restrict__ SA, int64_t m) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double cbuf[];  // [kCmpU][kCmpRow]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t u0 = (int64_t)blockIdx.x * kCmpU, j = blockIdx.y;
    const int nu = (int)(U - u0 < kCmpU ? U - u0 : kCmpU);
    const int64_t Up = (U + 7) & ~int64_t{7};  // row stride: 64-byte aligned runs of 8 ranks
    {
        const double* src = Tc + j * 1024 * Up + u0;
        const int uu = threadIdx.x % kCmpU, h0 = threadIdx.x / kCmpU;  // 32 h per pass, 8 ranks each
        double t[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) t[i] = uu < nu ? __ldcs(src + (int64_t)(h0 + 32 * i) * Up + uu) : 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int h = h0 + 32 * i;
            cbuf[uu * kCmpRow + cmp_swz(h >> 5, h & 31)] = t[i];
        }
    }
    __syncthreads();
    if (warp >= nu) return;
    double* buf = cbuf + warp * kCmpRow;
    double v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = buf[cmp_swz(lane, c)];  // h = 32 lane + c: bits 0-4 in the register
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
    for (int c = 0; c < 32; ++c) buf[cmp_swz(lane, c)] = v[c];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = buf[cmp_swz(c, lane)];  // h = 32 c + lane: bits 5-9 in the register
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    const int4 rg = ranges[u0 + warp];
    for (int q = rg.y; q < rg.z; ++q) {
        const int2 e = entries[q];
        const int h = e.x >> 10;
        double sel = 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) sel = c == (h >> 5) ? v[c] : sel;
        const double val = __shfl_sync(0xffffffffu, sel, h & 31);
        if (lane == 0) SA[(int64_t)e.y + j * m] = __dmul_rn(__dmul_rn(val, s1), s2);
    }
}

// ------------------------------------------------------------ L2-resident single launch (default)
// The two-kernel path moves every column three times through HBM (A read, T write, T read: 69 GB -> 208 GB per
// C4 sketch). This persistent kernel (one CTA per SM) keeps T on chip in the 126 MB L2 instead:
//   * T is a ring of NS column slots (NS x n_pad doubles, ~96 MB), each column stored TILE-MAJOR: the emitting
//     tile of W consecutive low indices x 2^H high combinations is one contiguous 8192-double block, c-major
//     inside ((b & 63) 128 + (b >> 6) W + w), so the emitting pass reads it with coalesced L2 loads and then
//     drops the lines with discard.global.L2 (no write-back unless L2 pressure evicted them first);
//   * phase-1 warps (8, one chunk each) work on CTA-wide items of 8 chunks q = c + 64 (8 g' + j), whose pieces
//     of every tile are adjacent, so an item stores whole 128-byte lines (the 16-byte pieces of a lone chunk
//     made ~4.6 G L2 write requests per C4 sketch; whole lines make 0.55-0.8 G). A is prefetched into L2
//     (cp.async.bulk.prefetch.tensor) 4 items ahead, then copied chunk by chunk into shared memory by TMA;
//   * two emitting groups (128 threads x 64 registers each: the two-round pass of srht_phase2_r2_kernel)
//     take tiles; setmaxnreg moves registers from the phase-1 warps to them;
//   * items and tiles are claimed in dependency order from two atomic counters: an emitting tile of column j
//     waits until every phase-1 item of j has stored (per-column counter, released once per run of a CTA's
//     items in one column), a phase-1 item of column j + NS until every tile of column j is emitted (its slot
//     is free). Every wait is on work claimed earlier by a running CTA, so no wait can deadlock, whatever the
//     residency;
//   * A arrives with an L2 evict-first hint (read once), T is stored with evict-last.
// Butterfly order, the sign flip and the two scalings are exactly those of the two-kernel path.
constexpr int kL2P1Warps = 8;        // phase-1 warps: one chunk of every item each (each a 2-slot TMA ring)
constexpr int kL2EmitThreads = 128;  // emitting group: two-round tiles of 128 threads x 64 registers
constexpr int kL2EmitGroups = 2;     // independent emitting groups (one warp of each per SM sub-partition)
constexpr int kL2Slots = 1;          // chunk buffers per phase-1 warp (A comes from L2: see kL2Prefetch)
constexpr int kL2Threads = kL2P1Warps * 32 + kL2EmitGroups * kL2EmitThreads;
constexpr int l2_threads(int eg) { return kL2P1Warps * 32 + eg * kL2EmitThreads; }
constexpr int kL2TileElems = kL2EmitThreads * 64;
// registers: the launch grants 168 per thread (384 threads); phase-1 warps hand some to the emitting group
// (64 doubles of tile per thread) with setmaxnreg: 256 x 128 + 128 x 232 <= 384 x 168
constexpr int kL2Prefetch = 4;  // phase-1 items whose A is prefetched into L2 ahead of the current one
constexpr int kL2Queue = 16;    // claimed-item queue (> prefetch distance + 1)
constexpr int kL2P1Regs = 96;
constexpr int kL2EmitRegs = 160;
static_assert(kL2P1Warps * 32 * kL2P1Regs + kL2EmitGroups * kL2EmitThreads * kL2EmitRegs <=
                  kL2Threads * ((65536 / kL2Threads) & ~7),
              "register budget");
// phase-1 rings (8 warps x 2 x 8 KiB) + padded exchange buffer + mbarriers + 1 KiB alignment slack
template <int HB, int S1 = kL2Slots, int EG = kL2EmitGroups>
constexpr size_t l2_smem() {
    return (size_t)(kL2P1Warps * S1 * kChunkDoubles +
                    EG * pad_r2<kL2EmitThreads, (kL2TileElems >> HB)>(kL2TileElems) + 2 * kL2P1Warps) *
               sizeof(double) +
           1024 + 64;
}

__device__ __forceinline__ void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st2_hint(double* p, double a, double b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
template <int HB, int P1T, bool TS, int S1, int EG>
__global__ void __launch_bounds__(l2_threads(EG), 1)
srht_l2_kernel(const __grid_constant__ ChunkMaps maps, const __grid_constant__ CUtensorMap tmap_T, const double* __restrict__ A, int64_t n, int64_t lda,
               const uint32_t* __restrict__ signbits, double* __restrict__ T, int64_t nfull, int64_t d, int ns,
               const int4* __restrict__ tiles, int n_tiles, const uint32_t* __restrict__ tile_bits,
               const int2* __restrict__ entries, double s1, double s2, double* __restrict__ SA, int64_t m,
               int* __restrict__ ctl, int discard, int dbg, int pf, int tpol) {
    static_assert(HB >= 9 && HB <= 12, "L2-resident tile geometry");
    constexpr int E = 64;                       // registers per emitting thread
    constexpr int R2 = HB - 6;                  // pass bits of round 2
    constexpr int GR = E >> R2;                 // round-2 columns per thread (1 .. 8)
    constexpr int TE = kL2TileElems;            // tile elements: W low indices x 2^HB high combinations
    constexpr int W = TE >> HB;                 // 2 (HB = 12) .. 16 (HB = 9)
    constexpr int LOGW = ilog2c(W);
    constexpr int NG = kL2EmitThreads / W;      // round-1 thread groups (= 2^(HB - 6))
    constexpr int64_t NPAD = int64_t{1} << (HB + kChunkL);
    constexpr int CPC = 1 << HB;                // chunks per column
    constexpr int P1W = kL2P1Warps / P1T;       // warps (= chunks) of a phase-1 item; P1T teams take items independently
    constexpr int IPC = CPC / P1W;              // phase-1 items per column
    constexpr int RUN = P1W * W;                // contiguous doubles one item stores into each tile
    constexpr int UPT = RUN / 2;                // ... as 16-byte units
    constexpr int SWZ = (W / 2) * (UPT >= 8 ? 1 : 8 / UPT);  // XOR stride of the chunk copies' 16-byte units
    static_assert(NG >= P1W && RUN % 8 == 0, "an item fills whole 64-byte halves of 128-byte lines");
    auto pad = [](int i) { return pad_r2<kL2EmitThreads, W>(i); };
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ unsigned char l2_raw[];
    double* base = align1024(l2_raw);
    double* rings = base;                                // kL2P1Warps x 2 chunk buffers (1 KiB aligned)
    // rings: slot sl of phase-1 warp w at rings + (sl kL2P1Warps + w) kChunkDoubles, so a team's chunks of one slot
    // are contiguous (the tensor store's item buffer)
    double* xs0 = base + kL2P1Warps * S1 * kChunkDoubles;  // emitting-tile exchange buffers (one per group)
    uint64_t* bars = reinterpret_cast<uint64_t*>(xs0 + EG * pad(TE));  // S1 per phase-1 warp
    __shared__ int s_claim_all[P1T][kL2Queue];
    __shared__ uint32_t s_bits[16];  // occupancy of the (<= 512) low-index tiles
    __shared__ int s_p2_all[EG][2];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t < 16) s_bits[t] = tile_bits[t];
    __syncthreads();
    int* p1_counter = ctl;
    int* p2_counter = ctl + 1;
    int* done1 = ctl + 2;
    int* done2 = ctl + 2 + d;
    if (warp < kL2P1Warps) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kL2P1Regs));
        // ---- phase-1 teams (P1T teams of P1W warps, named barriers 2 and 5). Item it of column col = it / IPC,
        // r = it % IPC, holds the P1W chunks q = (r & 63) + 64 (P1W (r >> 6) + j), j = warp in the team: their
        // high indices b = q differ only in b >> 6, so in the c-major tile layout below their W-element pieces of
        // every tile are adjacent — the item stores RUN contiguous doubles (whole 128-byte lines for 8-chunk
        // items, halves for 4) per tile instead of 16-byte scraps per chunk. Two teams overlap one team's chunk
        // copies with the other's butterflies.
        const int team = warp / P1W;
        const int j = warp % P1W;
        const int tt = t - team * P1W * 32;  // thread index in the team
        int* s_claim = s_claim_all[team];
        auto slotbuf = [&](int sl_, int w_) { return rings + ((size_t)sl_ * kL2P1Warps + w_) * kChunkDoubles; };
        uint64_t* bar = bars + S1 * warp;
        if (lane == 0) {
            tma::mbar_init(&bar[0], 1);
            if (S1 > 1) tma::mbar_init(&bar[1], 1);
            tma::fence_mbar_init();
        }
        __syncwarp();
        const GroupBar pbar{team == 0 ? 2 : 5, P1W * 32};
        const int64_t total = d * IPC;
        const uint64_t pol_first = policy_evict_first();
        const uint64_t pol_last = tpol == 1 ? policy_evict_normal() : tpol == 2 ? pol_first : policy_evict_last();
        auto chunk_of = [&](int64_t it, int jj) -> int64_t {
            const int r = (int)(it & (IPC - 1));
            return (r & 63) + 64 * ((r >> 6) * P1W + jj);
        };
        auto issue = [&](int64_t it, int sl) {
            if (it >= total || lane != 0) return;
            const int64_t q = chunk_of(it, j), col = it / IPC;
            if (q >= nfull) return;
            double* buf = slotbuf(sl, warp);
            tma::fence_proxy_async();
            tma::mbar_expect_tx(&bar[sl], kChunkDoubles * sizeof(double));
            tma::load_4d_hint(buf, &maps.even, 0, 0, (int)q, (int)col, &bar[sl], pol_first);
            tma::load_4d_hint(buf + kChunkDoubles / 2, &maps.odd, 0, 0, (int)q, (int)col, &bar[sl], pol_first);
        };
        // A of item it -> L2 (no shared memory): issued pf items ahead so the shared-memory copy, one
        // item ahead, comes from L2
        auto prefetch = [&](int64_t it) {
            if (it >= total || lane != 0) return;
            const int64_t q = chunk_of(it, j), col = it / IPC;
            if (q >= nfull) return;
            tma::prefetch_4d_l2(&maps.even, 0, 0, (int)q, (int)col);
            tma::prefetch_4d_l2(&maps.odd, 0, 0, (int)q, (int)col);
        };
        // claimed items: queue slot k % kL2Queue holds the k-th item of this CTA; thread 0 claims item k +
        // pf + 1 during item k (visible to the group after the item's barriers)
        if (tt == 0)
            for (int k = 0; k <= pf; ++k) s_claim[k] = atomicAdd(p1_counter, 1);
        pbar();
        int64_t cur = s_claim[0];
        issue(cur, 0);
        for (int k = 1; k < pf; ++k) prefetch(s_claim[k]);
        uint32_t phase = 0u;  // bit s: parity of slot s
        int sl = 0;
        int kq = 0;   // queue index of cur
        int run = 0;  // thread 0: items of the current column stored since the last release
        int64_t slot_ok_col = -1;  // thread 0: the latest column whose ring slot is known to be free
        // 16-byte units of a chunk's natural-order copy are XOR-swizzled by its warp so the item store's reads
        // (8 lanes = the 8 chunks' pieces of one tile) hit distinct banks
        auto swz = [](int e, int jj) { return ((((e >> 1) ^ ((jj * SWZ) & 7))) << 1) | (e & 1); };
        // the sign word of the current item's chunk, loaded one item ahead (its L2 round trip overlaps an item)
        auto sign_word = [&](int64_t it) -> uint32_t {
            if (it >= total) return 0u;
            const int64_t rl = (chunk_of(it, j) << kChunkL) + (lane << 5);
            return rl < n ? __ldg(signbits + (rl >> 5)) : 0u;
        };
        uint32_t sw = sign_word(cur);
        while (cur < total) {
            if (S1 > 1) issue(s_claim[(kq + 1) % kL2Queue], sl ^ 1);
            prefetch(s_claim[(kq + pf) % kL2Queue]);
            int claimed = 0;  // published only after the store loop: the atomic's round trip overlaps the item
            if (tt == 0) claimed = atomicAdd(p1_counter, 1);
            const int64_t q = chunk_of(cur, j), col = cur / IPC;
            const int64_t r0 = q << kChunkL;
            double* buf = slotbuf(sl, warp);
            if (q < nfull) {
                tma::mbar_wait(&bar[sl], (phase >> sl) & 1u);
                phase ^= 1u << sl;
            } else {
                p1_sync_load(buf, A + col * lda, n, r0);
            }
            // the ten low stages (as p1_transform_store_swz)
            const int64_t rl = r0 + (lane << 5);
            uint32_t flip = 0u;
            if (rl < n) {
                flip = ~sw;
                if (rl + 32 > n) flip &= (1u << (n - rl)) - 1u;
            }
            double v[32];
            double* row0 = buf + (lane << 4);
            double* row1 = buf + ((32 + lane) << 4);
            const int x = lane & 7;
            if (dbg != 2 && dbg != 4 && dbg != 5 && dbg != 6) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 a = *reinterpret_cast<const double2*>(row0 + ((u ^ x) << 1));
                const double2 b = *reinterpret_cast<const double2*>(row1 + ((u ^ x) << 1));
                v[2 * u] = a.x;
                v[2 * u + 1] = a.y;
                v[16 + 2 * u] = b.x;
                v[17 + 2 * u] = b.y;
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = flip_sign(v[c], (flip << (31 - c)) & 0x80000000u);
#pragma unroll
            for (int s_ = 0; s_ < 5; ++s_)
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (!(c & (1 << s_))) bfly(v[c], v[c | (1 << s_)]);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                *reinterpret_cast<double2*>(row0 + ((u ^ x) << 1)) = make_double2(v[2 * u], v[2 * u + 1]);
                *reinterpret_cast<double2*>(row1 + ((u ^ x) << 1)) = make_double2(v[16 + 2 * u], v[17 + 2 * u]);
            }
            __syncwarp();
            const double* colp = buf + ((lane >> 4) << 9) + (lane & 1);
            const int lu = (lane & 15) >> 1;
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = colp[(c << 4) + ((lu ^ (c & 7)) << 1)];
            __syncwarp();
#pragma unroll
            for (int s_ = 0; s_ < 5; ++s_)
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (!(c & (1 << s_))) bfly(v[c], v[c | (1 << s_)]);
            // element e = 32c + lane back into the slot in natural (swizzled) order
            if constexpr (TS) {
                // the item's output in the tensor-store box layout [te][chunk j][w] (128-byte swizzle, as the
                // store map's SWIZZLE_128B expects): it overwrites every slot of the team, so all chunks must
                // have been read first
                pbar();
                char* ib = reinterpret_cast<char*>(slotbuf(sl, team * P1W));
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int e = (c << 5) | lane;
                    const int L = (((e >> LOGW) * P1W + j) * W + (e & (W - 1))) * 8;
                    *reinterpret_cast<double*>(ib + (L ^ (((L >> 7) & 7) << 4))) = v[c];
                }
                tma::fence_proxy_async();  // generic writes before the async-proxy (TMA) read of the buffer
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) buf[swz((c << 5) | lane, j)] = v[c];
            }
            }  // dbg != 2
            // the slot's previous column must be fully emitted before it is overwritten
            if (tt == 0 && col >= ns && col != slot_ok_col) {
                while (ld_relaxed(done2 + (col - ns)) < n_tiles) __nanosleep(64);
                (void)ld_acquire(done2 + (col - ns));
                slot_ok_col = col;
            }
            pbar();  // every chunk of the item is in its slot; the column's ring slot is free
            // store: tile te gets, at c 128 + 8 (r >> 6) W (c = r & 63), the pieces [chunk j][w] of the 8 chunks
            const int r = (int)(cur & (IPC - 1));
            if constexpr (TS) {
                // one thread stores the whole item with (1024 / W) / 256 tensor copies: RUN contiguous doubles
                // into each tile, evict-last (the emitting side reads them next)
                constexpr int BOXT = (1024 / W) < 256 ? (1024 / W) : 256;
                if (tt == 0 && !(dbg >= 3 && dbg <= 5 || dbg == 7)) {
                    const char* ib = reinterpret_cast<const char*>(slotbuf(sl, team * P1W));
#pragma unroll
                    for (int h = 0; h < (1024 / W) / BOXT; ++h)
                        tma::store_5d_hint(&tmap_T, 0, (r >> 6) * P1W * W / 16, h * BOXT, r & 63, (int)(col % ns),
                                           ib + (size_t)h * BOXT * P1W * W * 8, pol_last);
                    tma::bulk_commit();
                    if (dbg != 8) tma::bulk_wait_read0();  // the slots are refilled by the next item's copies
                }
            }
            double* dst0 = T + (col % ns) * NPAD + (r & 63) * kL2EmitThreads + (r >> 6) * P1W * W;
#pragma unroll 4
            for (int i = 0; i < (TS || (dbg >= 3 && dbg <= 5 || dbg == 7) ? 0 : kChunkDoubles / 64); ++i) {
                const int u = i * (P1W * 32) + tt;  // 16-byte unit of the item's output
                const int te = u / UPT;
                const int kk = (u % UPT) << 1;            // double offset inside the run
                const int jj = kk >> LOGW, w = kk & (W - 1);
                if (!((s_bits[te >> 5] >> (te & 31)) & 1u)) continue;
                const double2 val = *reinterpret_cast<const double2*>(slotbuf(sl, team * P1W + jj) +
                                                                      swz((te << LOGW) + w, jj));
                st2_hint(dst0 + (int64_t)te * TE + kk, val.x, val.y, pol_last);
            }
            if (tt == 0) s_claim[(kq + pf + 1) % kL2Queue] = claimed;
            pbar();  // the item's stores are issued and every slot sl is read (the next TMA may refill it)
            if (S1 == 1) issue(s_claim[(kq + 1) % kL2Queue], 0);
            // completions are released once per run of this CTA's items in one column (its claims only move to
            // later columns): one release (a memory barrier for thread 0) per column instead of per item
            if (tt == 0) {
                ++run;
                const int64_t nx = s_claim[(kq + 1) % kL2Queue];
                if (nx >= total || nx / IPC != col) {
                    if constexpr (TS) {  // the tensor stores' global writes are performed and ordered before the
                        tma::bulk_wait0();  // release that publishes them
                        tma::fence_proxy_async_global();
                    }
                    red_release_add(done1 + col, run);
                    run = 0;
                }
            }
            ++kq;
            cur = s_claim[kq % kL2Queue];
            sw = sign_word(cur);
            if (S1 > 1) sl ^= 1;
        }
        return;
    }
    // ---- emitting group (warps 8-11, named barrier 1): tiles in (column, tile) order, each the two-round pass
    // of srht_phase2_r2_kernel over the c-major tile (element (b, w) at (b & 63) 128 + (b >> 6) W + w)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kL2EmitRegs));
    const int pg = (t - kL2P1Warps * 32) / kL2EmitThreads;  // emitting group
    const int gt = (t - kL2P1Warps * 32) % kL2EmitThreads;
    const int w = gt & (W - 1), g = gt >> LOGW;
    const GroupBar gbar{pg == 0 ? 1 : 3 + pg, kL2EmitThreads};
    double* xs = xs0 + pg * pad(TE);
    int* s_p2 = s_p2_all[pg];
    const int64_t total2 = d * (int64_t)n_tiles;
    if (gt == 0) s_p2[0] = atomicAdd(p2_counter, 1);
    gbar();
    int64_t item = s_p2[0];
    int par2 = 1;
    constexpr int64_t bmask = (int64_t{1} << HB) - 1;
    int run2 = 0;               // gt 0: tiles of the current column emitted since the last release
    int64_t ready_col = -1;     // gt 0: the latest column whose phase 1 is known complete
    while (item < total2) {
        int claimed = 0;  // claimed early (published at the end): its round trip overlaps this tile
        if (gt == 0) claimed = atomicAdd(p2_counter, 1);
        const int64_t col = item / n_tiles, ti = item % n_tiles;
        const int4 tile = __ldg(tiles + ti);
        if (gt == 0 && col != ready_col) {  // relaxed polls, one acquire (polling with ld.acquire would
            // invalidate the SM's L1 on every poll)
            while (ld_relaxed(done1 + col) < IPC) __nanosleep(32);
            (void)ld_acquire(done1 + col);
            ready_col = col;
        }
        gbar();
        if (dbg == 1 || dbg == 5 || dbg == 6 || dbg == 7) {  // timing probe: the emitting side only hands tiles on
            if (gt == 0) s_p2[par2] = claimed;
            gbar();
            if (gt == 0) {
                ++run2;
                const int64_t nx = s_p2[par2];
                if (nx >= total2 || nx / n_tiles != col) {
                    red_release_add(done2 + col, run2);
                    run2 = 0;
                }
            }
            item = s_p2[par2];
            par2 ^= 1;
            continue;
        }
        const double* tptr = T + (col % ns) * NPAD + (int64_t)(tile.x >> LOGW) * TE;
        double v[E];
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = __ldcg(tptr + c * kL2EmitThreads + gt);
#pragma unroll
        for (int s_ = 0; s_ < 6; ++s_)
#pragma unroll
            for (int c = 0; c < E; ++c)
                if (!(c & (1 << s_))) bfly(v[c], v[c | (1 << s_)]);
        // register c of this warp's 32 threads is one 256-byte run read by this warp only: once consumed, lane l
        // drops the runs of c = 2l, 2l + 1 (no write-back of T)
        if (discard) {
            __syncwarp();
            const double* lines = tptr + (gt & ~31);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                discard_l2(lines + ((2 * lane + k) * kL2EmitThreads));
                discard_l2(lines + ((2 * lane + k) * kL2EmitThreads) + 16);
            }
        }
#pragma unroll
        for (int c = 0; c < E; ++c) xs[pad((((g << 6) | c) * W) + w)] = v[c];
        gbar();
#pragma unroll
        for (int grp = 0; grp < GR; ++grp)
#pragma unroll
            for (int c2 = 0; c2 < (1 << R2); ++c2)
                v[grp * (1 << R2) + c2] = xs[pad(((c2 << 6) | (g + grp * NG)) * W + w)];
#pragma unroll
        for (int s_ = 0; s_ < R2; ++s_)
#pragma unroll
            for (int grp = 0; grp < GR; ++grp)
#pragma unroll
                for (int c2 = 0; c2 < (1 << R2); ++c2)
                    if (!(c2 & (1 << s_))) bfly(v[grp * (1 << R2) + c2], v[grp * (1 << R2) + (c2 | (1 << s_))]);
        gbar();  // every round-2 read is done before the buffer is rewritten
#pragma unroll
        for (int grp = 0; grp < GR; ++grp)
#pragma unroll
            for (int c2 = 0; c2 < (1 << R2); ++c2)
                xs[pad(((c2 << 6) | (g + grp * NG)) * W + w)] = v[grp * (1 << R2) + c2];
        gbar();
        for (int q = tile.y + gt; q < tile.z; q += kL2EmitThreads) {
            const int2 rk = entries[q];
            const int64_t rr = rk.x;
            const int b = (int)((rr >> kChunkL) & bmask);
            const int ww = (int)(rr & (W - 1));
            SA[(int64_t)rk.y + col * m] = __dmul_rn(__dmul_rn(xs[pad(b * W + ww)], s1), s2);
        }
        if (gt == 0) s_p2[par2] = claimed;
        gbar();  // the tile is emitted (xs free again) and every T read of it is done
        if (gt == 0) {
            ++run2;
            const int64_t nx = s_p2[par2];
            if (nx >= total2 || nx / n_tiles != col) {
                red_release_add(done2 + col, run2);
                run2 = 0;
            }
        }
        item = s_p2[par2];
        par2 ^= 1;
    }
}


// Row-sharded SRHT combine (H_{n_pad} = H_P (x) H_{n_pad/P}, shard index =
// top log2(P) row bits): U holds every shard's unscaled partial T_p[r_lo(k)]
// for every sampled row k ([P][m][d], shard-major, as an all-gather lays it
// out). The top stages run over p in increasing bit order exactly like the
// reference's high butterflies; the value at p = r_hi(k) is scaled twice.
template <int LOGP>
__global__ void srht_combine_kernel(const double* __restrict__ U, int64_t m, int64_t d,
                                    const uint8_t* __restrict__ hi, double s1, double s2, double* __restrict__ SA) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    constexpr int P = 1 << LOGP;
    const int64_t md = m * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < md; e += (int64_t)gridDim.x * blockDim.x) {
        double v[P];
#pragma unroll
        for (int p = 0; p < P; ++p) v[p] = U[p * md + e];
#pragma unroll
        for (int s = 0; s < LOGP; ++s)
#pragma unroll
            for (int p = 0; p < P; ++p)
                if (!(p & (1 << s))) bfly(v[p], v[p | (1 << s)]);
        const int target = hi[e % m];
        double out = v[0];
#pragma unroll
        for (int p = 1; p < P; ++p)
            if (p == target) out = v[p];
        SA[e] = __dmul_rn(__dmul_rn(out, s1), s2);
    }
}

int pass_w(int hb, int th) {
    const int rb1 = std::min(hb, 5);
    return th * (1 << rb1) / (1 << hb);
}
// elements of one phase-2 tile: W low indices x 2^hb pass combinations
// (32 th for hb >= 5, th * 2^hb below)
int64_t pass_tile_elems(int hb, int th) { return (int64_t)pass_w(hb, th) << hb; }
int pass_logw(const SrhtPlan& p) {
    int logw = 0;
    while ((1 << (logw + 1)) <= pass_w(p.pass_hb[p.npass - 1], p.p2t)) ++logw;
    return logw;
}

template <int L>
void launch_small(const SrhtPlan& p, const double* A, const uint32_t* signbits, const int2* entries, double* SA,
                  cudaStream_t st) {
    constexpr int N = 1 << L;
    constexpr int THREADS = N / 16 > 0 ? N / 16 : 1;
    const size_t smem = (size_t)padded(N) * sizeof(double) + 64;
    LAUNCH_PDL(srht_small_kernel<L>, (unsigned)p.d, THREADS, smem, st, A, p.n, p.lda, signbits, entries, (int)p.m,
           p.scale1, p.scale2, SA, p.sa_ld);
}
using SmallFn = void (*)(const SrhtPlan&, const double*, const uint32_t*, const int2*, double*, cudaStream_t);
const SmallFn kSmall[kSmallL + 1] = {launch_small<0>, launch_small<1>, launch_small<2>, launch_small<3>,
                                     launch_small<4>, launch_small<5>, launch_small<6>, launch_small<7>,
                                     launch_small<8>, launch_small<9>, launch_small<10>};

// 4-D map of the phase-1 output T (n_pad x d, column-major) for the two-round tiles: dims (low index, pass
// bits [6, HB), pass bits [0, 6), column), box (W, 2^(HB-6), 64, 1)
bool r2_tensor_map(const double* T, int64_t n_pad, int64_t d, int HB, CUtensorMap* out) {
    static const bool disabled = [] {
        const char* e = std::getenv("IHS_SRHT_R2_TMA");
        return e && e[0] == '0';
    }();
    if (disabled || (reinterpret_cast<uintptr_t>(T) & 15) != 0) return false;
    const int W = (HB == 12 ? 128 : 256) * 64 >> HB, NG = 1 << (HB - 6);
    const cuuint64_t dims[4] = {(cuuint64_t)1 << kChunkL, (cuuint64_t)NG, 64, (cuuint64_t)d};
    const cuuint64_t strides[3] = {(cuuint64_t)64 << (kChunkL + 3), (cuuint64_t)1 << (kChunkL + 3),
                                   (cuuint64_t)n_pad * sizeof(double)};
    const cuuint32_t box[4] = {(cuuint32_t)W, (cuuint32_t)NG, 64, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return tma_encode_fn()(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(T), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HB>
void launch_r2(const SrhtPlan& p, const double* T, const int4* tiles, int n_tiles, const int2* entries, double* SA,
               cudaStream_t st) {
    dim3 grid((unsigned)n_tiles, (unsigned)p.d);
    CUtensorMap map;
    if (r2_tensor_map(T, p.n_pad, p.d, HB, &map)) {
        IHS_SMEM_ATTR((srht_phase2_r2_kernel<HB, true>), (int)r2_smem<HB>());
        LAUNCH_PDL((srht_phase2_r2_kernel<HB, true>), grid, r2_threads<HB>(), r2_smem<HB>(), st, map, T, p.n_pad, tiles,
                   entries, p.scale1, p.scale2, SA, p.sa_ld);
    } else {
        std::memset(&map, 0, sizeof(map));
        IHS_SMEM_ATTR((srht_phase2_r2_kernel<HB, false>), (int)r2_smem<HB>());
        LAUNCH_PDL((srht_phase2_r2_kernel<HB, false>), grid, r2_threads<HB>(), r2_smem<HB>(), st, map, T, p.n_pad, tiles,
                   entries, p.scale1, p.scale2, SA, p.sa_ld);
    }
}

template <int HB, int TH>
void launch_pass(const SrhtPlan& p, double* T, int lo, const int4* tiles, int n_tiles, bool emit, const int2* entries,
                 double* SA, cudaStream_t st) {
    const size_t smem = (size_t)pad32((int)pass_tile_elems(HB, TH)) * sizeof(double) + 64;
    IHS_SMEM_ATTR((srht_phase2_kernel<HB, TH>), (int)smem);
    const int64_t tiles_per_col = p.n_pad / pass_tile_elems(HB, TH);
    const unsigned gx = emit ? (unsigned)n_tiles : (unsigned)tiles_per_col;
    if (gx == 0) return;
    dim3 grid(gx, (unsigned)p.d);
    LAUNCH_PDL((srht_phase2_kernel<HB, TH>), grid, TH, smem, st, T, p.n_pad, lo, tiles, emit ? 1 : 0, entries, p.scale1,
           p.scale2, SA, p.sa_ld);
}

// Tensor maps of the full 1024-row chunks of A (even / odd 128-byte rows of
// each chunk, see p1_tma_issue), cached per (A, lda, nfull, d); false when
// TMA is unavailable or disabled (IHS_SRHT_NO_TMA=1).
bool srht_chunk_maps(const double* A, int64_t lda, int64_t nfull, int64_t d, ChunkMaps* out) {
    static const bool disabled = [] {
        const char* e = std::getenv("IHS_SRHT_NO_TMA");
        return e && e[0] == '1';
    }();
    if (disabled || (lda * (int64_t)sizeof(double)) % 16 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0)
        return false;
    struct Entry {
        const double* A;
        int64_t lda, nfull, d;
        ChunkMaps maps;
    };
    static std::vector<Entry> cache;
    static std::mutex mu;  // rank threads of an emulated group share the process
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
        if (e.A == A && e.lda == lda && e.nfull == nfull && e.d == d) {
            *out = e.maps;
            return true;
        }
    ChunkMaps m;
    const cuuint64_t dims[4] = {16, 32, (cuuint64_t)nfull, (cuuint64_t)d};
    const cuuint64_t strides[3] = {256, 8192, (cuuint64_t)lda * sizeof(double)};
    const cuuint32_t box[4] = {16, 32, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    for (int h = 0; h < 2; ++h) {
        const CUresult r = tma_encode_fn()(h ? &m.odd : &m.even, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                           const_cast<double*>(A + 16 * h), dims, strides, box, estr,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return false;
    }
    if (cache.size() >= 32) cache.erase(cache.begin());
    cache.push_back(Entry{A, lda, nfull, d, m});
    *out = m;
    return true;
}

using PassFn = void (*)(const SrhtPlan&, double*, int, const int4*, int, bool, const int2*, double*, cudaStream_t);
const PassFn kPass[13] = {nullptr,
                          launch_pass<1, 256>,
                          launch_pass<2, 256>,
                          launch_pass<3, 256>,
                          launch_pass<4, 256>,
                          launch_pass<5, 256>,
                          launch_pass<6, 256>,
                          launch_pass<7, 256>,
                          launch_pass<8, 256>,
                          launch_pass<9, 256>,
                          launch_pass<10, 256>,
                          launch_pass<11, 256>,
                          launch_pass<12, 256>};
const PassFn kPass512[13] = {nullptr,
                             launch_pass<1, 512>,
                             launch_pass<2, 512>,
                             launch_pass<3, 512>,
                             launch_pass<4, 512>,
                             launch_pass<5, 512>,
                             launch_pass<6, 512>,
                             launch_pass<7, 512>,
                             launch_pass<8, 512>,
                             launch_pass<9, 512>,
                             launch_pass<10, 512>,
                             launch_pass<11, 512>,   // three-round tiles: 2^21 / 2^22 rows in one pass
                             launch_pass<12, 512>};
const PassFn kPass128[11] = {nullptr,
                             launch_pass<1, 128>,
                             launch_pass<2, 128>,
                             launch_pass<3, 128>,
                             launch_pass<4, 128>,
                             launch_pass<5, 128>,
                             launch_pass<6, 128>,
                             launch_pass<7, 128>,
                             launch_pass<8, 128>,
                             launch_pass<9, 128>,
                             launch_pass<10, 128>};
}  // namespace

// threads per phase-2 tile of the two-kernel path (IHS_SRHT_P2T=128/256/512 for A/B runs)
int p2_threads_default() {
    static const int v = [] {
        const char* e = std::getenv("IHS_SRHT_P2T");
        const int t = e ? std::atoi(e) : 0;
        return (t == 128 || t == 256 || t == 512) ? t : kP2Threads;
    }();
    return v;
}

SrhtPlan srht_plan(int64_t n, int64_t d, int64_t lda, int64_t m) {
    SrhtPlan p{};
    p.n = n;
    p.d = d;
    p.lda = lda;
    p.m = m;
    p.sa_ld = m;
    int64_t np = 1;
    int logn = 0;
    while (np < n) { np <<= 1; ++logn; }
    p.n_pad = np;
    p.logn = logn;
    if (logn > 30) fail(IHS_INVALID_INPUT, "srht_sketch: n_pad above 2^30 not supported");
    if (logn <= kSmallL) {
        p.L = logn;
        p.H = 0;
        p.npass = 0;
    } else {
        p.L = kChunkL;
        p.H = logn - kChunkL;
        if (p.H > 10 && p.H <= 12) {
            // one pass of 11-12 high bits with 512-thread three-round tiles (W = 8 / 4 low indices):
            // saves the T -> T round trip of a second pass (n_pad = 2^21, 2^22)
            p.npass = 1;
            p.pass_lo[0] = kChunkL;
            p.pass_hb[0] = p.H;
            p.scale1 = 1.0 / std::sqrt(static_cast<double>(np));
            p.scale2 = std::sqrt(static_cast<double>(np) / static_cast<double>(m));
            static const int p2t_env = [] {  // IHS_SRHT_P2T=256: 256-thread three-round tiles (A/B)
                const char* e = std::getenv("IHS_SRHT_P2T");
                return e ? std::atoi(e) : 0;
            }();
            static const bool r2_plan = [] {  // the two-round emitting pass (default; IHS_SRHT_R2=0: three rounds)
                const char* e = std::getenv("IHS_SRHT_R2");
                return !(e && e[0] == '0');
            }();
            // host tiles match the emitting pass: two-round 128-thread tiles for 12 bits (W = 2 = the 256-thread
            // three-round geometry), 256-thread ones for 11 (W = 8 = the 512-thread geometry)
            p.p2t = r2_plan ? (p.H == 12 ? 256 : 512) : (p2t_env == 256 ? 256 : 512);
            p.compact = 0;
            return p;
        }
        // split H into passes of <= 10 bits, as even as possible
        const int np_ = (p.H + 9) / 10;
        int lo = kChunkL;
        p.npass = np_;
        for (int i = 0; i < np_; ++i) {
            const int hb = p.H / np_ + (i < p.H % np_ ? 1 : 0);
            p.pass_lo[i] = lo;
            p.pass_hb[i] = hb;
            lo += hb;
        }
    }
    // exactly the reference's host expressions (sketch.hpp:47 and :95)
    p.scale1 = 1.0 / std::sqrt(static_cast<double>(np));
    p.scale2 = std::sqrt(static_cast<double>(np) / static_cast<double>(m));
    p.p2t = p2_threads_default();
    p.compact = 0;
    return p;
}

SrhtPlan srht_plan_shard(int64_t n_real, int64_t n_loc, int64_t d, int64_t lda, int64_t m) {
    if (n_loc < 32 || (n_loc & (n_loc - 1)) != 0) fail(IHS_INVALID_INPUT, "srht shard: rows per shard must be 2^k >= 32");
    SrhtPlan p = srht_plan(n_loc, d, lda, m);  // geometry of an n_loc-row transform
    p.n = n_real;                               // rows >= n_real are virtual zeros
    p.scale1 = 1.0;                             // unscaled partials; the combine applies both scalings
    p.scale2 = 1.0;
    return p;
}

void srht_combine(const double* d_U, int P, int64_t m, int64_t d, const uint8_t* d_hi, double s1, double s2,
                  double* d_SA, cudaStream_t st) {
    const int64_t md = m * d;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(md, 256), 148 * 16));
    switch (P) {
        case 1: LAUNCH_PDL(srht_combine_kernel<0>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 2: LAUNCH_PDL(srht_combine_kernel<1>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 4: LAUNCH_PDL(srht_combine_kernel<2>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 8: LAUNCH_PDL(srht_combine_kernel<3>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 16: LAUNCH_PDL(srht_combine_kernel<4>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        default: fail(IHS_INVALID_INPUT, "srht shard: number of shards must be 1, 2, 4, 8 or 16");
    }
}

__global__ void srht_unpack_kernel(const double* __restrict__ G, int64_t mq, int64_t m, int64_t d,
                                   double* __restrict__ SA) {
    pdl_wait();
    const int64_t md = m * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < md; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e % m, j = e / m;
        const int64_t q = k / mq, kk = k - q * mq;
        SA[e] = G[q * mq * d + kk + j * mq];
    }
}

void srht_unpack_blocks(const double* d_G, int P, int64_t mq, int64_t m, int64_t d, double* d_SA, cudaStream_t st) {
    (void)P;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m * d, 256), 148 * 16));
    LAUNCH_PDL(srht_unpack_kernel, blocks, 256, 0, st, d_G, mq, m, d, d_SA);
}

size_t srht_scratch_bytes(const SrhtPlan& p) { return p.H > 0 ? (size_t)p.n_pad * (size_t)p.d * sizeof(double) : 0; }

bool srht_plan_l2(SrhtPlan& p) {
    // default for single-pass plans with 9..12 high bits (IHS_SRHT_L2=0: the two-kernel path; IHS_SRHT_L2_NS sets
    // the ring depth). T stays in L2, so HBM sees A and SA only.
    // Measured (device sketch, ms, two-kernel -> L2): C4 n_pad 2^22 m 8192 40.4 -> 36.3, m 131072 48.6 -> 44.6
    // (ring depth 3, 96 MB); n_pad 2^20 m 65536: C3 7.02 -> 6.77, C5 27.4 -> 26.9 (depth >= 6). Shallower rings
    // couple the two halves column by column and lose (C4 depth 2: 40.3; n_pad 2^20 depth 3: 10.2).
    static const int mode = [] {
        const char* e = std::getenv("IHS_SRHT_L2");
        return e ? std::atoi(e) : -1;
    }();
    static const int ns_env = [] {
        const char* e = std::getenv("IHS_SRHT_L2_NS");
        return e ? std::atoi(e) : 0;
    }();
    // 9 high bits (a 2^19-row column: C4 over 8 GPUs, C5 over 2) measured 18.1 vs 20.4 ms for the two-kernel path
    // (n = 2^19, d = 2048, m = 4096, incl. the SA read-back)
    const int min_h = 9;
    if (mode == 0 || p.H < min_h || p.H > 12 || p.npass != 1 || p.compact) return false;
    p.l2 = 1;
    p.p2t = kL2TileElems / 32;  // tile geometry of the host's tiles: W = 8192 >> H low indices
    const int64_t col_bytes = p.n_pad * (int64_t)sizeof(double);
    p.l2_ns = ns_env > 0 ? ns_env : (int)std::max<int64_t>(2, std::min<int64_t>(12, (96ll << 20) / col_bytes));
    return true;
}
size_t srht_l2_scratch_bytes(const SrhtPlan& p) { return (size_t)p.l2_ns * (size_t)p.n_pad * sizeof(double); }
size_t srht_l2_ctl_bytes(const SrhtPlan& p) { return (size_t)(2 + 2 * p.d) * sizeof(int) + 64; }

bool srht_plan_compact(SrhtPlan& p, const int64_t* rows) {
    // IHS_SRHT_NO_COMPACT=1 disables it; IHS_SRHT_COMPACT_MAX overrides the distinct-low-index limit
    static const bool disabled = [] {
        const char* e = std::getenv("IHS_SRHT_NO_COMPACT");
        return e && e[0] == '1';
    }();
    static const int umax = [] {
        const char* e = std::getenv("IHS_SRHT_COMPACT_MAX");
        return e ? std::atoi(e) : 640;
    }();
    if (disabled || p.H != 10 || p.npass != 1) return false;
    // measured (profiles/r01_srht_compact.txt): compact phase 1 + emitting pass beat the masked T up to
    // ~640 distinct low indices (m ~ 1000 at n_pad = 2^20); beyond that the tiled pass is faster
    std::vector<uint8_t> seen(1024, 0);
    int U = 0;
    for (int64_t k = 0; k < p.m && U <= umax; ++k) {
        uint8_t& f = seen[(size_t)(rows[k] & 1023)];
        if (!f) f = 1, ++U;
    }
    if (U > umax) return false;
    p.compact = 1;
    return true;
}

void srht_build_entries(const SrhtPlan& p, const int64_t* rows, std::vector<int2>& entries, std::vector<int4>& tiles) {
    entries.clear();
    tiles.clear();
    if (p.compact) {
        // U tiles (l, begin, end) over the distinct low indices in increasing order, then the low-index ->
        // rank map as 1024 shorts packed into 128 trailing int4
        std::vector<int> cnt(1025, 0);
        for (int64_t k = 0; k < p.m; ++k) {
            if (rows[k] < 0 || rows[k] >= p.n_pad) fail(IHS_INTERNAL_ERROR, "srht: sampled row outside the padded range");
            cnt[(size_t)(rows[k] & 1023) + 1]++;
        }
        std::vector<short> lmap(1024, -1);
        int U = 0;
        for (int l = 0; l < 1024; ++l)
            if (cnt[(size_t)l + 1] > 0) lmap[(size_t)l] = (short)U++;
        for (int l = 0; l < 1024; ++l) cnt[(size_t)l + 1] += cnt[(size_t)l];
        entries.resize((size_t)p.m);
        std::vector<int> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t k = 0; k < p.m; ++k)
            entries[(size_t)fill[(size_t)(rows[k] & 1023)]++] = make_int2((int)rows[k], (int)k);
        for (int l = 0; l < 1024; ++l)
            if (lmap[(size_t)l] >= 0) tiles.push_back(make_int4(l, cnt[(size_t)l], cnt[(size_t)l + 1], 0));
        const size_t base = tiles.size();
        tiles.resize(base + 1024 * sizeof(short) / sizeof(int4));
        std::memcpy(tiles.data() + base, lmap.data(), 1024 * sizeof(short));
        return;
    }
    if (p.H == 0) {
        entries.resize((size_t)p.m);
        for (int64_t k = 0; k < p.m; ++k) entries[(size_t)k] = make_int2((int)rows[k], (int)k);
        tiles.push_back(make_int4(0, 0, (int)p.m, 0));
        return;
    }
    // tiles of the last pass: bits [lo, lo+hb) are the pass bits, bits [0, logW)
    // the in-tile low index; a tile is identified by its base row (pass bits and
    // low bits cleared). Counting sort of the sampled rows by tile.
    const int lo = p.pass_lo[p.npass - 1], hb = p.pass_hb[p.npass - 1];
    const int64_t W = pass_w(hb, p.p2t);
    const int64_t low_tiles = (int64_t{1} << lo) / W;
    const int64_t ntiles = p.n_pad / pass_tile_elems(hb, p.p2t);
    auto tile_of = [&](int64_t r) {
        const int64_t low = (r & ((int64_t{1} << lo) - 1)) / W;
        const int64_t high = r >> (lo + hb);
        return high * low_tiles + low;
    };
    std::vector<int> count((size_t)ntiles + 1, 0);
    for (int64_t k = 0; k < p.m; ++k) {
        if (rows[k] < 0 || rows[k] >= p.n_pad || tile_of(rows[k]) >= ntiles)
            fail(IHS_INTERNAL_ERROR, "srht: sampled row outside the padded range");
        count[(size_t)tile_of(rows[k]) + 1]++;
    }
    for (int64_t t = 0; t < ntiles; ++t) count[(size_t)t + 1] += count[(size_t)t];
    entries.resize((size_t)p.m);
    std::vector<int> fill(count.begin(), count.end() - 1);
    for (int64_t k = 0; k < p.m; ++k) entries[(size_t)fill[(size_t)tile_of(rows[k])]++] = make_int2((int)rows[k], (int)k);
    for (int64_t t = 0; t < ntiles; ++t)
        if (count[(size_t)t + 1] > count[(size_t)t]) {
            const int64_t base = ((t % low_tiles) * W) | ((t / low_tiles) << (lo + hb));
            tiles.push_back(make_int4((int)base, count[(size_t)t], count[(size_t)t + 1], 0));
        }
    if (p.l2) {  // occupancy bits of the (<= 512) low-index tiles, packed into 4 trailing int4
        uint32_t bits[16] = {};
        for (int64_t t = 0; t < ntiles; ++t)
            if (count[(size_t)t + 1] > count[(size_t)t]) bits[t >> 5] |= 1u << (t & 31);
        const size_t b0 = tiles.size();
        tiles.resize(b0 + 4);
        std::memcpy(tiles.data() + b0, bits, sizeof(bits));
    }
}

bool srht_build_mask(const SrhtPlan& p, const std::vector<int4>& tiles, uint32_t mask[8]) {
    for (int k = 0; k < 8; ++k) mask[k] = 0u;
    if (p.H == 0 || p.npass != 1) return false;
    const int logw = pass_logw(p);
    if (logw < 2) return false;  // more than 256 groups: store everything
    for (const int4& t : tiles) {
        const int g = (t.x & ((1 << kChunkL) - 1)) >> logw;
        mask[g >> 5] |= 1u << (g & 31);
    }
    return true;
}

// Tensor-store map of the T ring for the L2-resident launch's phase-1 items (TS), the c-major tile layout: dims
// (u & 15, u >> 4, tile, b & 63, slot), u = (b >> 6) W + w, strides (8, 128, 8 TE, 8 ET, 8 n_pad) bytes, box
// (16, P1W W / 16, <= 256 tiles, 1, 1) under SWIZZLE_128B. False when an item's run is narrower than 128 bytes or
// the driver rejects the map (the item store loop is used then).
bool srht_l2_store_map(double* T, int HB, int ns, int p1w, CUtensorMap* out) {
    struct Entry {
        double* T;
        int HB, ns, p1w;
        CUtensorMap map;
        bool ok;
    };
    static std::vector<Entry> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
        if (e.T == T && e.HB == HB && e.ns == ns && e.p1w == p1w) {
            *out = e.map;
            return e.ok;
        }
    const int64_t TE = kL2TileElems, W = TE >> HB, npad = int64_t{1} << (HB + kChunkL);
    // the 128 doubles u = (b >> 6) W + w of one (tile, b & 63) row are contiguous: split as (u & 15, u >> 4) so
    // the box's inner dimension is exactly the 128-byte swizzle span (a narrower one is padded to it in shared
    // memory)
    if (p1w * W < 16) return false;
    const cuuint64_t dims[5] = {16, (cuuint64_t)(kL2EmitThreads / 16), (cuuint64_t)(1024 / W), 64, (cuuint64_t)ns};
    const cuuint64_t strides[4] = {128, (cuuint64_t)(8 * TE), (cuuint64_t)(8 * kL2EmitThreads), (cuuint64_t)(8 * npad)};
    const cuuint32_t box[5] = {16, (cuuint32_t)(p1w * W / 16), (cuuint32_t)std::min<int64_t>(256, 1024 / W), 1, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUtensorMap m{};
    const CUresult r = tma_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, T, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cache.size() >= 32) cache.erase(cache.begin());
    cache.push_back(Entry{T, HB, ns, p1w, m, r == CUDA_SUCCESS});
    *out = m;
    return r == CUDA_SUCCESS;
}

template <int HB, int P1T, bool TS, int S1 = kL2Slots, int EG = kL2EmitGroups>
void launch_l2_t(const SrhtPlan& p, const ChunkMaps& maps, int64_t nfull, const double* A, const uint32_t* signbits,
               double* T, const int4* tiles, int n_tiles, const int2* entries, double* SA, int* ctl, int num_sms,
               cudaStream_t st) {
    IHS_SMEM_ATTR((srht_l2_kernel<HB, P1T, TS, S1, EG>), (int)(l2_smem<HB, S1, EG>()));
    static const bool discard = [] {  // IHS_SRHT_L2_DISCARD=0: keep the consumed T lines (A/B of the discard)
        const char* e = std::getenv("IHS_SRHT_L2_DISCARD");
        return !(e && e[0] == '0');
    }();
    static const int pf = [] {  // IHS_SRHT_L2_PF: prefetch distance in items (1 .. kL2Queue - 2)
        const char* e = std::getenv("IHS_SRHT_L2_PF");
        return e ? std::max(1, std::min(kL2Queue - 2, std::atoi(e))) : kL2Prefetch;
    }();
    static const int tpol = [] {  // IHS_SRHT_L2_TPOL: L2 policy of the T stores (0 evict-last, 1 normal, 2 first)
        const char* e = std::getenv("IHS_SRHT_L2_TPOL");
        return e ? std::atoi(e) : 0;
    }();
    static const int dbg = [] {  // IHS_SRHT_L2_DBG (timing probes, wrong results): 1 emitting side idle, 2 no
        const char* e = std::getenv("IHS_SRHT_L2_DBG");  // phase-1 transform, 3 no phase-1 store, 4 = 2 + 3,
                                                         // 5 = 1 + 2 + 3, 6 = 1 + 2, 7 = 1 + 3,
                                                         // 8 = no wait for the item store's shared reads
        return e ? std::atoi(e) : 0;
    }();
    CUDA_CHECK(cudaMemsetAsync(ctl, 0, srht_l2_ctl_bytes(p), st));
    const uint32_t* bits = reinterpret_cast<const uint32_t*>(tiles + n_tiles);
    // one launch at a time per device: each sizes its T ring to most of L2, so two concurrent launches (problems
    // on different streams) would evict each other's rings; launches from different streams are chained through
    // one event per device. (Concurrency would still be deadlock-free: items and tiles are claimed in dependency
    // order by running CTAs only, so no CTA ever waits on work held by a CTA that is not resident.)
    static std::mutex mu;
    static cudaEvent_t last[64] = {};
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (last[dev & 63] == nullptr) CUDA_CHECK(cudaEventCreateWithFlags(&last[dev & 63], cudaEventDisableTiming));
    CUDA_CHECK(cudaStreamWaitEvent(st, last[dev & 63], 0));
    // one CTA per SM (the launch-bounds/smem footprint allows one)
    CUtensorMap tmap{};
    if (TS && !srht_l2_store_map(T, HB, p.l2_ns, kL2P1Warps / P1T, &tmap)) fail(IHS_INTERNAL_ERROR, "srht: T store map");
    LAUNCH_PDL((srht_l2_kernel<HB, P1T, TS, S1, EG>), (unsigned)num_sms, l2_threads(EG), (l2_smem<HB, S1, EG>()), st, maps, tmap, A, p.n, p.lda, signbits, T, nfull,
               p.d, p.l2_ns, tiles, n_tiles, bits, entries, p.scale1, p.scale2, SA, p.sa_ld, ctl, discard ? 1 : 0, dbg, pf, tpol);
    CUDA_CHECK(cudaEventRecord(last[dev & 63], st));
}
template <int HB>
void launch_l2(const SrhtPlan& p, const ChunkMaps& maps, int64_t nfull, const double* A, const uint32_t* signbits,
               double* T, const int4* tiles, int n_tiles, const int2* entries, double* SA, int* ctl, int num_sms,
               cudaStream_t st) {
    // (measured and not kept: two 4-chunk phase-1 teams, two chunk slots with one emitting group — DESIGN §7; the
    // kernel's P1T / S1 / EG template parameters still describe those shapes)
    static const int ts_env = [] {  // IHS_SRHT_L2_TS=0: phase-1 items stored by the thread loop, not by TMA
        const char* e = std::getenv("IHS_SRHT_L2_TS");
        return e ? std::atoi(e) : 1;
    }();
    CUtensorMap probe{};
    const bool ts = ts_env != 0 && srht_l2_store_map(T, HB, p.l2_ns, kL2P1Warps, &probe);
    if (ts) launch_l2_t<HB, 1, true>(p, maps, nfull, A, signbits, T, tiles, n_tiles, entries, SA, ctl, num_sms, st);
    else launch_l2_t<HB, 1, false>(p, maps, nfull, A, signbits, T, tiles, n_tiles, entries, SA, ctl, num_sms, st);
}
using L2Fn = void (*)(const SrhtPlan&, const ChunkMaps&, int64_t, const double*, const uint32_t*, double*, const int4*,
                      int, const int2*, double*, int*, int, cudaStream_t);
const L2Fn kL2[13] = {nullptr, nullptr, nullptr,      nullptr,       nullptr,       nullptr,      nullptr,
                      nullptr, nullptr, launch_l2<9>, launch_l2<10>, launch_l2<11>, launch_l2<12>};

void srht_run_device(const SrhtPlan& p, const double* d_A, const uint32_t* d_signbits, const int2* d_entries,
                     const int4* d_tiles, int n_tiles, double* d_T, double* d_SA, cudaStream_t st,
                     unsigned long long* d_ctl, int num_sms, const uint32_t* d_mask) {
    if (p.d == 0) return;
    if (p.l2) {
        ChunkMaps maps{};
        const int64_t nfull = p.n >> kChunkL;
        if (!(nfull > 0 && srht_chunk_maps(d_A, p.lda, nfull, p.d, &maps)))
            fail(IHS_INTERNAL_ERROR, "srht: the L2-resident launch needs TMA chunk maps");
        if (n_tiles > 0)
            kL2[p.H](p, maps, nfull, d_A, d_signbits, d_T, d_tiles, n_tiles, d_entries, d_SA,
                     reinterpret_cast<int*>(d_ctl), num_sms, st);
        return;
    }
    if (p.H == 0) {
        kSmall[p.L](p, d_A, d_signbits, d_entries, d_SA, st);
        return;
    }
    ChunkMaps maps;
    const int64_t nfull = p.n >> kChunkL;
    const int64_t chunks_per_col = p.n_pad >> kChunkL;
    const int64_t total = chunks_per_col * p.d;
    // compact T: n_tiles distinct low indices, their rank map after the tiles
    const short* lmap = p.compact ? reinterpret_cast<const short*>(d_tiles + n_tiles) : nullptr;
    const int64_t U = p.compact ? n_tiles : 0;
    // single pass: phase 1 writes only the groups the emitting pass reads
    const bool masked = p.npass == 1 && d_mask != nullptr && !p.compact;
    const int logw = masked ? pass_logw(p) : 0;
    if (nfull > 0 && srht_chunk_maps(d_A, p.lda, nfull, p.d, &maps)) {
        IHS_SMEM_ATTR(srht_phase1_tma_kernel, (int)kP1TSmem);
        const int64_t blocks = std::min<int64_t>(ceil_div(total, kP1TWarps), (int64_t)num_sms);
        LAUNCH_PDL(srht_phase1_tma_kernel, (unsigned)blocks, 32 * kP1TWarps, kP1TSmem, st, maps, d_A, p.n, p.lda,
               d_signbits, d_T, p.n_pad, p.logn - kChunkL, nfull, total, masked ? d_mask : nullptr, logw, lmap, U);
    } else {
        const int64_t blocks = std::min<int64_t>(ceil_div(total, kP1AWarps), (int64_t)num_sms);
        const size_t smem = (size_t)kP1AWarps * 2 * kP1Buf * sizeof(double);
        IHS_SMEM_ATTR(srht_phase1_kernel, (int)smem);
        LAUNCH_PDL(srht_phase1_kernel, (unsigned)blocks, 32 * kP1AWarps, smem, st, d_A, p.n, p.lda, d_signbits, d_T,
               p.n_pad, p.logn - kChunkL, total, masked ? d_mask : nullptr, logw, lmap, U);
    }
    if (p.compact) {
        constexpr size_t smem = (size_t)kCmpU * kCmpRow * sizeof(double);
        IHS_SMEM_ATTR(srht_phase2_compact_kernel, (int)smem);
        if (U > 0)
            LAUNCH_PDL(srht_phase2_compact_kernel, dim3((unsigned)ceil_div(U, kCmpU), (unsigned)p.d), 256, smem, st,
                       (const double*)d_T, U, d_tiles, d_entries, p.scale1, p.scale2, d_SA, p.sa_ld);
        return;
    }
    static const bool r2 = [] {  // IHS_SRHT_R2=0: the three-round 512-thread emitting pass (A/B)
        const char* e = std::getenv("IHS_SRHT_R2");
        return !(e && e[0] == '0');
    }();
    for (int i = 0; i < p.npass; ++i) {
        const bool last = i == p.npass - 1;
        if (last && n_tiles == 0) break;
        if (r2 && last && p.npass == 1 && ((p.p2t == 256 && p.pass_hb[i] == 12) || (p.p2t == 512 && p.pass_hb[i] == 11))) {
            if (p.pass_hb[i] == 11) launch_r2<11>(p, d_T, d_tiles, n_tiles, d_entries, d_SA, st);
            else launch_r2<12>(p, d_T, d_tiles, n_tiles, d_entries, d_SA, st);
            continue;
        }
        (p.p2t == 128 ? kPass128 : p.p2t == 512 ? kPass512 : kPass)[p.pass_hb[i]](p, d_T, p.pass_lo[i], d_tiles,
                                                                                  n_tiles, last, d_entries, d_SA, st);
    }
}

}  // namespace ihs_b200
