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

#include <algorithm>
#include <cmath>
#include <vector>

namespace ihs_b200 {

namespace {
constexpr int kSmallL = 10;  // n_pad <= 2^10: single on-chip kernel
constexpr int kChunkL = 10;  // phase-1 chunk: 1024 rows per warp
constexpr int kP1Warps = 8;
constexpr int kTileElems = 8192;  // phase-2 tile: 2^13 doubles (64 KiB exchange buffer)
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
// One warp: bits 0..9 of the 1024-row chunk [r0, r0+1024) of column Acol ->
// dst[0..1024). STREAM: A loads are evict-first (read exactly once).
template <bool STREAM>
__device__ __forceinline__ void p1_chunk(double* __restrict__ xs, const double* __restrict__ Acol, int64_t n,
                                         const uint32_t* __restrict__ signbits, int64_t r0, double* __restrict__ dst,
                                         const uint32_t* __restrict__ mask = nullptr, int logw = 0) {
    const int lane = threadIdx.x & 31;
    double v[32];
    // coalesced load (lane = index bits 0-4, register c = bits 5-9), sign fused
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        const int64_t r = r0 + (c << 5) + lane;
        v[c] = (r < n) ? eps_mul(signbits, r, STREAM ? __ldcs(Acol + r) : __ldg(Acol + r)) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) xs[pad32((c << 5) | lane)] = v[c];
    __syncwarp();
    // register c = index bits 0-4: stages 0..4
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = xs[pad32((lane << 5) | c)];
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
    for (int c = 0; c < 32; ++c) xs[pad32((lane << 5) | c)] = v[c];
    __syncwarp();
    // register c = index bits 5-9: stages 5..9
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = xs[pad32((c << 5) | lane)];
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    if (mask == nullptr) {
#pragma unroll
        for (int c = 0; c < 32; ++c) dst[(c << 5) + lane] = v[c];
    } else {
        // store only the low-index groups a sampled row will read in phase 2
        uint32_t mw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) mw[k] = __ldg(mask + k);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const int e = (c << 5) + lane;
            const int g = e >> logw;
            if ((mw[g >> 5] >> (g & 31)) & 1u) dst[e] = v[c];
        }
    }
}

// 8-byte async copy global -> shared; src_valid == false zero-fills (+0.0).
__device__ __forceinline__ void cp_async8_zfill(double* dst, const double* src, bool src_valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(src_valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Persistent warp-per-chunk phase 1: bits 0..9 of every 1024-row chunk of
// every column -> T. Each warp streams its chunks through a two-slot ring of
// padded shared buffers filled by cp.async (the next chunk is in flight while
// the current one is transformed), so HBM sees ~kP1Warps x 8 KiB of reads in
// flight per SM at all times. The sign is applied on the first transposed
// read (lane holds rows 32*lane .. 32*lane+31: one sign word per lane).
constexpr int kP1Buf = 1024 + 32;
constexpr int kP1Stages = 2;
constexpr int kP1AWarps = 12;
__global__ void __launch_bounds__(32 * kP1AWarps, 1)
srht_phase1_kernel(const double* __restrict__ A, int64_t n, int64_t lda, const uint32_t* __restrict__ signbits,
                   double* __restrict__ T, int64_t n_pad, int64_t chunks_per_col, int64_t total_chunks,
                   const uint32_t* __restrict__ mask, int logw) {
    extern __shared__ double p1_smem[];  // kP1AWarps x kP1Stages x kP1Buf doubles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* ring = p1_smem + warp * (kP1Stages * kP1Buf);
    const int64_t nw = (int64_t)gridDim.x * kP1AWarps;
    auto issue = [&](int64_t chunk, int slot) {
        if (chunk < total_chunks) {
            const int64_t j = chunk / chunks_per_col;
            const int64_t r0 = (chunk % chunks_per_col) << kChunkL;
            const double* col = A + j * lda;
            double* buf = ring + slot * kP1Buf;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const int64_t r = r0 + (c << 5) + lane;
                cp_async8_zfill(buf + pad32((c << 5) | lane), r < n ? col + r : col, r < n);
            }
        }
        cp_async_commit();
    };
    uint32_t mw[4] = {0u, 0u, 0u, 0u};
    if (mask != nullptr)
        for (int k = 0; k < 4; ++k) mw[k] = __ldg(mask + k);
    int slot = 0;
    int64_t chunk = (int64_t)blockIdx.x * kP1AWarps + warp;
    issue(chunk, 0);
    for (; chunk < total_chunks; chunk += nw) {
        issue(chunk + nw, slot ^ 1);
        cp_async_wait1();
        __syncwarp();
        const int64_t j = chunk / chunks_per_col;
        const int64_t r0 = (chunk % chunks_per_col) << kChunkL;
        double* buf = ring + slot * kP1Buf;
        const int64_t rl = r0 + (lane << 5);  // this lane's 32 rows (register c = bits 0-4)
        const uint32_t sw = rl < n ? __ldg(signbits + (rl >> 5)) : 0u;
        double v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const double a = buf[pad32((lane << 5) | c)];
            v[c] = (rl + c < n) ? __dmul_rn(((sw >> c) & 1u) ? 1.0 : -1.0, a) : 0.0;
        }
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
#pragma unroll
        for (int c = 0; c < 32; ++c) buf[pad32((lane << 5) | c)] = v[c];
        __syncwarp();
        // register c = index bits 5-9: stages 5..9
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = buf[pad32((c << 5) | lane)];
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
        double* dst = T + j * n_pad + r0;
        if (mask == nullptr) {
#pragma unroll
            for (int c = 0; c < 32; ++c) dst[(c << 5) + lane] = v[c];
        } else {
            // store only the low-index groups a sampled row will read in phase 2
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const int e = (c << 5) + lane;
                const int g = e >> logw;
                if ((mw[g >> 5] >> (g & 31)) & 1u) dst[e] = v[c];
            }
        }
        __syncwarp();  // the slot is refilled by the next iteration's issue
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
template <int HB>
struct P2Geom {
    static constexpr int RB1 = HB < 5 ? HB : 5;
    static constexpr int E = 1 << RB1;                    // registers per thread
    static constexpr int W = kP2Threads * E / (1 << HB);  // consecutive low indices per tile
    static constexpr int LOGW = (W >= 256) ? 8 : (W >= 128) ? 7 : (W >= 64) ? 6 : (W >= 32) ? 5 : (W >= 16) ? 4 : 3;
};

// One CTA: bits [lo, lo+HB) of the tile whose element (b, w) sits at
// Tcol[(b << lo) + w]; emit -> the tile's sampled rows go to SA, else the
// tile is written back in place. CG: T loads bypass L1 (written by other
// CTAs of the same fused launch).
template <int HB, bool CG>
__device__ __forceinline__ void p2_tile(double* __restrict__ xs, double* __restrict__ Tcol, int lo, bool emit,
                                        int4 tile, const int2* __restrict__ entries, int64_t j, double s1, double s2,
                                        double* __restrict__ SA, int64_t m) {
    constexpr int RB1 = P2Geom<HB>::RB1;
    constexpr int RB2 = HB - RB1;
    constexpr int E = P2Geom<HB>::E;
    constexpr int W = P2Geom<HB>::W;
    const int t = threadIdx.x;
    const int w = t % W;
    const int g = t / W;  // 2^RB2 groups
    double v[E];
    // round 1: register c = pass bits [0, RB1), g = pass bits [RB1, HB)
#pragma unroll
    for (int c = 0; c < E; ++c) {
        const double* src = Tcol + ((int64_t)((g << RB1) | c) << lo) + w;
        v[c] = CG ? __ldcg(src) : *src;
    }
#pragma unroll
    for (int s = 0; s < RB1; ++s)
#pragma unroll
        for (int c = 0; c < E; ++c)
            if (!(c & (1 << s))) bfly(v[c], v[c | (1 << s)]);
    if constexpr (RB2 > 0) {
        // exchange: element (b, w) at xs[pad32(b*W + w)]
#pragma unroll
        for (int c = 0; c < E; ++c) xs[pad32(((g << RB1) | c) * W + w)] = v[c];
        __syncthreads();
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
        __syncthreads();
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
    __syncthreads();
    const int64_t bmask = (int64_t{1} << HB) - 1;
    for (int q = tile.y + t; q < tile.z; q += kP2Threads) {
        const int2 rk = entries[q];
        const int64_t r = rk.x;
        const int b = (int)((r >> lo) & bmask);
        const int ww = (int)(r & (W - 1));
        SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(xs[pad32(b * W + ww)], s1), s2);
    }
}

// One CTA per (tile, column) of a phase-2 pass.
template <int HB>
__global__ void __launch_bounds__(kP2Threads)
srht_phase2_kernel(double* __restrict__ T, int64_t n_pad, int lo, const int4* __restrict__ tiles, int emit,
                   const int2* __restrict__ entries, double s1, double s2, double* __restrict__ SA, int64_t m) {
    extern __shared__ double xs[];
    constexpr int LOGW = P2Geom<HB>::LOGW;
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
    p2_tile<HB, false>(xs, T + j * n_pad + base, lo, emit != 0, tile, entries, j, s1, s2, SA, m);
}

// ------------------------------------------------------------ fused (one pass of high bits)
// Persistent work queue over column groups of G columns: items in the order
// P1(0), P1(1), P2(0), P1(2), P2(1), ..., P2(ng-1), handed out by an atomic
// counter to running CTAs only. P1(g) = phase-1 chunks of group g (8 per
// item, one per warp) into ring slot g % NSLOT of T; P2(g) = the emitting
// pass over the active tiles of group g. A P2(g) item waits until all P1(g)
// items are done; a P1(g) item waits until P2(g - NSLOT) released its slot.
// Every awaited item precedes the waiter in the hand-out order and is held
// by a running CTA, so the queue cannot deadlock. The ring (NSLOT x G
// columns of T) is sized to stay in L2, so T never round-trips through HBM.
struct FusedCtl {
    unsigned long long next;  // hand-out counter; followed by done1[ng], done2[ng] (int)
};

__device__ __forceinline__ void wait_count(const int* ctr, int target) {
    if (threadIdx.x == 0) {
        int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(128);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void signal_done(int* ctr) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(ctr, 1);
}

template <int HB>
__global__ void __launch_bounds__(kP2Threads)
srht_fused_kernel(const double* __restrict__ A, int64_t n, int64_t lda, const uint32_t* __restrict__ signbits,
                  double* __restrict__ T, int64_t n_pad, int64_t d, int G, int nslot, int ng, int n1, int n2,
                  int64_t cpc, const int4* __restrict__ tiles, int n_tiles, const int2* __restrict__ entries, int lo,
                  double s1, double s2, double* __restrict__ SA, int64_t m, unsigned long long* __restrict__ ctl) {
    static_assert(kP2Threads == 32 * kP1Warps, "one block shape for both item kinds");
    extern __shared__ double smem[];
    __shared__ long long item_s;
    int* done1 = reinterpret_cast<int*>(ctl + 1);
    int* done2 = done1 + ng;
    const long long per = (long long)n1 + n2;
    const long long total = (long long)ng * per;
    const int warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) item_s = (long long)atomicAdd(ctl, 1ULL);
        __syncthreads();
        const long long item = item_s;
        __syncthreads();
        if (item >= total) break;
        // decode the hand-out order P1(0), [P1(s), P2(s-1)] for s = 1..ng-1, P2(ng-1)
        bool p1;
        int g;
        long long w;
        if (item < n1) {
            p1 = true; g = 0; w = item;
        } else {
            const long long i2 = item - n1;
            const long long s = 1 + i2 / per;
            if (s < ng) {
                const long long within = i2 % per;
                p1 = within < n1;
                g = p1 ? (int)s : (int)s - 1;
                w = p1 ? within : within - n1;
            } else {
                p1 = false; g = ng - 1; w = i2 - (long long)(ng - 1) * per;
            }
        }
        const int slot = g % nslot;
        if (p1) {
            if (g >= nslot) wait_count(done2 + (g - nslot), n2);
            const int64_t c = w * kP1Warps + warp;  // chunk within the group
            const int64_t jj = c / cpc;
            const int64_t j = (int64_t)g * G + jj;
            if (jj < G && j < d) {
                const int64_t r0 = (c % cpc) << kChunkL;
                p1_chunk<true>(smem + warp * (1024 + 32), A + j * lda, n, signbits, r0,
                               T + ((int64_t)slot * G + jj) * n_pad + r0);
            }
            signal_done(done1 + g);
        } else {
            wait_count(done1 + g, n1);
            const int64_t jj = w / n_tiles;
            const int64_t j = (int64_t)g * G + jj;
            if (j < d) {
                const int4 tile = tiles[w % n_tiles];
                p2_tile<HB, true>(smem, T + ((int64_t)slot * G + jj) * n_pad + tile.x, lo, true, tile, entries, j, s1,
                                  s2, SA, m);
            }
            signal_done(done2 + g);
        }
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

int pass_w(int hb) {
    const int rb1 = std::min(hb, 5);
    return kP2Threads * (1 << rb1) / (1 << hb);
}
// elements of one phase-2 tile: W low indices x 2^hb pass combinations
// (kTileElems for hb >= 5, 256 * 2^hb below)
int64_t pass_tile_elems(int hb) { return (int64_t)pass_w(hb) << hb; }

template <int L>
void launch_small(const SrhtPlan& p, const double* A, const uint32_t* signbits, const int2* entries, double* SA,
                  cudaStream_t st) {
    constexpr int N = 1 << L;
    constexpr int THREADS = N / 16 > 0 ? N / 16 : 1;
    const size_t smem = (size_t)padded(N) * sizeof(double) + 64;
    LAUNCH(srht_small_kernel<L>, (unsigned)p.d, THREADS, smem, st, A, p.n, p.lda, signbits, entries, (int)p.m,
           p.scale1, p.scale2, SA, p.m);
}
using SmallFn = void (*)(const SrhtPlan&, const double*, const uint32_t*, const int2*, double*, cudaStream_t);
const SmallFn kSmall[kSmallL + 1] = {launch_small<0>, launch_small<1>, launch_small<2>, launch_small<3>,
                                     launch_small<4>, launch_small<5>, launch_small<6>, launch_small<7>,
                                     launch_small<8>, launch_small<9>, launch_small<10>};

template <int HB>
void launch_pass(const SrhtPlan& p, double* T, int lo, const int4* tiles, int n_tiles, bool emit, const int2* entries,
                 double* SA, cudaStream_t st) {
    const size_t smem = (size_t)pad32(kTileElems) * sizeof(double) + 64;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(srht_phase2_kernel<HB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
        attr = true;
    }
    const int64_t tiles_per_col = p.n_pad / pass_tile_elems(HB);
    const unsigned gx = emit ? (unsigned)n_tiles : (unsigned)tiles_per_col;
    if (gx == 0) return;
    dim3 grid(gx, (unsigned)p.d);
    LAUNCH(srht_phase2_kernel<HB>, grid, kP2Threads, smem, st, T, p.n_pad, lo, tiles, emit ? 1 : 0, entries,
           p.scale1, p.scale2, SA, p.m);
}

constexpr size_t kP1Smem = (size_t)kP1Warps * (1024 + 32) * sizeof(double);
constexpr size_t kP2Smem = (size_t)(kTileElems + kTileElems / 32) * sizeof(double) + 64;
constexpr size_t kFusedSmem = kP1Smem > kP2Smem ? kP1Smem : kP2Smem;  // covers both item kinds

template <int HB>
void launch_fused(const SrhtPlan& p, const double* A, const uint32_t* signbits, double* T, int G, int nslot,
                  const int4* tiles, int n_tiles, const int2* entries, double* SA, unsigned long long* ctl,
                  int num_sms, cudaStream_t st) {
    static int max_blocks_per_sm = 0;
    if (!max_blocks_per_sm) {
        CUDA_CHECK(cudaFuncSetAttribute(srht_fused_kernel<HB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kFusedSmem));
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, srht_fused_kernel<HB>, kP2Threads,
                                                                 kFusedSmem));
        if (max_blocks_per_sm < 1) max_blocks_per_sm = 1;
    }
    const int64_t cpc = p.n_pad >> kChunkL;
    const int ng = (int)ceil_div(p.d, G);
    const int n1 = (int)ceil_div((int64_t)G * cpc, kP1Warps);
    const int n2 = G * n_tiles;
    const int64_t total = (int64_t)ng * (n1 + n2);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, (int64_t)num_sms * max_blocks_per_sm));
    CUDA_CHECK(cudaMemsetAsync(ctl, 0, sizeof(unsigned long long) + 2 * sizeof(int) * (size_t)ng, st));
    LAUNCH(srht_fused_kernel<HB>, grid, kP2Threads, kFusedSmem, st, A, p.n, p.lda, signbits, T, p.n_pad, p.d, G, nslot,
           ng, n1, n2, cpc, tiles, n_tiles, entries, p.pass_lo[0], p.scale1, p.scale2, SA, p.m, ctl);
}
using FusedFn = void (*)(const SrhtPlan&, const double*, const uint32_t*, double*, int, int, const int4*, int,
                         const int2*, double*, unsigned long long*, int, cudaStream_t);
const FusedFn kFused[11] = {nullptr, launch_fused<1>, launch_fused<2>, launch_fused<3>, launch_fused<4>,
                            launch_fused<5>, launch_fused<6>, launch_fused<7>, launch_fused<8>, launch_fused<9>,
                            launch_fused<10>};
constexpr int kFusedSlots = 3;
constexpr int64_t kFusedRingBytes = 60ll << 20;  // T ring budget: well inside the 126 MB L2

int fused_group_cols(const SrhtPlan& p) {
    const int64_t per_col = p.n_pad * (int64_t)sizeof(double);
    return (int)std::max<int64_t>(1, std::min<int64_t>(p.d, kFusedRingBytes / (kFusedSlots * per_col)));
}
using PassFn = void (*)(const SrhtPlan&, double*, int, const int4*, int, bool, const int2*, double*, cudaStream_t);
const PassFn kPass[11] = {nullptr, launch_pass<1>, launch_pass<2>, launch_pass<3>, launch_pass<4>, launch_pass<5>,
                          launch_pass<6>, launch_pass<7>, launch_pass<8>, launch_pass<9>, launch_pass<10>};
}  // namespace

SrhtPlan srht_plan(int64_t n, int64_t d, int64_t lda, int64_t m) {
    SrhtPlan p{};
    p.n = n;
    p.d = d;
    p.lda = lda;
    p.m = m;
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
        case 1: LAUNCH(srht_combine_kernel<0>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 2: LAUNCH(srht_combine_kernel<1>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 4: LAUNCH(srht_combine_kernel<2>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 8: LAUNCH(srht_combine_kernel<3>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        case 16: LAUNCH(srht_combine_kernel<4>, blocks, 256, 0, st, d_U, m, d, d_hi, s1, s2, d_SA); break;
        default: fail(IHS_INVALID_INPUT, "srht shard: number of shards must be 1, 2, 4, 8 or 16");
    }
}

size_t srht_scratch_bytes(const SrhtPlan& p) { return p.H > 0 ? (size_t)p.n_pad * (size_t)p.d * sizeof(double) : 0; }

void srht_build_entries(const SrhtPlan& p, const int64_t* rows, std::vector<int2>& entries, std::vector<int4>& tiles) {
    entries.clear();
    tiles.clear();
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
    const int64_t W = pass_w(hb);
    const int64_t low_tiles = (int64_t{1} << lo) / W;
    const int64_t ntiles = p.n_pad / pass_tile_elems(hb);
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
}

size_t srht_fused_scratch_bytes(const SrhtPlan& p, size_t* ctl_bytes) {
    if (ctl_bytes) *ctl_bytes = sizeof(unsigned long long) + 2 * sizeof(int) * (size_t)(p.d + 1) + 64;
    if (p.H == 0 || p.npass != 1) return srht_scratch_bytes(p);
    return (size_t)kFusedSlots * fused_group_cols(p) * p.n_pad * sizeof(double);
}

bool srht_build_mask(const SrhtPlan& p, const std::vector<int4>& tiles, uint32_t mask[4]) {
    mask[0] = mask[1] = mask[2] = mask[3] = 0u;
    if (p.H == 0 || p.npass != 1) return false;
    int logw = 0;
    while ((1 << (logw + 1)) <= pass_w(p.pass_hb[0])) ++logw;
    for (const int4& t : tiles) {
        const int g = (t.x & ((1 << kChunkL) - 1)) >> logw;
        mask[g >> 5] |= 1u << (g & 31);
    }
    return true;
}

void srht_run_device(const SrhtPlan& p, const double* d_A, const uint32_t* d_signbits, const int2* d_entries,
                     const int4* d_tiles, int n_tiles, double* d_T, double* d_SA, cudaStream_t st,
                     unsigned long long* d_ctl, int num_sms, const uint32_t* d_mask) {
    if (p.d == 0) return;
    if (p.H == 0) {
        kSmall[p.L](p, d_A, d_signbits, d_entries, d_SA, st);
        return;
    }
    if (p.npass == 1 && n_tiles > 0 && d_ctl != nullptr) {
        // one launch, T kept in an L2-resident ring of column groups
        kFused[p.pass_hb[0]](p, d_A, d_signbits, d_T, fused_group_cols(p), kFusedSlots, d_tiles, n_tiles, d_entries,
                             d_SA, d_ctl, num_sms, st);
        return;
    }
    const int64_t chunks_per_col = p.n_pad >> kChunkL;
    const int64_t total = chunks_per_col * p.d;
    const int64_t blocks = std::min<int64_t>(ceil_div(total, kP1AWarps), (int64_t)num_sms);
    const size_t smem = (size_t)kP1AWarps * kP1Stages * kP1Buf * sizeof(double);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(srht_phase1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    // single pass: phase 1 writes only the groups the emitting pass reads
    const bool masked = p.npass == 1 && d_mask != nullptr;
    int logw = 0;
    if (masked)
        while ((1 << (logw + 1)) <= pass_w(p.pass_hb[0])) ++logw;
    LAUNCH(srht_phase1_kernel, (unsigned)blocks, 32 * kP1AWarps, smem, st, d_A, p.n, p.lda, d_signbits, d_T, p.n_pad,
           chunks_per_col, total, masked ? d_mask : nullptr, logw);
    for (int i = 0; i < p.npass; ++i) {
        const bool last = i == p.npass - 1;
        if (last && n_tiles == 0) break;
        kPass[p.pass_hb[i]](p, d_T, p.pass_lo[i], d_tiles, n_tiles, last, d_entries, d_SA, st);
    }
}

}  // namespace ihs_b200
