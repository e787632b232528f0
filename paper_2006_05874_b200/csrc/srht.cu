// srht.cu — SRHT sketch SA = sqrt(n_pad/m) * R * H * D * A on sm_100a.
//
// Reference: srht_sketch (sketch.hpp:77-108) with fwht_inplace
// (sketch.hpp:33-49). The reference materializes a zero-padded n_pad x d copy
// B, multiplies row i by eps_i, runs radix-2 butterflies per column for
// h = 1, 2, ..., n_pad/2 (bit 0 first), scales by 1/sqrt(n_pad), and gathers
// the m sampled rows scaled by sqrt(n_pad/m).
//
// B200 design (bit-exact with the reference):
//   * no padded copy: rows >= n are virtual zeros, the sign flip is fused
//     into the load (eps_i * a as a real multiply by +-1.0, like :91);
//   * n_pad = 2^(L+H). Phase 1 transforms each column in blocks of 2^L
//     contiguous rows entirely on chip (bits 0..L-1, in 4-bit register rounds
//     staged through padded shared memory), reading A exactly once;
//   * phase 2 (only if H > 0) runs bits L..L+H-1 for tiles of W consecutive
//     low indices across all 2^H blocks, and only for tiles that contain a
//     sampled row; it emits just the sampled rows;
//   * every butterfly is computed as in the reference (v[j] = s + t,
//     v[j+h] = s - t, stages in increasing bit order), and the two scalings
//     are separate rounded multiplies (:47-48 then :95-97), so SA matches the
//     reference bit for bit.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace ihs_b200 {

namespace {
constexpr int kMaxL = 13;   // phase-1 block = 2^13 doubles = 64 KiB (+ padding)
constexpr int kTileW = 16;  // phase-2 tile width (low indices), 128 B per block row

__host__ __device__ constexpr int padded(int i) { return i + (i >> 4); }

// Phase 1: one CTA per (row block, column). THREADS = max(1, 2^L / 16).
template <int L>
__global__ void __launch_bounds__((1 << L) / 16 > 0 ? (1 << L) / 16 : 1)
srht_phase1_kernel(const double* __restrict__ A, int64_t n, int64_t lda, const uint32_t* __restrict__ signbits,
                   int H, double* __restrict__ T, int64_t n_pad,
                   // H == 0 only: emit sampled rows directly
                   const int2* __restrict__ entries, int n_entries, double s1, double s2, double* __restrict__ SA,
                   int64_t m) {
    constexpr int N = 1 << L;
    constexpr int THREADS = N / 16 > 0 ? N / 16 : 1;
    constexpr int E = N / THREADS;  // elements per thread: 16, or N when N < 16
    extern __shared__ double xs[];

    const int64_t blk = blockIdx.x;
    const int64_t j = blockIdx.y;
    const int64_t r0 = blk * N;
    const double* Acol = A + j * lda;
    const int t = threadIdx.x;

    // coalesced load with the sign flip fused (B.row(i) = eps_i * A.row(i))
    for (int e = t; e < N; e += THREADS) {
        const int64_t r = r0 + e;
        double v = 0.0;
        if (r < n) {
            const uint32_t w = __ldg(signbits + (r >> 5));
            const double eps = ((w >> (r & 31)) & 1u) ? 1.0 : -1.0;
            v = __dmul_rn(eps, __ldg(Acol + r));
        }
        xs[padded(e)] = v;
    }
    __syncthreads();

    if constexpr (L < 4) {
        // tiny transform: one thread, all stages in registers
        double v[E];
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = xs[padded(c)];
#pragma unroll
        for (int s = 0; s < L; ++s) {
#pragma unroll
            for (int c = 0; c < E; ++c)
                if (!(c & (1 << s))) {
                    const double a = v[c], b = v[c | (1 << s)];
                    v[c] = __dadd_rn(a, b);
                    v[c | (1 << s)] = __dsub_rn(a, b);
                }
        }
#pragma unroll
        for (int c = 0; c < E; ++c) xs[padded(c)] = v[c];
        __syncthreads();
    } else {
        // rounds of 4 bits at positions b0 = 0, 4, 8, ... (last round shifted
        // down to L-4, applying only the stages not yet done)
        int done = 0;
        while (done < L) {
            const int b0 = (done + 4 <= L) ? done : L - 4;
            const int lo_stage = done - b0;  // first stage (within the round) still to apply
            const int low_mask = (1 << b0) - 1;
            const int base = ((t >> b0) << (b0 + 4)) | (t & low_mask);
            double v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = xs[padded(base | (c << b0))];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                if (s < lo_stage) continue;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    if (!(c & (1 << s))) {
                        const double a = v[c], b = v[c | (1 << s)];
                        v[c] = __dadd_rn(a, b);
                        v[c | (1 << s)] = __dsub_rn(a, b);
                    }
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < 16; ++c) xs[padded(base | (c << b0))] = v[c];
            __syncthreads();
            done = b0 + 4;
        }
    }

    if (H == 0) {
        // the column is complete: emit the sampled rows (all rows live in this block)
        for (int q = t; q < n_entries; q += THREADS) {
            const int2 rk = entries[q];
            const double v = xs[padded(rk.x)];
            SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(v, s1), s2);
        }
    } else {
        double* Tcol = T + j * n_pad + r0;
        for (int e = t; e < N; e += THREADS) Tcol[e] = xs[padded(e)];
    }
}

// Phase 2: one CTA per (active tile, column); bits L .. L+H-1 over the 2^H
// blocks for kTileW consecutive low indices, then emit the tile's samples.
__global__ void __launch_bounds__(256)
srht_phase2_kernel(const double* __restrict__ T, int64_t n_pad, int L, int H, const int4* __restrict__ tiles,
                   const int2* __restrict__ entries, double s1, double s2, double* __restrict__ SA, int64_t m) {
    extern __shared__ double xs[];
    const int4 tile = tiles[blockIdx.x];  // (rlo0, entry_begin, entry_end, -)
    const int64_t j = blockIdx.y;
    const int NB = 1 << H;
    const int64_t stride_b = int64_t{1} << L;
    const double* Tcol = T + j * n_pad + tile.x;
    const int total = NB * kTileW;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int b = e / kTileW, w = e % kTileW;
        xs[e] = Tcol[(int64_t)b * stride_b + w];
    }
    __syncthreads();
    const int half = total / 2;
    for (int s = 0; s < H; ++s) {
        for (int p = threadIdx.x; p < half; p += blockDim.x) {
            const int w = p % kTileW;
            const int bp = p / kTileW;  // index over b with bit s removed
            const int b_lo = bp & ((1 << s) - 1);
            const int b = ((bp >> s) << (s + 1)) | b_lo;
            const int i0 = b * kTileW + w, i1 = (b | (1 << s)) * kTileW + w;
            const double a = xs[i0], c = xs[i1];
            xs[i0] = __dadd_rn(a, c);
            xs[i1] = __dsub_rn(a, c);
        }
        __syncthreads();
    }
    for (int q = tile.y + threadIdx.x; q < tile.z; q += blockDim.x) {
        const int2 rk = entries[q];
        const int64_t r = rk.x;
        const int b = (int)(r >> L);
        const int w = (int)((r & (stride_b - 1)) - tile.x);
        const double v = xs[b * kTileW + w];
        SA[(int64_t)rk.y + j * m] = __dmul_rn(__dmul_rn(v, s1), s2);
    }
}

template <int L>
void launch_phase1(const SrhtPlan& p, const double* A, const uint32_t* signbits, double* T, const int2* entries,
                   int n_entries, double* SA, cudaStream_t st) {
    constexpr int N = 1 << L;
    constexpr int THREADS = N / 16 > 0 ? N / 16 : 1;
    const size_t smem = (size_t)padded(N) * sizeof(double) + 64;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(srht_phase1_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    dim3 grid((unsigned)(p.n_pad >> L), (unsigned)p.d);
    LAUNCH(srht_phase1_kernel<L>, grid, THREADS, smem, st, A, p.n, p.lda, signbits, p.H, T, p.n_pad, entries,
           n_entries, p.scale1, p.scale2, SA, p.m);
}

using Phase1Fn = void (*)(const SrhtPlan&, const double*, const uint32_t*, double*, const int2*, int, double*,
                          cudaStream_t);
const Phase1Fn kPhase1[kMaxL + 1] = {
    launch_phase1<0>, launch_phase1<1>, launch_phase1<2>,  launch_phase1<3>,  launch_phase1<4>,
    launch_phase1<5>, launch_phase1<6>, launch_phase1<7>,  launch_phase1<8>,  launch_phase1<9>,
    launch_phase1<10>, launch_phase1<11>, launch_phase1<12>, launch_phase1<13>};
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
    p.L = std::min(logn, kMaxL);
    p.H = logn - p.L;
    if (p.H > 12) fail(IHS_INVALID_INPUT, "srht_sketch: n_pad above 2^25 not supported");
    // exactly the reference's host expressions (sketch.hpp:47 and :95)
    p.scale1 = 1.0 / std::sqrt(static_cast<double>(np));
    p.scale2 = std::sqrt(static_cast<double>(np) / static_cast<double>(m));
    return p;
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
    // counting sort of the sampled rows by low-index tile
    const int64_t low = int64_t{1} << p.L;
    const int64_t ntiles = low / kTileW;
    std::vector<int> count((size_t)ntiles + 1, 0);
    for (int64_t k = 0; k < p.m; ++k) count[(size_t)((rows[k] & (low - 1)) / kTileW) + 1]++;
    for (int64_t t = 0; t < ntiles; ++t) count[(size_t)t + 1] += count[(size_t)t];
    entries.resize((size_t)p.m);
    std::vector<int> fill(count.begin(), count.end() - 1);
    for (int64_t k = 0; k < p.m; ++k) {
        const int64_t t = (rows[k] & (low - 1)) / kTileW;
        entries[(size_t)fill[(size_t)t]++] = make_int2((int)rows[k], (int)k);
    }
    for (int64_t t = 0; t < ntiles; ++t)
        if (count[(size_t)t + 1] > count[(size_t)t])
            tiles.push_back(make_int4((int)(t * kTileW), count[(size_t)t], count[(size_t)t + 1], 0));
}

void srht_run_device(const SrhtPlan& p, const double* d_A, const uint32_t* d_signbits, const int2* d_entries,
                     const int4* d_tiles, int n_tiles, double* d_T, double* d_SA, cudaStream_t st) {
    if (p.d == 0) return;
    kPhase1[p.L](p, d_A, d_signbits, d_T, d_entries, p.H == 0 ? (int)p.m : 0, d_SA, st);
    if (p.H > 0 && n_tiles > 0) {
        const size_t smem = (size_t)(kTileW << p.H) * sizeof(double);
        if (smem > 200 * 1024) fail(IHS_INVALID_INPUT, "srht_sketch: n_pad too large for one phase-2 tile");
        static size_t attr = 0;
        if (smem > attr) {
            CUDA_CHECK(cudaFuncSetAttribute(srht_phase2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = smem;
        }
        dim3 grid((unsigned)n_tiles, (unsigned)p.d);
        LAUNCH(srht_phase2_kernel, grid, 256, smem, st, d_T, p.n_pad, p.L, p.H, d_tiles, d_entries, p.scale1,
               p.scale2, d_SA, p.m);
    }
}

}  // namespace ihs_b200
