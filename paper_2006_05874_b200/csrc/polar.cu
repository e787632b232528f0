// polar.cu — the reference's Gaussian stream (fill_gaussian, rng.hpp:35-40) in two passes over substreams, with
// no raw-draw buffer, no library scan and (on one GPU, S materialised) no host round trip.
//
// libstdc++'s normal_distribution (polar method) turns attempt a = draws (2a, 2a+1) of mt19937_64 into two
// normals when it is accepted (y * mult first, the cached x * mult second), so the position of a normal depends
// on how many attempts before it were accepted. The draws are split into emitting substreams of `fine` draws:
//   count  (polar_count_kernel): one CTA per jump-ahead substream of `big` draws (start state by F2 jump-ahead,
//          mt_jump.cu; big = fine unless that would need more than ~32k jump polynomials) counts the accepted
//          attempts of each of its fine substreams, and can dump the 312-word MT state at each fine boundary;
//   scan   (count_scan_kernel): exclusive prefix over the fine substreams in one CTA -> first normal of each;
//   emit   (polar_emit_kernel): one CTA per fine substream regenerates it from its window and writes each
//          accepted attempt's pair (the rank inside a twist from warp ballots) — raw (y, x) for pairs inside the
//          requested window, finished on the spot at its two edges — keeping only [first, first + count);
//   finish (polar_finish_kernel): mult = sqrt(-2 log r2 / r2) for every interior pair, fully parallel (the log
//          is off the regeneration's serial critical path).
// Draws are regenerated rather than stored (a twist costs a few instructions per word; storing 16 bytes per
// attempt and reading them back costs more), and any substream range can be counted or emitted, which is what lets
// a row shard count only its 1/P share and emit only its own window (runtime.cpp).
#include "common.cuh"

#include "mt_core.cuh"
#include "mt_jump.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace ihs_b200 {

namespace {
using mt::MM;
using mt::NN;
using mt::temper;
constexpr int64_t kFine = kJumpStride;   // 2^18 draws per emitting substream
constexpr int64_t kMaxJumpSubs = 32768;  // jump polynomials kept per stride (about 650 MB of bit lists)

// libstdc++ generate_canonical<double,53>(mt19937_64): one draw, clamped below 1.
__device__ __forceinline__ double canonical(uint64_t raw) {
    double u = __dmul_rn(__ull2double_rn(raw), 0x1p-64);
    if (u >= 1.0) u = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
    return u;
}
__device__ __forceinline__ bool polar_accept(uint64_t d0, uint64_t d1, double& x, double& y, double& r2) {
    x = __dsub_rn(__dmul_rn(2.0, canonical(d0)), 1.0);
    y = __dsub_rn(__dmul_rn(2.0, canonical(d1)), 1.0);
    r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return !(r2 > 1.0 || r2 == 0.0);
}
__device__ __forceinline__ double polar_mult(double x, double y) {
    const double r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
}
__device__ __forceinline__ double polar_out(double v, double mult, double stddev) {
    return __dadd_rn(__dmul_rn(__dmul_rn(v, mult), stddev), 0.0);  // ret * stddev + mean, mean = 0
}

// Thread k (even, < 156) of a twist owns attempt pairs (base + k, base + k + 1) (lo words) and
// (base + 156 + k, base + 157 + k) (hi words); the odd neighbour's words arrive by one shuffle.
struct TwistPairs {
    uint64_t lo0, lo1, hi0, hi1;
    bool lo_ok, hi_ok;
};
__device__ __forceinline__ TwistPairs twist_pairs(mt::Twister& tw, int64_t base, int64_t end) {
    uint64_t lo = 0, hi = 0;
    tw.next(lo, hi);
    const int k = threadIdx.x;
    const uint64_t tlo = temper(lo), thi = temper(hi);
    TwistPairs p;
    p.lo0 = tlo;
    p.hi0 = thi;
    p.lo1 = __shfl_down_sync(0xffffffffu, tlo, 1);
    p.hi1 = __shfl_down_sync(0xffffffffu, thi, 1);
    const bool even_worker = k < MM && !(k & 1);
    p.lo_ok = even_worker && base + k + 1 < end;
    p.hi_ok = even_worker && base + MM + k + 1 < end;
    return p;
}

__device__ __forceinline__ int block_sum(int c, int* wsum) {
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    int s = 0;
#pragma unroll
    for (int w = 0; w < (int)(mt::THREADS / 32); ++w) s += wsum[w];
    __syncthreads();
    return s;
}

// CTA = jump substream bq0 + blockIdx.x of `big` draws: accepted-attempt counts of its fine substreams
// (cnt[fine index]); with fwin, also the 312-word window (the state words preceding the fine substream's first
// draw) of each of them at fwin[(fine index - fwin0) * 312].
__global__ void __launch_bounds__(mt::THREADS) polar_count_kernel(const uint64_t* __restrict__ jwin, int64_t big,
                                                                   int64_t fine, int64_t bq0, int64_t draws,
                                                                   int* __restrict__ cnt, uint64_t* __restrict__ fwin,
                                                                   int64_t fwin0) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    __shared__ int wsum[mt::THREADS / 32];
    const int64_t qr = blockIdx.x;
    for (int i = threadIdx.x; i < NN; i += blockDim.x) buf[i] = jwin[qr * NN + i];
    __syncthreads();
    const int64_t beg = (bq0 + qr) * big, end = min(draws, beg + big);
    const int64_t f_first = beg / fine;
    if (fwin)  // the first fine substream starts at the jump window itself
        for (int i = threadIdx.x; i < NN; i += blockDim.x) fwin[(f_first - fwin0) * NN + i] = buf[i];
    mt::Twister tw{buf, 0};
    int64_t seg_end = min(end, beg + fine);  // current fine substream [seg_end - fine, seg_end)
    int64_t f = f_first;
    int c_cur = 0, c_next = 0;
    for (int64_t base = beg; base < end; base += NN) {
        const TwistPairs p = twist_pairs(tw, base, end);
        double x, y, r2;
        // an attempt belongs to the fine substream of its first draw (fine boundaries are even)
        if (p.lo_ok && polar_accept(p.lo0, p.lo1, x, y, r2)) {
            if (base + threadIdx.x < seg_end) ++c_cur;
            else ++c_next;
        }
        if (p.hi_ok && polar_accept(p.hi0, p.hi1, x, y, r2)) {
            if (base + MM + threadIdx.x < seg_end) ++c_cur;
            else ++c_next;
        }
        if (base + NN >= seg_end) {  // the fine boundary seg_end falls in this block (uniform decision)
            const int s = block_sum(c_cur, wsum);
            if (threadIdx.x == 0) cnt[f] = s;
            c_cur = c_next;
            c_next = 0;
            if (fwin && seg_end < end) {
                // window of the next fine substream: state words [seg_end - 312, seg_end), spread over the
                // previous block [base - 312, base) and this one [base, base + 312)
                const uint64_t* cur = buf + tw.cur * NN;
                const uint64_t* prev = buf + (tw.cur ^ 1) * NN;
                for (int i = threadIdx.x; i < NN; i += blockDim.x) {
                    const int64_t j = seg_end - NN + i;
                    fwin[(f + 1 - fwin0) * NN + i] = j < base ? prev[j - (base - NN)] : cur[j - base];
                }
                __syncthreads();  // the next twist overwrites the previous block
            }
            ++f;
            seg_end = min(end, seg_end + fine);
        }
    }
}

// base[q] = sum of cnt[0..q), base[nsub] = total (one CTA of 1024 threads, contiguous segments per thread)
__global__ void __launch_bounds__(1024) count_scan_kernel(const int* __restrict__ cnt, int64_t nsub,
                                                          long long* __restrict__ base) {
    pdl_wait();
    __shared__ long long wpart[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t per = (nsub + 1023) / 1024;
    const int64_t b0 = min(nsub, (int64_t)t * per), b1 = min(nsub, b0 + per);
    long long s = 0;
    for (int64_t i = b0; i < b1; ++i) s += cnt[i];
    long long incl = s;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wpart[w] = incl;
    __syncthreads();
    if (w == 0) {
        long long v = wpart[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        wpart[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    long long run = (w > 0 ? wpart[w - 1] : 0) + incl - s;  // exclusive prefix of this thread's segment
    for (int64_t i = b0; i < b1; ++i) {
        base[i] = run;
        run += cnt[i];
    }
    if (t == 1023) base[nsub] = wpart[31];
}

// CTA = fine substream fq0 + blockIdx.x (window fwin[(f - fwin0) * 312]): normals of [first, first + count)
// -> out[k - first]. Pairs inside the window are written raw (y at k, x at k + 1; polar_finish_kernel applies
// the multiplier), the at most two pairs straddling an edge are finished here. A window not covered by the
// generated draws poisons its last entry with NaN (no CTA writes it, so the sketch fails the finite check of
// SketchedSystem::factorize instead of going on silently).
__global__ void __launch_bounds__(mt::THREADS) polar_emit_kernel(const uint64_t* __restrict__ fwin, int64_t fwin0,
                                                                  int64_t fine, int64_t fq0, int64_t draws,
                                                                  const long long* __restrict__ base, int64_t nsub,
                                                                  int64_t first, int64_t count, double stddev,
                                                                  double* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    __shared__ int wl[2][mt::THREADS / 32], wh[2][mt::THREADS / 32];
    const int64_t f = fq0 + blockIdx.x;
    const int64_t end_n = first + count;
    if (f == nsub - 1 && threadIdx.x == 0 && 2 * base[nsub] < end_n)
        out[count - 1] = __longlong_as_double(0x7ff8000000000000LL);
    const int64_t n_beg = 2 * base[f], n_end = 2 * base[f + 1];
    if (n_end <= first || n_beg >= end_n) return;  // no normal of this substream lies in the window
    for (int i = threadIdx.x; i < NN; i += blockDim.x) buf[i] = fwin[(f - fwin0) * NN + i];
    __syncthreads();
    mt::Twister tw{buf, 0};
    const int64_t beg = f * fine, end = min(draws, beg + fine);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int64_t running = n_beg;  // normal index of the next accepted attempt's first normal
    int par = 0;
    auto put = [&](int64_t k, double x, double y) {
        if (k + 1 < first || k >= end_n) return;
        if (k >= first && k + 1 < end_n) {  // interior pair: raw values, finished in bulk
            out[k - first] = y;
            out[k + 1 - first] = x;
            return;
        }
        const double mult = polar_mult(x, y);  // an edge pair: one of its two normals is in the window
        if (k >= first) out[k - first] = polar_out(y, mult, stddev);
        else out[k + 1 - first] = polar_out(x, mult, stddev);
    };
    for (int64_t b = beg; b < end && running < end_n; b += NN) {
        const TwistPairs p = twist_pairs(tw, b, end);
        double xl = 0, yl = 0, rl = 0, xh = 0, yh = 0, rh = 0;
        const bool al = p.lo_ok && polar_accept(p.lo0, p.lo1, xl, yl, rl);
        const bool ah = p.hi_ok && polar_accept(p.hi0, p.hi1, xh, yh, rh);
        const unsigned bl = __ballot_sync(0xffffffffu, al), bh = __ballot_sync(0xffffffffu, ah);
        if (lane == 0) {
            wl[par][w] = __popc(bl);
            wh[par][w] = __popc(bh);
        }
        __syncthreads();
        int before_l = 0, tot_l = 0, before_h = 0, tot_h = 0;
#pragma unroll
        for (int v = 0; v < (int)(mt::THREADS / 32); ++v) {
            before_l += v < w ? wl[par][v] : 0;
            tot_l += wl[par][v];
            before_h += v < w ? wh[par][v] : 0;
            tot_h += wh[par][v];
        }
        // lo attempts precede hi attempts in the draw order
        if (al) put(running + 2 * (int64_t)(before_l + __popc(bl & lt)), xl, yl);
        if (ah) put(running + 2 * (int64_t)(tot_l + before_h + __popc(bh & lt)), xh, yh);
        running += 2 * (int64_t)(tot_l + tot_h);
        par ^= 1;  // the next twist writes the other slot (its barrier orders the reuse)
    }
}

// interior pairs of the window (stream index k even, k >= first, k + 1 < first + count): (y, x) -> normals
__global__ void polar_finish_kernel(double* __restrict__ out, int64_t first, int64_t count, double stddev) {
    pdl_wait();
    const int64_t k0 = first + (first & 1);  // first even stream index in the window
    const int64_t npairs = (first + count - k0) / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs; i += (int64_t)gridDim.x * blockDim.x) {
        double* o = out + (k0 - first) + 2 * i;
        const double y = o[0], x = o[1];
        const double mult = polar_mult(x, y);
        o[0] = polar_out(y, mult, stddev);
        o[1] = polar_out(x, mult, stddev);
    }
}

__global__ void counts_to_double_kernel(const int* __restrict__ cnt, int64_t f0, int64_t nf, int64_t len,
                                        double* __restrict__ out) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = i < nf ? (double)cnt[f0 + i] : 0.0;
}
__global__ void counts_from_double_kernel(const double* __restrict__ in, int64_t nsub, int* __restrict__ cnt) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsub; i += (int64_t)gridDim.x * blockDim.x)
        cnt[i] = (int)in[i];
}

// number of draws to generate so that `count` normals are almost surely covered (+6 sigma)
int64_t polar_draws_for(int64_t count) {
    const double pairs = (double)((count + 1) / 2);
    const double attempts = pairs / 0.7853981633974483 * 1.002 + 6.0 * std::sqrt(pairs) + 64.0;
    return 2 * (int64_t)attempts;
}
unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }
}  // namespace

GaussPlan gauss_plan(int64_t total_normals) {
    static const int64_t max_jump = [] {  // IHS_GAUSS_MAX_JUMP_SUBS: tests force big > fine on small streams
        const char* e = std::getenv("IHS_GAUSS_MAX_JUMP_SUBS");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? (int64_t)v : kMaxJumpSubs;
    }();
    static const int fine_log2 = [] {  // IHS_GAUSS_FINE_LOG2: emitting-substream length (A/B)
        const char* e = std::getenv("IHS_GAUSS_FINE_LOG2");
        return e ? std::atoi(e) : 0;
    }();
    GaussPlan g{};
    g.draws = polar_draws_for(total_normals);
    // shorter emitting substreams for short streams: the per-CTA regeneration is latency-bound, so more CTAs
    // win until the jump-ahead (linear in the substream count) dominates (C2: 2^17 -> ~1300 CTAs)
    g.fine = fine_log2 >= 12 && fine_log2 <= 24 ? int64_t{1} << fine_log2
                                                : (g.draws < (int64_t{1} << 31) ? kFine / 2 : kFine);
    g.nsub = ceil_div(g.draws, g.fine);
    g.big = g.fine;
    while (ceil_div(g.draws, g.big) > max_jump) g.big *= 2;
    g.nbig = ceil_div(g.draws, g.big);
    return g;
}

size_t gauss_scratch_bytes(const GaussPlan& g, int64_t nbig_win, int64_t nfine_win) {
    const int64_t fw = g.big == g.fine ? 0 : nfine_win;
    return (size_t)(nbig_win + fw) * NN * 8 + (size_t)kJumpSeqWords * 8 + (size_t)g.nsub * 4 +
           (size_t)(g.nsub + 1) * 8 + 1024;
}

GaussScratch gauss_scratch(const GaussPlan& g, int64_t nbig_win, int64_t nfine_win, void* d_scratch) {
    GaussScratch s{};
    char* p = static_cast<char*>(d_scratch);
    s.jwin = reinterpret_cast<uint64_t*>(p);
    p += (size_t)nbig_win * NN * 8;
    s.fwin = g.big == g.fine ? s.jwin : reinterpret_cast<uint64_t*>(p);  // fine = jump substreams: one set
    if (g.big != g.fine) p += (size_t)nfine_win * NN * 8;
    s.xseq = reinterpret_cast<uint64_t*>(p);
    p += (size_t)kJumpSeqWords * 8;
    s.base = reinterpret_cast<long long*>(p);
    p += (size_t)(g.nsub + 1) * 8;
    s.cnt = reinterpret_cast<int*>(p);
    return s;
}

void gauss_jump(uint64_t seed, const GaussPlan& g, int64_t bq0, int64_t bnq, GaussScratch& s, cudaStream_t st) {
    s.j0 = bq0;
    if (g.big == g.fine) s.f0 = bq0;  // the jump windows are the fine windows
    if (bnq > 0) mt_jump_starts(seed, g.big, bnq, s.jwin, s.xseq, st, bq0);
}

void gauss_count(const GaussPlan& g, int64_t bq0, int64_t bnq, GaussScratch& s, bool dump, cudaStream_t st) {
    if (bnq <= 0) return;
    uint64_t* fwin = nullptr;
    if (dump && g.big != g.fine) {
        fwin = s.fwin;
        s.f0 = bq0 * (g.big / g.fine);
    }
    LAUNCH_PDL(polar_count_kernel, (unsigned)bnq, mt::THREADS, 0, st, (const uint64_t*)(s.jwin + (bq0 - s.j0) * NN),
               g.big, g.fine, bq0, g.draws, s.cnt, fwin, s.f0);
}

void gauss_scan(const GaussPlan& g, const GaussScratch& s, cudaStream_t st) {
    LAUNCH_PDL(count_scan_kernel, 1, 1024, 0, st, (const int*)s.cnt, g.nsub, s.base);
}

void gauss_fine_windows(uint64_t seed, const GaussPlan& g, int64_t fq0, int64_t fnq, GaussScratch& s,
                        cudaStream_t st) {
    if (fnq <= 0) return;
    const int64_t ratio = g.big / g.fine;
    const int64_t bq0 = fq0 / ratio, bq1 = ceil_div(fq0 + fnq, ratio);
    gauss_jump(seed, g, bq0, bq1 - bq0, s, st);
    if (g.big != g.fine) gauss_count(g, bq0, bq1 - bq0, s, true, st);  // dump pass (recounts identical values)
}

void gauss_emit(const GaussPlan& g, int64_t fq0, int64_t fnq, const GaussScratch& s, int64_t first, int64_t count,
                double stddev, double* d_out, cudaStream_t st) {
    if (fnq <= 0 || count <= 0) return;
    LAUNCH_PDL(polar_emit_kernel, (unsigned)fnq, mt::THREADS, 0, st, (const uint64_t*)s.fwin, s.f0, g.fine, fq0,
               g.draws, (const long long*)s.base, g.nsub, first, count, stddev, d_out);
    LAUNCH_PDL(polar_finish_kernel, grid_for(count / 2 + 1), 256, 0, st, d_out, first, count, stddev);
}

void gauss_counts_to_double(const GaussScratch& s, int64_t f0, int64_t nf, int64_t len, double* d_out, cudaStream_t st) {
    LAUNCH_PDL(counts_to_double_kernel, grid_for(len), 256, 0, st, (const int*)s.cnt, f0, nf, len, d_out);
}
void gauss_counts_from_double(const double* d_in, const GaussPlan& g, const GaussScratch& s, cudaStream_t st) {
    LAUNCH_PDL(counts_from_double_kernel, grid_for(g.nsub), 256, 0, st, d_in, g.nsub, s.cnt);
}

// Fine substreams whose normals intersect [first, first + count), from the host copy of base (nsub + 1 entries).
void gauss_window_range(const std::vector<long long>& h_base, int64_t first, int64_t count, int64_t* q0,
                        int64_t* nq) {
    const int64_t nsub = (int64_t)h_base.size() - 1;
    // first q with 2 base[q + 1] > first, then the first q with 2 base[q] >= first + count
    int64_t lo = 0, hi = nsub;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (2 * h_base[(size_t)mid + 1] > first) hi = mid;
        else lo = mid + 1;
    }
    const int64_t a = lo;
    lo = a, hi = nsub;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (2 * h_base[(size_t)mid] < first + count) lo = mid + 1;
        else hi = mid;
    }
    *q0 = a;
    *nq = std::max<int64_t>(0, lo - a);
}

}  // namespace ihs_b200
