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

#include <cub/device/device_scan.cuh>

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

// Substream raw generator: CTA q starts from the 312-word window in
// starts[q] (state after q*stride draws), produces draws
// [q*stride, min((q+1)*stride, count)).
__global__ void __launch_bounds__(mt::THREADS) mt_substream_kernel(const uint64_t* __restrict__ starts, int64_t stride,
                                                                   int64_t count, uint64_t* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    const int64_t q = blockIdx.x;
    for (int i = threadIdx.x; i < NN; i += blockDim.x) buf[i] = starts[q * NN + i];
    __syncthreads();
    mt::Twister tw{buf, 0};
    const int k = threadIdx.x;
    const int64_t beg = q * stride;
    const int64_t end = min(count, beg + stride);
    for (int64_t base = beg; base < end; base += NN) {
        uint64_t lo, hi;
        tw.next(lo, hi);
        if (tw.worker()) {
            if (base + k < end) out[base + k] = temper(lo);
            if (base + mt::MM + k < end) out[base + mt::MM + k] = temper(hi);
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

// libstdc++ generate_canonical<double,53>(mt19937_64): one draw.
__device__ __forceinline__ double canonical(uint64_t raw) {
    double u = __dmul_rn(__ull2double_rn(raw), 0x1p-64);
    if (u >= 1.0) u = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
    return u;
}

// Polar attempt a consumes draws 2a, 2a+1 (random.tcc normal_distribution).
__device__ __forceinline__ bool polar_attempt(const uint64_t* raw, int64_t a, double& x, double& y, double& r2) {
    x = __dsub_rn(__dmul_rn(2.0, canonical(raw[2 * a])), 1.0);
    y = __dsub_rn(__dmul_rn(2.0, canonical(raw[2 * a + 1])), 1.0);
    r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return !(r2 > 1.0 || r2 == 0.0);
}

__global__ void polar_flags_kernel(const uint64_t* __restrict__ raw, int64_t attempts, int* __restrict__ flags) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < attempts; a += (int64_t)gridDim.x * blockDim.x) {
        double x, y, r2;
        flags[a] = polar_attempt(raw, a, x, y, r2) ? 1 : 0;
    }
}

// normals [first, first + count) of the stream -> out[0 .. count)
__global__ void polar_emit_kernel(const uint64_t* __restrict__ raw, int64_t attempts, const int* __restrict__ pos,
                                  int64_t first, int64_t count, double stddev, double* __restrict__ out,
                                  int64_t carry) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t end = first + count;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < attempts; a += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = carry + 2 * (int64_t)pos[a];  // normal index (carry: normals of earlier chunks)
        if (k >= end || k + 1 < first) continue;
        double x, y, r2;
        if (!polar_attempt(raw, a, x, y, r2)) continue;
        const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
        if (k >= first) out[k - first] = __dadd_rn(__dmul_rn(__dmul_rn(y, mult), stddev), 0.0);
        if (k + 1 >= first && k + 1 < end) out[k + 1 - first] = __dadd_rn(__dmul_rn(__dmul_rn(x, mult), stddev), 0.0);
    }
}

__global__ void last_total_kernel(const int* __restrict__ pos, const int* __restrict__ flags, int64_t attempts,
                                  long long* __restrict__ total) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    *total = (long long)pos[attempts - 1] + flags[attempts - 1];
}

// number of draws to generate so that `count` normals are almost surely covered
int64_t draws_for(int64_t count) {
    const double pairs = (double)((count + 1) / 2);
    const double attempts = pairs / 0.7853981633974483 * 1.002 + 6.0 * std::sqrt(pairs) + 64.0;
    int64_t a = (int64_t)attempts;
    return 2 * a;
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

size_t gaussian_scratch_bytes(int64_t count) {
    const int64_t draws = draws_for(count);
    const int64_t attempts = draws / 2;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, (int*)nullptr, (int*)nullptr, (int)attempts);
    const int64_t nsub = ceil_div(draws, kJumpStride);
    return (size_t)draws * 8 + (size_t)attempts * 8 + temp + 256 + (size_t)nsub * NN * 8 + (size_t)kJumpSeqWords * 8 + 1024;
}

void mt_fill_gaussian(uint64_t seed, int64_t first, int64_t count, double stddev, double* d_out, void* d_scratch,
                      cudaStream_t st) {
    if (count <= 0) return;
    const int64_t draws = draws_for(first + count);
    const int64_t attempts = draws / 2;
    if (attempts >= (int64_t)INT32_MAX) fail(IHS_INVALID_INPUT, "fill_gaussian: stream longer than 2^31 attempts");
    char* p = static_cast<char*>(d_scratch);
    uint64_t* raw = reinterpret_cast<uint64_t*>(p);
    p += (size_t)draws * 8;
    int* flags = reinterpret_cast<int*>(p);
    int* pos = flags + attempts;
    p += (size_t)attempts * 8;
    long long* total = reinterpret_cast<long long*>(p);
    p += 256;
    uint64_t* starts = reinterpret_cast<uint64_t*>(p);
    const int64_t nsub = ceil_div(draws, kJumpStride);
    p += (size_t)nsub * NN * 8;
    uint64_t* xseq = reinterpret_cast<uint64_t*>(p);
    p += (size_t)kJumpSeqWords * 8;
    void* temp = p;
    size_t temp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, flags, pos, (int)attempts);

    if (nsub <= 1) {
        mt_generate_raw(seed, draws, raw, st);
    } else {
        // jump-ahead start windows for substreams q*stride (host F2 polynomial
        // arithmetic, cached per stride), expanded on the device
        mt_jump_starts(seed, kJumpStride, nsub, starts, xseq, st);
        LAUNCH_PDL(mt_substream_kernel, (unsigned)nsub, 160, 0, st, starts, (int64_t)kJumpStride, draws, raw);
    }
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>(ceil_div(attempts, threads), 148 * 16);
    LAUNCH_PDL(polar_flags_kernel, blocks, threads, 0, st, raw, attempts, flags);
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flags, pos, (int)attempts, st));
    note_launch();
    LAUNCH_PDL(last_total_kernel, 1, 1, 0, st, pos, flags, attempts, total);
    long long h_total = 0;
    CUDA_CHECK(cudaMemcpyAsync(&h_total, total, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (2 * h_total < first + count) fail(IHS_INTERNAL_ERROR, "fill_gaussian: draw estimate too small");
    LAUNCH_PDL(polar_emit_kernel, blocks, threads, 0, st, raw, attempts, pos, first, count, stddev, d_out,
               (int64_t)0);
}

// ---- streamed normals (the Gaussian sketch of tall matrices, S never materialised)
namespace {
int64_t stream_subs() {  // substreams per chunk (IHS_GAUSS_STREAM_SUBS overrides; tests use 1)
    static const int64_t v = [] {
        const char* e = std::getenv("IHS_GAUSS_STREAM_SUBS");
        const long long x = e ? std::atoll(e) : 0;
        return x > 0 ? (int64_t)x : (int64_t)64;
    }();
    return v;
}
}  // namespace

int64_t gaussian_stream_chunk_attempts() { return stream_subs() * kStreamStride / 2; }

size_t gaussian_stream_scratch_bytes() {
    const int64_t draws = stream_subs() * kStreamStride, attempts = draws / 2;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, (int*)nullptr, (int*)nullptr, (int)attempts);
    return (size_t)draws * 8 + (size_t)attempts * 8 + temp + 256 + (size_t)stream_subs() * NN * 8 +
           (size_t)kJumpSeqWords * 8 + 1024;
}

void mt_gaussian_stream(uint64_t seed, int64_t first, int64_t count, double stddev, double* buf, int64_t cap,
                        int64_t block, void* d_scratch, cudaStream_t st,
                        const std::function<int64_t(int64_t, int64_t)>& consume) {
    if (count <= 0) return;
    const int64_t Q = stream_subs(), draws = Q * kStreamStride, attempts = draws / 2;
    char* p = static_cast<char*>(d_scratch);
    uint64_t* raw = reinterpret_cast<uint64_t*>(p);
    p += (size_t)draws * 8;
    int* flags = reinterpret_cast<int*>(p);
    int* pos = flags + attempts;
    p += (size_t)attempts * 8;
    long long* total = reinterpret_cast<long long*>(p);
    p += 256;
    uint64_t* starts = reinterpret_cast<uint64_t*>(p);
    p += (size_t)Q * NN * 8;
    uint64_t* xseq = reinterpret_cast<uint64_t*>(p);
    p += (size_t)kJumpSeqWords * 8;
    void* temp = p;
    size_t temp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, flags, pos, (int)attempts);
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>(ceil_div(attempts, threads), 148 * 16);
    const int64_t end = first + count;
    int64_t carry = 0;   // normals produced by the chunks so far
    int64_t base = first; // normal index held by buf[0]
    for (int64_t c = 0; carry < end; ++c) {
        // chunk c: substreams [c Q, (c + 1) Q) of kStreamStride draws, attempts from draw 2 c Q stride
        mt_jump_starts(seed, kStreamStride, Q, starts, xseq, st, c * Q);
        LAUNCH_PDL(mt_substream_kernel, (unsigned)Q, 160, 0, st, starts, (int64_t)kStreamStride, draws, raw);
        LAUNCH_PDL(polar_flags_kernel, blocks, threads, 0, st, raw, attempts, flags);
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flags, pos, (int)attempts, st));
        note_launch();
        LAUNCH_PDL(last_total_kernel, 1, 1, 0, st, pos, flags, attempts, total);
        long long h_total = 0;
        CUDA_CHECK(cudaMemcpyAsync(&h_total, total, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        const int64_t produced = 2 * (int64_t)h_total;
        if (carry + produced > first) {
            if (std::min(carry + produced, end) - base > cap) fail(IHS_INTERNAL_ERROR, "gaussian stream: buffer too small");
            // normals [max(carry, base), min(carry + produced, end)) -> buf[k - base]
            LAUNCH_PDL(polar_emit_kernel, blocks, threads, 0, st, raw, attempts, pos, base, end - base, stddev, buf,
                       carry);
        }
        carry += produced;
        const int64_t ready = std::min(carry, end) - base;
        if (ready >= block || carry >= end) {
            const int64_t used = consume(base, ready);
            const int64_t left = ready - used;
            if (left > used) fail(IHS_INTERNAL_ERROR, "gaussian stream: block smaller than two columns");
            if (left > 0)
                CUDA_CHECK(cudaMemcpyAsync(buf, buf + used, (size_t)left * sizeof(double), cudaMemcpyDeviceToDevice,
                                           st));
            base += used;
        }
    }
}

}  // namespace ihs_b200
