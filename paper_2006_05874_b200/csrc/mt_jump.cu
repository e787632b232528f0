// mt_jump.cu — F2-linear jump-ahead for std::mt19937_64 (rng.hpp:30-32).
//
// The MT19937-64 state transition T is linear over GF(2) on its 19937-bit
// effective state. With P(x) its characteristic polynomial and
// x^J mod P(x) = sum_i a_i x^i, the state after J draws is
// W_J = sum_i a_i W_i, where W_i is the 312-word sliding window
// (x_i, ..., x_{i+311}) of the untempered word sequence (x_0..x_311 is the
// seeded array, x_{312+j} the word tempered into draw j). The window's
// oldest word contributes only its top bit, so the 31 "junk" bits of the
// XOR-combination never reach an output.
//
// Host: P(x) by Berlekamp-Massey on 40000 output bits (once per process);
// the jump polynomials x^(q*stride) mod P are seed-independent and cached.
// Device: one CTA per substream XOR-accumulates the windows selected by its
// polynomial from the first 20248 words of the seeded stream (in smem).
#include "common.cuh"
#include "mt_core.cuh"
#include "mt_jump.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <thread>

namespace ihs_b200 {

namespace {
constexpr int NN = 312;
constexpr int DEG = 19937;          // degree of the characteristic polynomial
constexpr int PW = 312;             // words per reduced polynomial (19968 bits)
constexpr int NX = DEG + NN - 1;    // words of the untempered sequence the windows need

using Poly = std::vector<uint64_t>;

inline bool getbit(const uint64_t* v, int64_t i) { return (v[i >> 6] >> (i & 63)) & 1ULL; }
inline void flipbit(uint64_t* v, int64_t i) { v[i >> 6] ^= 1ULL << (i & 63); }

// v ^= (src << shift), src has n words; dst must have room for n+1+shift/64 words
inline void xor_shifted(uint64_t* dst, const uint64_t* src, int n, int64_t shift) {
    const int64_t ws = shift >> 6;
    const int bs = (int)(shift & 63);
    if (bs == 0) {
        for (int i = 0; i < n; ++i) dst[ws + i] ^= src[i];
    } else {
        uint64_t carry = 0;
        for (int i = 0; i < n; ++i) {
            dst[ws + i] ^= (src[i] << bs) | carry;
            carry = src[i] >> (64 - bs);
        }
        dst[ws + n] ^= carry;
    }
}

Poly berlekamp_massey_charpoly() {
    // sequence: low bit of successive draws of a default-seeded generator
    const int N = 2 * DEG + 128;
    std::mt19937_64 gen(5489u);
    const int NW = (N + 63) / 64 + 2;
    std::vector<uint64_t> rs(NW, 0);  // reversed sequence: rs bit k = s_{N-1-k}
    {
        std::vector<uint8_t> s(N);
        for (int i = 0; i < N; ++i) s[i] = (uint8_t)(gen() & 1ULL);
        for (int k = 0; k < N; ++k)
            if (s[N - 1 - k]) rs[k >> 6] |= 1ULL << (k & 63);
    }
    const int CW = (DEG + 64) / 64 + 4;
    std::vector<uint64_t> Cp(CW + 8, 0), Bp(CW + 8, 0), Tp(CW + 8, 0);
    Cp[0] = Bp[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < N; ++n) {
        // d = sum_{i=0..L} C_i s_{n-i} = sum_i C_i rs[N-1-n+i]
        const int64_t o = (int64_t)N - 1 - n;
        const int64_t ow = o >> 6;
        const int ob = (int)(o & 63);
        uint64_t acc = 0;
        const int words = L / 64 + 1;
        for (int w = 0; w < words; ++w) {
            uint64_t lo = rs[ow + w];
            uint64_t hi = (ow + w + 1 < NW) ? rs[ow + w + 1] : 0;
            uint64_t seg = ob ? ((lo >> ob) | (hi << (64 - ob))) : lo;
            acc ^= Cp[w] & seg;
        }
        // mask off coefficients above L in the last word
        const int lastbits = (L % 64) + 1;
        if (lastbits < 64) {
            const int w = L / 64;
            uint64_t lo = rs[ow + w];
            uint64_t hi = (ow + w + 1 < NW) ? rs[ow + w + 1] : 0;
            uint64_t seg = ob ? ((lo >> ob) | (hi << (64 - ob))) : lo;
            const uint64_t over = Cp[w] & seg & ~((1ULL << lastbits) - 1ULL);
            acc ^= over;
        }
        const int dbit = __builtin_parityll(acc);
        if (!dbit) {
            ++m;
        } else if (2 * L <= n) {
            Tp = Cp;
            xor_shifted(Cp.data(), Bp.data(), CW - (m >> 6) - 2 > 0 ? CW - (int)(m >> 6) - 2 : 0, m);
            L = n + 1 - L;
            Bp = Tp;
            m = 1;
        } else {
            xor_shifted(Cp.data(), Bp.data(), CW - (m >> 6) - 2 > 0 ? CW - (int)(m >> 6) - 2 : 0, m);
            ++m;
        }
    }
    if (L != DEG) fail(IHS_INTERNAL_ERROR, "mt19937_64 jump: Berlekamp-Massey found degree " + std::to_string(L));
    // P(x) = x^L C(1/x): P_j = C_{L-j}
    Poly P(PW + 1, 0);
    for (int j = 0; j <= L; ++j)
        if (getbit(Cp.data(), L - j)) flipbit(P.data(), j);
    return P;
}

struct PolyRing {
    Poly P;                              // degree DEG, PW+1 words
    std::vector<Poly> Pshift;            // P << s, s = 0..63 (PW+2 words)
    PolyRing() : P(berlekamp_massey_charpoly()) {
        Pshift.assign(64, Poly(PW + 3, 0));
        for (int s = 0; s < 64; ++s) xor_shifted(Pshift[s].data(), P.data(), PW + 1, s);
    }
    // r (2*PW+2 words, degree < 2*DEG) -> r mod P in place (low PW words valid)
    void reduce(uint64_t* r) const {
        for (int64_t i = 2 * (int64_t)DEG; i >= DEG; --i) {
            if (!getbit(r, i)) continue;
            const int64_t sh = i - DEG;
            const Poly& ps = Pshift[sh & 63];
            const int64_t ws = sh >> 6;
            for (int w = 0; w < PW + 2; ++w) r[ws + w] ^= ps[w];
        }
    }
    Poly mulmod(const Poly& a, const Poly& b) const {
        std::vector<Poly> bs(64, Poly(PW + 2, 0));
        for (int s = 0; s < 64; ++s) xor_shifted(bs[s].data(), b.data(), PW, s);
        std::vector<uint64_t> r(2 * PW + 8, 0);
        for (int wa = 0; wa < PW; ++wa) {
            uint64_t w = a[wa];
            while (w) {
                const int s = __builtin_ctzll(w);
                w &= w - 1;
                const uint64_t* src = bs[s].data();
                uint64_t* dst = r.data() + wa;
                for (int k = 0; k < PW + 1; ++k) dst[k] ^= src[k];
            }
        }
        reduce(r.data());
        return Poly(r.begin(), r.begin() + PW);
    }
    Poly sqrmod(const Poly& a) const {
        std::vector<uint64_t> r(2 * PW + 8, 0);
        for (int64_t i = 0; i < (int64_t)PW * 64; ++i)
            if (getbit(a.data(), i)) flipbit(r.data(), 2 * i);
        reduce(r.data());
        return Poly(r.begin(), r.begin() + PW);
    }
    Poly powmod_x(uint64_t e) const {  // x^e mod P
        Poly result(PW, 0);
        result[0] = 1;
        Poly base(PW, 0);
        base[0] = 2;  // x
        while (e) {
            if (e & 1) result = mulmod(result, base);
            e >>= 1;
            if (e) base = sqrmod(base);
        }
        return result;
    }
    Poly powmod(const Poly& b, uint64_t e) const {
        Poly result(PW, 0);
        result[0] = 1;
        Poly base = b;
        while (e) {
            if (e & 1) result = mulmod(result, base);
            e >>= 1;
            if (e) base = sqrmod(base);
        }
        return result;
    }
};

std::mutex g_mu;
PolyRing* g_ring = nullptr;
std::map<int64_t, std::vector<uint64_t>> g_polys;  // stride -> packed polys

PolyRing& ring() {
    if (!g_ring) g_ring = new PolyRing();
    return *g_ring;
}

// untempered word sequence x_0 .. x_{nx-1} of mt19937_64(seed)
__global__ void __launch_bounds__(mt::THREADS) mt_wordseq_kernel(uint64_t seed, int nx, uint64_t* __restrict__ X) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t buf[2 * NN];
    mt::seed_array(buf, seed);
    __syncthreads();
    for (int i = threadIdx.x; i < NN; i += blockDim.x) X[i] = buf[i];
    mt::Twister tw{buf, 0};
    const int k = threadIdx.x;
    for (int base = NN; base < nx; base += NN) {
        uint64_t lo, hi;
        tw.next(lo, hi);
        if (tw.worker()) {
            if (base + k < nx) X[base + k] = lo;
            if (base + mt::MM + k < nx) X[base + mt::MM + k] = hi;
        }
    }
}

// CTA (q, chunk) XORs the windows W_i (i = set coefficient positions of
// substream q's polynomial inside position range chunk*kSpan ..) into the
// start state. Positions come as host-built sorted lists; each warp takes
// every 8th position and XORs the 312-word window with 10 words per lane.
// Partial states combine with atomicXor (XOR is associative and commutative,
// so the start state is exact regardless of order); starts is pre-zeroed.
constexpr int kChunks = 8;
constexpr int kSpan = (DEG + kChunks - 1) / kChunks;  // 2493 coefficient positions per chunk
constexpr int kApplyThreads = 256;
__global__ void __launch_bounds__(kApplyThreads) mt_jump_apply_kernel(const uint64_t* __restrict__ X,
                                                                      const uint16_t* __restrict__ pos,
                                                                      const int* __restrict__ ptr,
                                                                      uint64_t* __restrict__ starts) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ uint64_t xs[kSpan + NN];
    __shared__ unsigned long long red[NN];
    const int q = blockIdx.x, chunk = blockIdx.y;
    const int b0 = ptr[q * (kChunks + 1) + chunk], b1 = ptr[q * (kChunks + 1) + chunk + 1];
    if (b0 >= b1) return;  // uniform
    const int base = chunk * kSpan;
    const int nload = min(NX - base, kSpan + NN);
    for (int i = threadIdx.x; i < nload; i += blockDim.x) xs[i] = X[base + i];
    for (int i = threadIdx.x; i < NN; i += blockDim.x) red[i] = 0ULL;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = kApplyThreads / 32;
    uint64_t acc[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) acc[k] = 0;
    for (int b = b0 + warp; b < b1; b += NW) {
        const int i = (int)pos[b] - base;
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (lane + 32 * k < NN) acc[k] ^= xs[i + lane + 32 * k];
    }
#pragma unroll
    for (int k = 0; k < 10; ++k)
        if (lane + 32 * k < NN) atomicXor(&red[lane + 32 * k], (unsigned long long)acc[k]);
    __syncthreads();
    for (int w = threadIdx.x; w < NN; w += blockDim.x)
        atomicXor(reinterpret_cast<unsigned long long*>(starts + (size_t)q * NN + w), red[w]);
}
}  // namespace

const std::vector<uint64_t>& mt_charpoly() {
    std::lock_guard<std::mutex> lk(g_mu);
    return ring().P;
}

const std::vector<uint64_t>& mt_jump_polys(int64_t stride, int64_t nsub) {
    std::lock_guard<std::mutex> lk(g_mu);
    PolyRing& R = ring();
    auto& vec = g_polys[stride];
    const int64_t have = (int64_t)(vec.size() / PW);
    if (have >= nsub) return vec;
    const Poly base = R.powmod_x((uint64_t)stride);
    vec.resize((size_t)nsub * PW);
    // chains of consecutive q computed in parallel threads
    const int64_t todo = nsub - have;
    const int nthreads = (int)std::max<int64_t>(1, std::min<int64_t>(todo, std::max(1u, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
        const int64_t q0 = have + todo * t / nthreads;
        const int64_t q1 = have + todo * (t + 1) / nthreads;
        if (q0 >= q1) continue;
        th.emplace_back([&, q0, q1] {
            Poly cur = R.powmod(base, (uint64_t)q0);
            for (int64_t q = q0; q < q1; ++q) {
                std::memcpy(vec.data() + (size_t)q * PW, cur.data(), PW * 8);
                if (q + 1 < q1) cur = R.mulmod(cur, base);
            }
        });
    }
    for (auto& t : th) t.join();
    return vec;
}

void mt_jump_starts(uint64_t seed, int64_t stride, int64_t nsub, uint64_t* d_starts, uint64_t* d_X, cudaStream_t st,
                    int64_t q0) {
    const int64_t qend = q0 + nsub;  // substreams [q0, qend)
    // device copies of the set-bit lists of x^(q*stride) mod P, cached per
    // (device, stride) and grown on demand (seed-independent)
    struct DevLists {
        uint16_t* pos = nullptr;
        int* ptr = nullptr;
        int64_t count = 0;
    };
    static std::mutex mu;
    static std::map<std::pair<int, int64_t>, DevLists> dev;
    int dev_id = 0;
    CUDA_CHECK(cudaGetDevice(&dev_id));
    DevLists L;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto key = std::make_pair(dev_id, stride);
        auto it = dev.find(key);
        if (it == dev.end() || it->second.count < qend) {
            const int64_t nall = qend;
            const std::vector<uint64_t>& polys = mt_jump_polys(stride, nall);
            std::vector<uint16_t> pos;
            std::vector<int> ptr((size_t)nall * (kChunks + 1));
            pos.reserve((size_t)nall * DEG / 2 + 64);
            for (int64_t q = 0; q < nall; ++q) {
                const uint64_t* a = polys.data() + (size_t)q * PW;
                for (int c = 0; c < kChunks; ++c) {
                    ptr[(size_t)q * (kChunks + 1) + c] = (int)pos.size();
                    const int i1 = std::min(DEG, (c + 1) * kSpan);
                    for (int i = c * kSpan; i < i1; ++i)
                        if ((a[i >> 6] >> (i & 63)) & 1ULL) pos.push_back((uint16_t)i);
                }
                ptr[(size_t)q * (kChunks + 1) + kChunks] = (int)pos.size();
            }
            if (it != dev.end()) {
                CUDA_CHECK(cudaFree(it->second.pos));
                CUDA_CHECK(cudaFree(it->second.ptr));
            }
            CUDA_CHECK(cudaMalloc(&L.pos, pos.size() * sizeof(uint16_t) + 16));
            CUDA_CHECK(cudaMalloc(&L.ptr, ptr.size() * sizeof(int)));
            CUDA_CHECK(cudaMemcpy(L.pos, pos.data(), pos.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
            CUDA_CHECK(cudaMemcpy(L.ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice));
            L.count = nall;
            dev[key] = L;
        } else {
            L = it->second;
        }
    }
    CUDA_CHECK(cudaMemsetAsync(d_starts, 0, (size_t)nsub * NN * 8, st));
    LAUNCH_PDL(mt_wordseq_kernel, 1, mt::THREADS, 0, st, seed, NX, d_X);
    LAUNCH_PDL(mt_jump_apply_kernel, dim3((unsigned)nsub, kChunks), kApplyThreads, 0, st, d_X, L.pos,
               L.ptr + q0 * (kChunks + 1), d_starts);
}

}  // namespace ihs_b200
