// gradient.cu — fused g = A^T (A x - b) + nu^2 x for one or two iterates.
//
// Reference: gradient (problem.hpp:59-69) evaluates two Eigen GEMVs, reading
// A twice per call, and the adaptive loop calls it once per candidate
// (solver.hpp:162, candidates at :182 and :190).
//
// B200 design: persistent CTAs walk 32-row panels of column-major A.
//   sweep 1: warps stride over columns, lanes over the 32 rows (256 B
//            coalesced loads straight from HBM), r = A_p x - b_p in registers,
//            reduced across warps in a fixed order;
//   sweep 2: the same panel, now hot in L2, is staged through padded shared
//            memory in 64-column chunks and contracted with r into per-CTA
//            column partials (no atomics);
// a second kernel sums the per-CTA partials in fixed order and adds nu^2 x,
// so the result is deterministic run to run. Two right-hand sides share
// every load (both heavy-ball candidates of one iteration in one pass).
#include "common.cuh"

#include <cstdlib>

namespace ihs_b200 {

namespace {
constexpr int R = 32;        // rows per panel
constexpr int THREADS = 256; // 8 warps
constexpr int WARPS = THREADS / 32;
constexpr int CH = 64;       // columns per sweep-2 chunk
constexpr int UNROLL = 8;

template <int NRHS>
__global__ void __launch_bounds__(THREADS, 2)
grad_partial_kernel(const double* __restrict__ A, int64_t n, int64_t d, int64_t lda, const double* __restrict__ b,
                    const double* __restrict__ X, double* __restrict__ work) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double sm[];
    double* xs = sm;                          // NRHS * d
    double* gp = xs + NRHS * d;               // NRHS * d   per-CTA column partials
    double* red = gp + NRHS * d;              // WARPS * NRHS * R
    double* rv = red + WARPS * NRHS * R;      // NRHS * R
    double* tile = rv + NRHS * R;             // CH * (R+1)
    double* qp = tile + CH * (R + 1);         // 4 * NRHS * CH

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int64_t e = t; e < NRHS * d; e += THREADS) {
        xs[e] = X[e];
        gp[e] = 0.0;
    }
    __syncthreads();

    const int64_t npanels = (n + R - 1) / R;
    for (int64_t p = blockIdx.x; p < npanels; p += gridDim.x) {
        const int64_t i0 = p * R;
        const int64_t row = i0 + lane;
        const bool live = row < n;
        // ---- sweep 1: r = A_p x
        double acc[NRHS];
#pragma unroll
        for (int q = 0; q < NRHS; ++q) acc[q] = 0.0;
        const double* Arow = A + row;
        int64_t j = warp;
        for (; j + (UNROLL - 1) * WARPS < d; j += UNROLL * WARPS) {
            double a[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) a[u] = live ? __ldg(Arow + (j + u * WARPS) * lda) : 0.0;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) acc[q] = fma(a[u], xs[q * d + j + u * WARPS], acc[q]);
        }
        for (; j < d; j += WARPS) {
            const double a = live ? __ldg(Arow + j * lda) : 0.0;
#pragma unroll
            for (int q = 0; q < NRHS; ++q) acc[q] = fma(a, xs[q * d + j], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < NRHS; ++q) red[(warp * NRHS + q) * R + lane] = acc[q];
        __syncthreads();
        if (t < NRHS * R) {
            const int q = t / R, i = t % R;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) s += red[(w * NRHS + q) * R + i];
            const int64_t gi = i0 + i;
            rv[q * R + i] = gi < n ? s - b[gi] : 0.0;
        }
        __syncthreads();
        // ---- sweep 2: gp += A_p^T r (panel re-read from L2 through smem)
        for (int64_t j0 = 0; j0 < d; j0 += CH) {
            const int cw = (int)imin64(CH, d - j0);
            for (int c = warp; c < cw; c += WARPS)
                tile[c * (R + 1) + lane] = live ? __ldg(A + row + (j0 + c) * lda) : 0.0;
            __syncthreads();
            {
                const int c = t % CH, quarter = t / CH;  // 4 quarters of 8 rows
                if (c < cw) {
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) {
                        double s = 0.0;
#pragma unroll
                        for (int i = 0; i < R / 4; ++i) {
                            const int ii = quarter * (R / 4) + i;
                            s = fma(tile[c * (R + 1) + ii], rv[q * R + ii], s);
                        }
                        qp[(quarter * NRHS + q) * CH + c] = s;
                    }
                }
            }
            __syncthreads();
            if (t < NRHS * CH) {
                const int q = t / CH, c = t % CH;
                if (c < cw) {
                    const double s = (qp[(0 * NRHS + q) * CH + c] + qp[(1 * NRHS + q) * CH + c]) +
                                     (qp[(2 * NRHS + q) * CH + c] + qp[(3 * NRHS + q) * CH + c]);
                    gp[q * d + j0 + c] += s;
                }
            }
            // next chunk's tile writes are ordered after this read by the
            // __syncthreads at the top of the following iteration's compute
            __syncthreads();
        }
    }
    for (int64_t e = t; e < NRHS * d; e += THREADS) work[(int64_t)blockIdx.x * NRHS * d + e] = gp[e];
}

// ---------------------------------------------------------------- v2
// A is read exactly once: R x d row panels are streamed into shared memory
// with 8-byte cp.async (odd padded column stride R+1: conflict-free for both
// sweeps) and double buffered, so the next panel's HBM traffic overlaps both
// sweeps of the current one. Column partials live in registers.
constexpr int T2 = 512;
constexpr int W2 = T2 / 32;

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

// NS-stage ring of unpadded RR x d panels (16-byte cp.async.cg, L2 only);
// sweep 2 reads each column with a rotation of (j*RR/16) rows so the 32 lanes
// of a warp hit 16 distinct bank pairs.
template <int NRHS, int RR, int MAXC, int NS>
__global__ void __launch_bounds__(T2, 1)
grad_smem_kernel(const double* __restrict__ A, int64_t d, int64_t lda, const double* __restrict__ b,
                 const double* __restrict__ X, double* __restrict__ work) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double sm[];
    const int64_t stage = d * RR;
    double* panel = sm;                       // NS stages
    double* xs = panel + NS * stage;          // NRHS * d
    double* red = xs + NRHS * d;              // W2 * NRHS * RR
    double* rv = red + W2 * NRHS * RR;        // NRHS * RR
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int64_t e = t; e < NRHS * d; e += T2) xs[e] = X[e];

    double gacc[NRHS][MAXC];
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) gacc[q][c] = 0.0;

    const int64_t npanels = lda / RR;
    const int64_t chunks = (int64_t)RR * d / 2;  // 16-byte chunks per panel
    auto issue = [&](int64_t p, int s) {
        if (p < npanels) {
            double* dst = panel + s * stage;
            const double* src = A + p * RR;
            for (int64_t c = t; c < chunks; c += T2) {
                const int i = (int)(c % (RR / 2)) * 2;
                const int64_t j = c / (RR / 2);
                cp_async16(dst + j * RR + i, src + i + j * lda);
            }
        }
        cp_async_commit();  // one group per slot, possibly empty, keeps the wait count uniform
    };
    int64_t p = blockIdx.x;
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) issue(p + (int64_t)k * gridDim.x, k);
    int s = 0;
    for (; p < npanels; p += gridDim.x) {
        issue(p + (int64_t)(NS - 1) * gridDim.x, (s + NS - 1) % NS);
        cp_async_wait<NS - 1>();
        __syncthreads();
        const double* P = panel + s * stage;
        // ---- sweep 1: r = A_p x - b_p
        {
            const int i = t % RR;
            const int jg = t / RR;
            constexpr int G = T2 / RR;
            double acc[NRHS];
#pragma unroll
            for (int q = 0; q < NRHS; ++q) acc[q] = 0.0;
            for (int64_t j = jg; j < d; j += G) {
                const double a = P[j * RR + i];
#pragma unroll
                for (int q = 0; q < NRHS; ++q) acc[q] = fma(a, xs[q * d + j], acc[q]);
            }
#pragma unroll
            for (int off = RR; off < 32; off <<= 1)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
            if (lane < RR)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) red[(warp * NRHS + q) * RR + lane] = acc[q];
        }
        __syncthreads();
        if (t < NRHS * RR) {
            const int q = t / RR, i = t % RR;
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < W2; ++w) sum += red[(w * NRHS + q) * RR + i];
            rv[q * RR + i] = sum - b[p * RR + i];
        }
        __syncthreads();
        // ---- sweep 2: g += A_p^T r
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int64_t j = t + (int64_t)c * T2;
            if (j < d) {
                const int rot = (int)((j * RR / 16) & (RR - 1));
#pragma unroll
                for (int q = 0; q < NRHS; ++q) {
                    double sum = 0.0;
#pragma unroll
                    for (int i = 0; i < RR; ++i) {
                        const int ii = (i + rot) & (RR - 1);
                        sum = fma(P[j * RR + ii], rv[q * RR + ii], sum);
                    }
                    gacc[q][c] += sum;
                }
            }
        }
        __syncthreads();  // stage s is refilled by the next iteration's prefetch
        s = (s + 1) % NS;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int64_t j = t + (int64_t)c * T2;
            if (j < d) work[((int64_t)blockIdx.x * NRHS + q) * d + j] = gacc[q][c];
        }
}

size_t grad_smem_v2(int64_t d, int R, int nrhs, int ns) {
    return sizeof(double) * ((size_t)ns * d * R + (size_t)nrhs * d + (size_t)W2 * nrhs * R + (size_t)nrhs * R);
}

template <int NRHS, int RR, int NS>
void launch_v2(const GradPlan& p, const double* A, const double* b, const double* X, double* work, cudaStream_t st) {
    const size_t smem = grad_smem_v2(p.d, RR, NRHS, NS);
    const int maxc = (int)ceil_div(p.d, T2);
#define IHS_V2(MC)                                                                                                  \
    do {                                                                                                            \
        IHS_SMEM_ATTR((grad_smem_kernel<NRHS, RR, MC, NS>), 220 * 1024);                                                                                                           \
        LAUNCH_PDL((grad_smem_kernel<NRHS, RR, MC, NS>), p.grid, T2, smem, st, A, p.d, p.lda, b, X, work);              \
    } while (0)
    if (maxc <= 1) IHS_V2(1);
    else if (maxc <= 2) IHS_V2(2);
    else IHS_V2(4);
#undef IHS_V2
}

template <int NRHS>
void launch_v2_dispatch(const GradPlan& p, const double* A, const double* b, const double* X, double* work,
                        cudaStream_t st) {
    const int key = p.R * 10 + p.stages;
    switch (key) {
        case 163: launch_v2<NRHS, 16, 3>(p, A, b, X, work, st); break;
        case 164: launch_v2<NRHS, 16, 4>(p, A, b, X, work, st); break;
        case 83: launch_v2<NRHS, 8, 3>(p, A, b, X, work, st); break;
        case 84: launch_v2<NRHS, 8, 4>(p, A, b, X, work, st); break;
        case 42: launch_v2<NRHS, 4, 2>(p, A, b, X, work, st); break;
        case 43: launch_v2<NRHS, 4, 3>(p, A, b, X, work, st); break;
        default: fail(IHS_INTERNAL_ERROR, "gradient: no kernel for the chosen panel geometry");
    }
}

// G[q][j] = sum_c work[c][q][j] (fixed order) + nu2 * X[q][j]
// 256 threads = 16 entries x 16 part-groups; group g sums parts g, g+16, ...
// in order, then the 16 group sums are added in a fixed tree.
__global__ void __launch_bounds__(256) grad_reduce_kernel(const double* __restrict__ work, int nparts, int64_t d,
                                                          int nrhs, const double* __restrict__ X, double nu2,
                                                          double* __restrict__ G) {
    __shared__ double s[16][17];
    pdl_wait();  // launched programmatically after the partial-sum kernel
    pdl_trigger();
    const int64_t total = (int64_t)nrhs * d;
    const int c = threadIdx.x % 16, g = threadIdx.x / 16;
    const int64_t e = (int64_t)blockIdx.x * 16 + c;
    double acc = 0.0;
    if (e < total)
        for (int p = g; p < nparts; p += 16) acc += work[(int64_t)p * total + e];
    s[g][c] = acc;
    __syncthreads();
    if (threadIdx.x < 16 && e < total) {
        double t8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t8[i] = s[2 * i][c] + s[2 * i + 1][c];
#pragma unroll
        for (int i = 0; i < 4; ++i) t8[i] = t8[2 * i] + t8[2 * i + 1];
        const double sum = (t8[0] + t8[1]) + (t8[2] + t8[3]);
        G[e] = sum + nu2 * X[e];
    }
}

size_t grad_smem(int64_t d, int nrhs) {
    return sizeof(double) * ((size_t)nrhs * d * 2 + (size_t)WARPS * nrhs * R + (size_t)nrhs * R + (size_t)CH * (R + 1) +
                             (size_t)4 * nrhs * CH);
}
}  // namespace

GradPlan grad_plan(int64_t n, int64_t d, int64_t lda, int num_sms) {
    GradPlan p{};
    p.n = n;
    p.d = d;
    p.lda = lda;
    p.grid_sms = num_sms;
    // v2: one 512-thread CTA per SM streaming R x d panels through an NS-deep
    // cp.async ring (>= 3 x 64 KiB in flight per SM when it fits); prefer
    // 128/64 B column segments (R = 16/8), fall back to 32 B (R = 4).
    struct Cand { int R, ns; };
    const Cand cands[] = {{16, 4}, {16, 3}, {8, 4}, {8, 3}, {4, 3}, {4, 2}};
    p.version = 1;
    if (lda % 32 == 0 && d <= 2048) {
        for (const Cand& c : cands) {
            const size_t sm = grad_smem_v2(d, c.R, 2, c.ns);
            const size_t stage_bytes = (size_t)c.R * d * 8;
            if (sm <= 215u * 1024 && stage_bytes <= 64u * 1024) {
                p.version = 2;
                p.R = c.R;
                p.stages = c.ns;
                p.smem = sm;
                const int64_t npanels = lda / c.R;
                p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(npanels, (int64_t)num_sms));
                return p;
            }
        }
    }
    p.R = R;
    const int64_t npanels = (n + R - 1) / R;
    p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(npanels, (int64_t)num_sms * 2));
    p.smem = grad_smem(d, 2);
    if (p.smem > 220 * 1024) fail(IHS_INVALID_INPUT, "gradient: d too large for the fused kernel");
    return p;
}

// ---- v6: A too large for a row-major copy and too large for L2 — two streaming passes over column-major A.
// The fused column-major kernels (v2/v3) stage R-row panels, so each column contributes only an R x 8-byte
// segment per panel (1.2 TB/s at C4's shape); here every access is a long contiguous column run instead:
//   pass 1: R = A X - b, one CTA per 1024 rows, the columns streamed 4 at a time (8 KiB runs per column);
//   pass 2: per-block partials of A^T R, one CTA per 4096 rows (R's block in shared memory), one warp per
//           column at a time (32 KiB runs), partials reduced in fixed order by grad_reduce_kernel (+ nu^2 X).
constexpr int GC1_ROWS = 1024, GC2_ROWS = 4096;
template <int NR>
__global__ void __launch_bounds__(256) gcol_residual_kernel(const double* __restrict__ A, int64_t d, int64_t lda,
                                                            const double* __restrict__ b, const double* __restrict__ X,
                                                            double* __restrict__ R) {
    pdl_wait();
    extern __shared__ double gxs[];  // NR x d
    for (int64_t e = threadIdx.x; e < (int64_t)NR * d; e += 256) gxs[e] = X[e];
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * GC1_ROWS + threadIdx.x;
    double acc[NR][4];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[q][v] = 0.0;
    for (int64_t j = 0; j < d; j += 4) {
        double a[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t i = i0 + 256 * v;
                a[u][v] = (j + u < d && i < lda) ? __ldcs(A + i + (j + u) * lda) : 0.0;
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (j + u < d)
#pragma unroll
                for (int q = 0; q < NR; ++q) {
                    const double xv = gxs[q * d + j + u];
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[q][v] = fma(a[u][v], xv, acc[q][v]);
                }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const int64_t i = i0 + 256 * v;
        if (i < lda)
#pragma unroll
            for (int q = 0; q < NR; ++q) R[q * lda + i] = acc[q][v] - b[i];
    }
}

template <int NR>
__global__ void __launch_bounds__(256) gcol_partial_kernel(const double* __restrict__ A, int64_t d, int64_t lda,
                                                           const double* __restrict__ R, double* __restrict__ part) {
    pdl_wait();
    extern __shared__ double grs[];  // NR x GC2_ROWS
    const int64_t i0 = (int64_t)blockIdx.x * GC2_ROWS;
    const int rows = (int)(lda - i0 < GC2_ROWS ? lda - i0 : GC2_ROWS);
    for (int e = threadIdx.x; e < NR * GC2_ROWS; e += 256) {
        const int q = e / GC2_ROWS, i = e % GC2_ROWS;
        grs[e] = i < rows ? R[q * lda + i0 + i] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* out = part + (int64_t)blockIdx.x * NR * d;
    for (int64_t j = w; j < d; j += 8) {
        const double* col = A + j * lda + i0;
        double s[NR][2];
#pragma unroll
        for (int q = 0; q < NR; ++q) s[q][0] = s[q][1] = 0.0;
        for (int t = lane; t < rows; t += 256) {
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = t + 32 * u < rows ? __ldcs(col + t + 32 * u) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int q = 0; q < NR; ++q) s[q][u & 1] = fma(a[u], grs[q * GC2_ROWS + t + 32 * u], s[q][u & 1]);
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            double v = s[q][0] + s[q][1];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) out[q * d + j] = v;
        }
    }
}

size_t grad_work_doubles(const GradPlan& p) {
    return (size_t)p.grid * 2 * p.d + (p.version == 6 ? (size_t)2 * p.lda : 0);
}

bool grad_plan_use_rowmajor(GradPlan& p) {
    static const bool disabled = [] {
        const char* e = std::getenv("IHS_GRAD_NO_ROWMAJOR");
        return e && e[0] == '1';
    }();
    static const bool no_rr = [] {
        const char* e = std::getenv("IHS_GRAD_NO_RR");
        return e && e[0] == '1';
    }();
    int R = 0, ns = 0;
    if (disabled) return false;
    if (!no_rr && grad_rr_geometry(p.d, p.lda, &R, &ns)) {
        p.version = 5;
        p.smem = grad_rr_smem(p.d, R, ns);
    } else if (grad_rm_geometry(p.d, p.lda, &R, &ns)) {
        p.version = 4;
        p.smem = grad_rm_smem(p.d, R, 2, ns);
    } else {
        return false;
    }
    p.R = R;
    p.stages = ns;
    const int64_t npanels = p.lda / R;
    p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(npanels, (int64_t)p.grid_sms));
    return true;
}

void grad_plan_attach_tma(GradPlan& p, const double* d_A) {
    static const bool disabled = [] {
        const char* e = std::getenv("IHS_GRAD_NO_TMA");
        return e && e[0] == '1';
    }();
    static const bool no_colpass = [] {  // IHS_GRAD_NO_COLPASS=1: keep the fused column-major kernels (A/B)
        const char* e = std::getenv("IHS_GRAD_NO_COLPASS");
        return e && e[0] == '1';
    }();
    // A beyond L2 by far (> 1 GiB): the two streaming passes (x in shared memory: d <= 8192)
    if (!no_colpass && 8.0 * (double)p.lda * (double)p.d > (double)(1ll << 30) && p.d <= 8192) {
        p.version = 6;
        p.grid = (int)ceil_div(p.lda, (int64_t)GC2_ROWS);
        return;
    }
    if (disabled || p.version != 2) return;
    if (grad_tma_smem(p.d, p.R, 2, p.stages) > 225u * 1024) return;
    if (!grad_tma_make_map(d_A, p.lda, p.d, p.R, p.tmap)) return;
    p.version = 3;
}

void grad_run(const GradPlan& p, const double* d_A, const double* d_b, double nu2, const double* d_X, int nrhs,
              double* d_G, double* d_work, cudaStream_t st, const double* d_Arm, const CandSpec* cs) {
    if (cs) {
        d_X = cs->out;
        if (p.version != 5)
            candidates(cs->x, cs->xprev, cs->gt, cs->mu_p, cs->beta_p, cs->mu_gd, p.d, nrhs == 2 ? cs->out : nullptr,
                       nrhs == 2 ? cs->out + p.d : cs->out, st);
    }
    if (p.version == 6) {
        double* R = d_work + (size_t)p.grid * 2 * p.d;
        const size_t xs = (size_t)nrhs * p.d * sizeof(double), rs = (size_t)nrhs * GC2_ROWS * sizeof(double);
        const unsigned g1 = (unsigned)ceil_div(p.lda, (int64_t)GC1_ROWS);
        if (nrhs == 1) {
            IHS_SMEM_ATTR((gcol_residual_kernel<1>), 64 * 1024);
            IHS_SMEM_ATTR((gcol_partial_kernel<1>), 64 * 1024);
            LAUNCH_PDL(gcol_residual_kernel<1>, g1, 256, xs, st, d_A, p.d, p.lda, d_b, d_X, R);
            LAUNCH_PDL(gcol_partial_kernel<1>, (unsigned)p.grid, 256, rs, st, d_A, p.d, p.lda, (const double*)R, d_work);
        } else {
            IHS_SMEM_ATTR((gcol_residual_kernel<2>), 128 * 1024);
            IHS_SMEM_ATTR((gcol_partial_kernel<2>), 64 * 1024);
            LAUNCH_PDL(gcol_residual_kernel<2>, g1, 256, xs, st, d_A, p.d, p.lda, d_b, d_X, R);
            LAUNCH_PDL(gcol_partial_kernel<2>, (unsigned)p.grid, 256, rs, st, d_A, p.d, p.lda, (const double*)R, d_work);
        }
        const int64_t total = (int64_t)nrhs * p.d;
        LAUNCH_PDL(grad_reduce_kernel, dim3((unsigned)ceil_div(total, 16)), dim3(256), 0, st, (const double*)d_work,
                   p.grid, p.d, nrhs, d_X, nu2, d_G);
        return;
    }
    if (p.version >= 2) {
        if (p.version == 5) grad_rr_run(p, d_Arm, d_b, d_X, nrhs, d_work, st, cs);
        else if (p.version == 4) grad_rm_run(p, d_Arm, d_b, d_X, nrhs, d_work, st);
        else if (p.version == 3) grad_tma_run(p, d_b, d_X, nrhs, d_work, st);
        else if (nrhs == 1) launch_v2_dispatch<1>(p, d_A, d_b, d_X, d_work, st);
        else launch_v2_dispatch<2>(p, d_A, d_b, d_X, d_work, st);
        const int64_t total = (int64_t)nrhs * p.d;
        LAUNCH_PDL(grad_reduce_kernel, dim3((unsigned)ceil_div(total, 16)), dim3(256), 0, st, (const double*)d_work,
                   p.grid, p.d, nrhs, d_X, nu2, d_G);
        return;
    }
    const size_t smem = grad_smem(p.d, nrhs);
    IHS_SMEM_ATTR((grad_partial_kernel<1>), 220 * 1024);
    IHS_SMEM_ATTR((grad_partial_kernel<2>), 220 * 1024);
    if (nrhs == 1)
        LAUNCH_PDL(grad_partial_kernel<1>, p.grid, THREADS, smem, st, d_A, p.n, p.d, p.lda, d_b, d_X, d_work);
    else
        LAUNCH_PDL(grad_partial_kernel<2>, p.grid, THREADS, smem, st, d_A, p.n, p.d, p.lda, d_b, d_X, d_work);
    const int64_t total = (int64_t)nrhs * p.d;
    LAUNCH_PDL(grad_reduce_kernel, (unsigned)ceil_div(total, 16), 256, 0, st, d_work, p.grid, p.d, nrhs, d_X, nu2, d_G);
}

}  // namespace ihs_b200
