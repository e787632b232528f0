// grad_rm.cu — fused gradient over a row-major copy of A (sm_100a).
//
// Column-major R-row panels are R*8-byte segments 8*lda bytes apart, so a
// panel read opens a DRAM page per column and the gradient stalls on HBM
// locality well below the copy roofline. The problem therefore also keeps A
// row-major (one transpose at upload); a panel of R rows is then one
// contiguous R*d*8-byte block, moved into shared memory by a single 1D bulk
// TMA copy (cp.async.bulk) per stage with mbarrier completion.
//   sweep 1: warps own rows (two warps per row when R = 8), lanes stride the
//            contiguous row, warp-shuffle reduction -> r = A_p x - b_p;
//   sweep 2: thread per column, conflict-free reads down the R rows,
//            r held in registers -> per-CTA column partials.
// Same fixed-order partial reduction as the other variants (deterministic).
#include "common.cuh"

namespace ihs_b200 {

namespace {
constexpr int TT = 512;
constexpr int TW = TT / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// the same with an L2 cache policy: panels [0, keep) of A are loaded evict-last so they stay in L2 from one pass to
// the next (A a few times larger than L2: C2), the rest evict-first so they do not displace them
__device__ __forceinline__ void bulk_load_pol(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
                 "%4;" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}

// RR rows per panel, MAXC = ceil(d / 512) columns per thread, NS stages.
template <int NRHS, int RR, int MAXC, int NS>
__global__ void __launch_bounds__(TT, 1)
grad_rm_kernel(const double* __restrict__ Arm, int64_t d, int64_t npanels, const double* __restrict__ b,
               const double* __restrict__ X, double* __restrict__ work) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ __align__(128) double sm[];
    const int64_t stage = (int64_t)RR * d;
    double* panel = sm;
    double* xs = panel + NS * stage;     // interleaved [j][q]
    double* red = xs + NRHS * d;         // TW * NRHS
    double* rv = red + TW * NRHS;        // NRHS * RR
    uint64_t* full = reinterpret_cast<uint64_t*>(rv + NRHS * RR + 2);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t stage_bytes = (uint32_t)(stage * sizeof(double));
    if (t == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int64_t e = t; e < NRHS * d; e += TT) {
        const int64_t q = e / d, j = e % d;
        xs[j * NRHS + q] = X[e];
    }
    __syncthreads();
    auto issue = [&](int64_t p, int s) {  // thread 0
        if (p >= npanels) return;
        mbar_expect_tx(&full[s], stage_bytes);
        bulk_load(panel + s * stage, Arm + p * stage, stage_bytes, &full[s]);
    };
    int64_t p = blockIdx.x;
    if (t == 0)
        for (int k = 0; k < NS; ++k) issue(p + (int64_t)k * gridDim.x, k);

    double gacc[NRHS][MAXC];
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) gacc[q][c] = 0.0;

    // sweep-1 ownership: WPR warps per row (TW >= RR), each a contiguous 1/WPR of the row
    constexpr int WPR = TW / RR > 0 ? TW / RR : 1;
    constexpr int ROWS_PER_WARP = RR > TW ? RR / TW : 1;
    int s = 0;
    uint32_t phase = 0;
    for (; p < npanels; p += gridDim.x) {
        mbar_wait(&full[s], phase);
        const double* P = panel + s * stage;
        // ---- sweep 1
#pragma unroll
        for (int rr = 0; rr < ROWS_PER_WARP; ++rr) {
            const int row = (warp / WPR) * ROWS_PER_WARP + rr;
            const int part = warp % WPR;
            const int64_t seg = (d + WPR - 1) / WPR;
            const int64_t len = min(seg, d - part * seg);
            const double* Prow = P + (int64_t)row * d + part * seg;
            const double* xr = xs + part * seg * NRHS;
            double acc[NRHS];
#pragma unroll
            for (int q = 0; q < NRHS; ++q) acc[q] = 0.0;
#pragma unroll 4
            for (int64_t j = lane; j < len; j += 32) {
                const double a = Prow[j];
                if constexpr (NRHS == 2) {
                    const double2 xv = *reinterpret_cast<const double2*>(xr + 2 * j);
                    acc[0] = fma(a, xv.x, acc[0]);
                    acc[1] = fma(a, xv.y, acc[1]);
                } else {
                    acc[0] = fma(a, xr[j], acc[0]);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) red[(row * WPR + part) * NRHS + q] = acc[q];
        }
        __syncthreads();
        if (t < NRHS * RR) {
            const int q = t / RR, i = t % RR;
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < WPR; ++w) sum += red[(i * WPR + w) * NRHS + q];
            rv[q * RR + i] = sum - b[p * RR + i];
        }
        __syncthreads();
        // ---- sweep 2
        {
            double r[NRHS][RR];
#pragma unroll
            for (int q = 0; q < NRHS; ++q)
#pragma unroll
                for (int i = 0; i < RR; ++i) r[q][i] = rv[q * RR + i];
#pragma unroll
            for (int c = 0; c < MAXC; ++c) {
                const int64_t j = t + (int64_t)c * TT;
                if (j < d) {
#pragma unroll
                    for (int i = 0; i < RR; ++i) {
                        const double a = P[(int64_t)i * d + j];
#pragma unroll
                        for (int q = 0; q < NRHS; ++q) gacc[q][c] = fma(a, r[q][i], gacc[q][c]);
                    }
                }
            }
        }
        __syncthreads();  // stage s consumed
        if (t == 0) issue(p + (int64_t)NS * gridDim.x, s);
        if (++s == NS) {
            s = 0;
            phase ^= 1;
        }
    }
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int64_t j = t + (int64_t)c * TT;
            if (j < d) work[((int64_t)blockIdx.x * NRHS + q) * d + j] = gacc[q][c];
        }
}

// row-major copy: Arm[i * ldo + j] = A[i + j * lda], 32x32 tiles through smem
__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t d,
                                 double* __restrict__ Arm, int64_t ldo) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int64_t i = i0 + tx, j = j0 + k;
        tile[k][tx] = (i < rows && j < d) ? A[i + j * lda] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t i = i0 + k, j = j0 + tx;
        if (i < rows && j < d) Arm[i * ldo + j] = tile[tx][k];
    }
}


// ---- v5: register-resident rows (d <= 512). Warp w of the 8 consumer warps
// owns rows w, w+8, ... of every panel; lane l holds the column pairs
// 2l + 64k of its row in registers, so one shared read of the row serves both
// sweeps: r = A_i x - b_i is a warp xor-allreduce (bitwise identical on every
// lane: each step adds the same two values), then the lane updates its
// column-pair partials with A_i^T r. No CTA barrier per panel: lane 0 of warp
// 0 refills a stage once all 8 warps arrived on its "empty" mbarrier (no
// dedicated producer warp: with 8 warps = 2 per SM sub-partition every thread
// may hold up to 255 registers). The per-warp
// partials are summed in warp order at the end (deterministic, like the other
// variants).
constexpr int RW = 8;  // consumer warps
constexpr int RTHREADS = 32 * RW;

// CG column groups: a row's d columns are split over CG warps (64 KP columns each; CG = 1 for d <= 512),
// so x and the column partials of every warp stay in registers up to d = 4096. The CG warps of a row
// group (RW / CG of them run side by side) combine their partial row dots through shared memory and one
// named barrier per row, summing them in column-group order: every warp of the group forms the same r.
template <int NRHS, int KP, int RR, int NS, int CG>
__global__ void __launch_bounds__(RTHREADS, 1)
grad_rr_kernel(const double* __restrict__ Arm, int64_t d, int64_t npanels, const double* __restrict__ b,
               const double* __restrict__ X, double* __restrict__ work, CandSpec cs, int64_t keep) {
    constexpr int RG = RW / CG;  // row groups (rows in flight)
    extern __shared__ __align__(128) double sm[];
    const int64_t stage = (int64_t)RR * d;
    double* panel = sm;
    uint64_t* full = reinterpret_cast<uint64_t*>(panel + NS * stage);
    uint64_t* empty = full + NS;
    double* dotp = reinterpret_cast<double*>(empty + NS);  // [2][RG][CG][NRHS] partial row dots
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int cg = warp % CG, rg = warp / CG;
    const int64_t c0 = (int64_t)cg * 64 * KP;  // first column of this warp
    if (t == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], RW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t stage_bytes = (uint32_t)(stage * sizeof(double));
    uint64_t pol_last = 0, pol_first = 0;
    if (keep > 0) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    }
    // prologue: the first NS panels (A is constant for the whole solve, so these loads may overlap the
    // tail of the previous kernel under programmatic dependent launch)
    if (t == 0) {
        int64_t p = blockIdx.x;
        for (int k = 0; k < NS && p < npanels; ++k, p += gridDim.x) {
            mbar_expect_tx(&full[k], stage_bytes);
            if (keep > 0) bulk_load_pol(panel + k * stage, Arm + p * stage, stage_bytes, &full[k], p < keep ? pol_last : pol_first);
            else bulk_load(panel + k * stage, Arm + p * stage, stage_bytes, &full[k]);
        }
    }
    pdl_wait();  // x / the heavy-ball state and the work buffer belong to the previous kernels
    {
        // ---------------- consumers
        // x of the right-hand sides in registers: read, or (cs.x != nullptr) formed here from the
        // heavy-ball state exactly like candidates_kernel (solver.hpp:182,190; no FMA contraction),
        // CTA 0 publishing them for the caller
        double2 xr[NRHS][KP];
        if (cs.x == nullptr) {
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int64_t j = c0 + 2 * lane + 64 * k;
#pragma unroll
                for (int q = 0; q < NRHS; ++q)
                    xr[q][k] = j < d ? *reinterpret_cast<const double2*>(X + q * d + j) : make_double2(0.0, 0.0);
            }
        } else {
            // all loads first (16-byte, independent), then the candidate arithmetic
            double2 xa[KP], ga[KP], pa[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int64_t j = c0 + 2 * lane + 64 * k;
                const bool in = j < d;
                xa[k] = in ? *reinterpret_cast<const double2*>(cs.x + j) : make_double2(0.0, 0.0);
                ga[k] = in ? *reinterpret_cast<const double2*>(cs.gt + j) : make_double2(0.0, 0.0);
                pa[k] = in && NRHS == 2 ? *reinterpret_cast<const double2*>(cs.xprev + j) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int64_t j = c0 + 2 * lane + 64 * k;
                double xv[2][NRHS];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double xi = h ? xa[k].y : xa[k].x, gi = h ? ga[k].y : ga[k].x;
                    const double xg = __dsub_rn(xi, __dmul_rn(cs.mu_gd, gi));
                    if (NRHS == 2) {
                        const double xp = h ? pa[k].y : pa[k].x;
                        xv[h][0] = __dadd_rn(__dsub_rn(xi, __dmul_rn(cs.mu_p, gi)),
                                             __dmul_rn(cs.beta_p, __dsub_rn(xi, xp)));
                        xv[h][NRHS - 1] = xg;
                    } else {
                        xv[h][0] = xg;
                    }
                }
#pragma unroll
                for (int q = 0; q < NRHS; ++q) {
                    xr[q][k] = j < d ? make_double2(xv[0][q], xv[1][q]) : make_double2(0.0, 0.0);
                    if (blockIdx.x == 0 && rg == 0 && j < d)
                        *reinterpret_cast<double2*>(cs.out + q * d + j) = make_double2(xv[0][q], xv[1][q]);
                }
            }
        }
        double2 g[NRHS][KP];
#pragma unroll
        for (int q = 0; q < NRHS; ++q)
#pragma unroll
            for (int k = 0; k < KP; ++k) g[q][k] = make_double2(0.0, 0.0);
        int s = 0;
        uint32_t ph = 0;
        int par = 0;  // dotp buffer parity (alternates per row)
        // this warp's observations one panel ahead (global-load latency hidden behind a whole panel)
        double bq[RR / RG];
#pragma unroll
        for (int rr = 0; rr < RR / RG; ++rr)
            bq[rr] = (int64_t)blockIdx.x < npanels ? __ldg(b + (int64_t)blockIdx.x * RR + rg + RG * rr) : 0.0;
        for (int64_t p = blockIdx.x; p < npanels; p += gridDim.x) {
            double bn[RR / RG];
            const int64_t pn_b = p + gridDim.x < npanels ? p + gridDim.x : p;
#pragma unroll
            for (int rr = 0; rr < RR / RG; ++rr) bn[rr] = __ldg(b + pn_b * RR + rg + RG * rr);
            mbar_wait(&full[s], ph);
            const double* P = panel + s * stage;
#pragma unroll
            for (int rr = 0; rr < RR / RG; ++rr) {
                const int row = rg + RG * rr;
                const double bi = bq[rr];
                double2 a[KP];
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    const int64_t j = c0 + 2 * lane + 64 * k;
                    a[k] = j < d ? *reinterpret_cast<const double2*>(P + row * d + j) : make_double2(0.0, 0.0);
                }
                // the row dot product runs as four independent chains per right-hand side, summed in a
                // fixed tree (then over the column groups in order)
                double r[NRHS];
#pragma unroll
                for (int q = 0; q < NRHS; ++q) {
                    double c4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int k = 0; k < KP; ++k) {
                        c4[(2 * k) & 3] = fma(a[k].x, xr[q][k].x, c4[(2 * k) & 3]);
                        c4[(2 * k + 1) & 3] = fma(a[k].y, xr[q][k].y, c4[(2 * k + 1) & 3]);
                    }
                    double acc = (c4[0] + c4[1]) + (c4[2] + c4[3]);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    r[q] = acc;
                }
                if constexpr (CG > 1) {
                    double* slot = dotp + ((par * RG + rg) * CG) * NRHS;
                    if (lane == 0)
#pragma unroll
                        for (int q = 0; q < NRHS; ++q) slot[cg * NRHS + q] = r[q];
                    // the group's CG warps; the next row uses the other buffer, and this barrier of the
                    // next row orders its writes after every read below
                    asm volatile("bar.sync %0, %1;" ::"r"(1 + rg), "r"(32 * CG) : "memory");
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) {
                        double acc = slot[q];
#pragma unroll
                        for (int c = 1; c < CG; ++c) acc += slot[c * NRHS + q];
                        r[q] = acc;
                    }
                    par ^= 1;
                }
#pragma unroll
                for (int q = 0; q < NRHS; ++q) r[q] -= bi;
#pragma unroll
                for (int q = 0; q < NRHS; ++q)
#pragma unroll
                    for (int k = 0; k < KP; ++k) {
                        g[q][k].x = fma(a[k].x, r[q], g[q][k].x);
                        g[q][k].y = fma(a[k].y, r[q], g[q][k].y);
                    }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            if (t == 0) {
                // producer: refill stage s with panel p + NS*grid once every warp released it
                const int64_t pn = p + (int64_t)NS * gridDim.x;
                if (pn < npanels) {
                    mbar_wait(&empty[s], ph);
                    mbar_expect_tx(&full[s], stage_bytes);
                    if (keep > 0)
                        bulk_load_pol(panel + s * stage, Arm + pn * stage, stage_bytes, &full[s],
                                      pn < keep ? pol_last : pol_first);
                    else
                        bulk_load(panel + s * stage, Arm + pn * stage, stage_bytes, &full[s]);
                }
            }
            if (++s == NS) {
                s = 0;
                ph ^= 1u;
            }
#pragma unroll
            for (int rr = 0; rr < RR / RG; ++rr) bq[rr] = bn[rr];
        }
        // per-row-group partials -> shared [rg][q][d] (the ring is free once every warp is here)
        pdl_trigger();  // the fixed-order reduce may be scheduled now; it waits for this grid to finish
        __syncthreads();
        double* red = panel;
#pragma unroll
        for (int q = 0; q < NRHS; ++q)
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int64_t j = c0 + 2 * lane + 64 * k;
                if (j < d) *reinterpret_cast<double2*>(red + ((int64_t)rg * NRHS + q) * d + j) = g[q][k];
            }
        __syncthreads();
        for (int64_t e = t; e < NRHS * d; e += 32 * RW) {
            const int64_t q = e / d, j = e % d;
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < RG; ++w) sum += red[((int64_t)w * NRHS + q) * d + j];
            work[((int64_t)blockIdx.x * NRHS + q) * d + j] = sum;
        }
    }
}

template <int NRHS, int KP, int RR, int NS, int CG>
void launch_rr(const GradPlan& p, const double* Arm, const double* b, const double* X, double* work, cudaStream_t st,
               const CandSpec& cs) {
    const size_t smem = grad_rr_smem(p.d, RR, NS);
    IHS_SMEM_ATTR((grad_rr_kernel<NRHS, KP, RR, NS, CG>), 227 * 1024);
    // A up to ~4x L2: keep its first ~80 MiB of panels L2-resident across passes (IHS_GRAD_L2_KEEP_MB, 0 = off);
    // larger A gains nothing from it and its evict-last lines would crowd the SRHT's L2 ring
    static const int64_t keep_mb = [] {
        const char* e = std::getenv("IHS_GRAD_L2_KEEP_MB");
        return e ? (int64_t)std::atoll(e) : (int64_t)80;
    }();
    const int64_t a_bytes = p.lda * p.d * (int64_t)sizeof(double);
    const int64_t stage_b = (int64_t)RR * p.d * (int64_t)sizeof(double);
    const int64_t keep = (keep_mb > 0 && a_bytes <= (512ll << 20)) ? std::min<int64_t>(p.lda / RR, (keep_mb << 20) / stage_b)
                                                                   : 0;
    LAUNCH_PDL((grad_rr_kernel<NRHS, KP, RR, NS, CG>), dim3(p.grid), dim3(RTHREADS), smem, st, Arm, p.d,
               p.lda / RR, b, X, work, cs, keep);
}

template <int NRHS, int RR, int NS>
void launch_rm(const GradPlan& p, const double* Arm, const double* b, const double* X, double* work, cudaStream_t st) {
    const size_t smem = grad_rm_smem(p.d, RR, NRHS, NS);
    const int maxc = (int)ceil_div(p.d, TT);
#define IHS_RM(MC)                                                                                                  \
    do {                                                                                                            \
        IHS_SMEM_ATTR((grad_rm_kernel<NRHS, RR, MC, NS>), 227 * 1024);                                                                                                           \
        LAUNCH_PDL((grad_rm_kernel<NRHS, RR, MC, NS>), p.grid, TT, smem, st, Arm, p.d, p.lda / RR, b, X, work);         \
    } while (0)
    if (maxc <= 1) IHS_RM(1);
    else if (maxc <= 2) IHS_RM(2);
    else if (maxc <= 4) IHS_RM(4);
    else IHS_RM(8);
#undef IHS_RM
}
}  // namespace

size_t grad_rm_smem(int64_t d, int R, int nrhs, int ns) {
    return sizeof(double) * ((size_t)ns * R * d + (size_t)nrhs * d + (size_t)TW * nrhs + (size_t)nrhs * R + 2) +
           (size_t)ns * 8 + 128;
}

// column groups per row (power of two): 64 * 8 columns per warp at most
int rr_cg(int64_t d) { return d <= 512 ? 1 : d <= 1024 ? 2 : d <= 2048 ? 4 : 8; }

size_t grad_rr_smem(int64_t d, int R, int ns) {
    const size_t red = (size_t)(RW / rr_cg(d)) * 2 * d * sizeof(double);
    return std::max((size_t)ns * R * d * sizeof(double), red) + (size_t)2 * ns * 8 + 2 * RW * 2 * 8 + 128;
}

// v5 geometry: d <= 4096 (even). d <= 512: 16-row panels (8-row when 16 do not fit), as many stages as fit
// 200 KiB (<= 6); wider rows: 64 KiB panels (8 / 4 / 2 rows for 2 / 4 / 8 column groups), 3 stages
bool grad_rr_geometry(int64_t d, int64_t lda, int* R, int* ns) {
    if (d > 4096 || d % 2 || d < 2) return false;
    const int cg = rr_cg(d);
    if (cg > 1) {
        const int r = 16 / cg;
        if (lda % r) return false;
        *R = r;
        *ns = 3;
        return grad_rr_smem(d, r, 3) <= 200u * 1024;
    }
    for (int r : {16, 8}) {
        if (lda % r) continue;
        int k = 6;
        while (k >= 2 && grad_rr_smem(d, r, k) > 200u * 1024) --k;
        if (k >= 2) {
            *R = r;
            *ns = k;
            return true;
        }
    }
    return false;
}

void grad_rr_run(const GradPlan& p, const double* Arm, const double* b, const double* X, int nrhs, double* work,
                 cudaStream_t st, const CandSpec* csp) {
    const CandSpec cs = csp ? *csp : CandSpec{};
    const int cg = rr_cg(p.d);
    const int kp = (int)ceil_div(ceil_div(p.d, cg), 64);
    const int kpc = kp <= 2 ? 2 : kp <= 4 ? 4 : 8;
#define IHS_RR(KPv, RRv, NSv, CGv)                                                                \
    if (cg == CGv && kpc == KPv && p.R == RRv && p.stages == NSv) {                               \
        if (nrhs == 1) launch_rr<1, KPv, RRv, NSv, CGv>(p, Arm, b, X, work, st, cs);               \
        else launch_rr<2, KPv, RRv, NSv, CGv>(p, Arm, b, X, work, st, cs);                         \
        return;                                                                                    \
    }
#define IHS_RR_NS(KPv, RRv) \
    IHS_RR(KPv, RRv, 2, 1) IHS_RR(KPv, RRv, 3, 1) IHS_RR(KPv, RRv, 4, 1) IHS_RR(KPv, RRv, 5, 1) IHS_RR(KPv, RRv, 6, 1)
    IHS_RR_NS(2, 16) IHS_RR_NS(4, 16) IHS_RR_NS(8, 16)
    IHS_RR_NS(2, 8) IHS_RR_NS(4, 8) IHS_RR_NS(8, 8)
    IHS_RR(8, 8, 3, 2) IHS_RR(8, 4, 3, 4) IHS_RR(8, 2, 3, 8)  // wider rows: 257..512 columns per warp
#undef IHS_RR_NS
#undef IHS_RR
    fail(IHS_INTERNAL_ERROR, "gradient (register rows): no kernel for the chosen geometry");
}

// panel rows / ring depth for the row-major kernel: 64 KiB contiguous panels
bool grad_rm_geometry(int64_t d, int64_t lda, int* R, int* ns) {
    if (d > 4096) return false;
    int r = 1;
    while (r * 2 <= 16 && (int64_t)(r * 2) * d <= 8192) r *= 2;  // power of two, <= 64 KiB panels
    if (lda % r || ((int64_t)r * d) % 2) return false;           // 16-byte aligned bulk copies
    for (int k = 4; k >= 2; --k)
        if (grad_rm_smem(d, r, 2, k) <= 220u * 1024) {
            *R = r;
            *ns = k;
            return true;
        }
    if (r > 1) {  // very wide rows: smaller panels
        r /= 2;
        for (int k = 4; k >= 2; --k)
            if (grad_rm_smem(d, r, 2, k) <= 220u * 1024) {
                *R = r;
                *ns = k;
                return true;
            }
    }
    return false;
}

void transpose_to_rowmajor(const double* A, int64_t lda, int64_t rows, int64_t d, double* Arm, cudaStream_t st,
                           int64_t ldo) {
    dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(d, 32));
    LAUNCH_PDL(transpose_kernel, grid, dim3(32, 8), 0, st, A, lda, rows, d, Arm, ldo > 0 ? ldo : d);
}

void grad_rm_run(const GradPlan& p, const double* Arm, const double* b, const double* X, int nrhs, double* work,
                 cudaStream_t st) {
    const int key = p.R * 10 + p.stages;
#define IHS_CASE(RRv, NSv)                                                         \
    case RRv * 10 + NSv:                                                           \
        if (nrhs == 1) launch_rm<1, RRv, NSv>(p, Arm, b, X, work, st);             \
        else launch_rm<2, RRv, NSv>(p, Arm, b, X, work, st);                       \
        return;
    switch (key) {
        IHS_CASE(16, 2) IHS_CASE(16, 3) IHS_CASE(16, 4)
        IHS_CASE(8, 2) IHS_CASE(8, 3) IHS_CASE(8, 4)
        IHS_CASE(4, 2) IHS_CASE(4, 3) IHS_CASE(4, 4)
        IHS_CASE(2, 2) IHS_CASE(2, 3) IHS_CASE(2, 4)
        IHS_CASE(1, 2) IHS_CASE(1, 3) IHS_CASE(1, 4)
    }
#undef IHS_CASE
    fail(IHS_INTERNAL_ERROR, "gradient (row-major): no kernel for the chosen panel geometry");
}

}  // namespace ihs_b200
