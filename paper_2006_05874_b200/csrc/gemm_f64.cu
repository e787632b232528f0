// gemm_f64.cu — fp64 GEMM on the DMMA tensor path (mma.sync m8n8k4 .f64).
//
// sm_100a has no fp64 tcgen05 kind (tcgen05.mma offers f16/tf32/f8f6f4/i8/mx*
// only), so double-precision tensor work uses the legacy DMMA instruction.
// Used for:
//   * Gaussian sketch  S*A            (sketch.hpp:68)          N,N   split-K
//   * Gram SYRK        SA^T*SA        (sketched_system.hpp:78)  T,N   lower
//   * Woodbury inner   SA*SA^T        (sketched_system.hpp:74)  N,T   lower
//   * Cholesky trailing update A22 -= L21 L21^T                N,T   lower
// CTA tile 64x64x16, 4 warps (2x2) of 32x32, register-staged prefetch of the
// next K tile, deterministic split-K through a workspace (fixed-order sum).
#include "common.cuh"

#include <cstdlib>

namespace ihs_b200 {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDS = 68;  // padded row stride: conflict-free m8n8k4 fragment loads
constexpr int THREADS = 128;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS)
dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
             const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
             int lower_only, int64_t k_per_split, double* __restrict__ work, int64_t sA = 0, int64_t sB = 0,
             int64_t sC = 0) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int64_t n0 = (int64_t)blockIdx.y * BN;
    if (lower_only && n0 > m0 + BM - 1) return;
    // strided batch (sC != 0): blockIdx.z is the problem index, no split-K
    const bool batched = sC != 0;
    if (batched) {
        A += (int64_t)blockIdx.z * sA;
        B += (int64_t)blockIdx.z * sB;
        C += (int64_t)blockIdx.z * sC;
    }
    const int64_t kbeg = batched ? 0 : (int64_t)blockIdx.z * k_per_split;
    const int64_t kend = min(K, kbeg + k_per_split);

    __shared__ double As[BK][LDS];
    __shared__ double Bs[BK][LDS];

    const int t = threadIdx.x;
    const int lane = t & 31;
    const int warp = t >> 5;
    const int wm = (warp & 1) * 32;
    const int wn = (warp >> 1) * 32;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double ra[8], rb[8];
    auto load_tile = [&](int64_t k0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = t + THREADS * u;
            int mm, kk;
            if (!TA) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            double v = 0.0;
            if (gm < M && gk < kend) v = TA ? __ldg(A + gk + gm * lda) : __ldg(A + gm + gk * lda);
            ra[u] = v;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = t + THREADS * u;
            int nn, kk;
            if (!TB) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
            const int64_t gn = n0 + nn, gk = k0 + kk;
            double v = 0.0;
            if (gn < N && gk < kend) v = TB ? __ldg(B + gn + gk * ldb) : __ldg(B + gk + gn * ldb);
            rb[u] = v;
        }
    };
    auto store_tile = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = t + THREADS * u;
            int mm, kk;
            if (!TA) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
            As[kk][mm] = ra[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = t + THREADS * u;
            int nn, kk;
            if (!TB) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
            Bs[kk][nn] = rb[u];
        }
    };

    if (kbeg < kend) load_tile(kbeg);
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
        __syncthreads();
        store_tile();
        __syncthreads();
        if (k0 + BK < kend) load_tile(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
            const int kr = kk + (lane & 3);
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[kr][wm + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[kr][wn + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }

    // epilogue: lane holds rows (lane>>2), cols 2*(lane&3)+{0,1} of each 8x8 tile
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gm = m0 + wm + i * 8 + (lane >> 2);
                const int64_t gn = n0 + wn + j * 8 + 2 * (lane & 3) + h;
                if (gm >= M || gn >= N) continue;
                const double v = acc[i][j][h];
                if (work) {
                    work[(int64_t)blockIdx.z * M * N + gm + gn * M] = v;
                } else {
                    double out = alpha * v;
                    if (beta != 0.0) out += beta * C[gm + gn * ldc];
                    C[gm + gn * ldc] = out;
                }
            }
}


// ---- large GEMM: 128x128 CTA tile, 8 warps of 64x32, 4-stage cp.async ring, any transposition.
// Each operand is staged so its 16-byte cp.async writes and the m8n8k4 fragment reads are conflict-free:
//   m-contiguous A (NN/NT: A(m,k) at A + m + k lda) -> k-major As[k][m], row stride 132;
//   k-contiguous A (TN/TT: A(m,k) at A + k + m lda) -> m-major As[m][k], row stride 20;
//   k-contiguous B (NN/TN: B(k,n) at B + k + n ldb) -> n-major Bs[n][k], row stride 20;
//   n-contiguous B (NT/TT: B(k,n) at B + n + k ldb) -> k-major Bs[k][n], row stride 132.
// Used for S*A (NN), the Gram SYRK SA^T SA (TN, lower tiles only), the Woodbury inner SA SA^T (NT, lower) and
// H_S^{-1} = W^T W (TN). lower_only skips the CTA tiles strictly above the diagonal (the consumers read the
// lower triangle); per-split partials go to a workspace summed in fixed order (deterministic split-K).
constexpr int GBM = 128, GBN = 128, GBK = 16, GST = 4;
constexpr int GLA = 132, GLB = 20;
constexpr int GTHREADS = 256;
constexpr int big_stage_doubles(bool kmajor_a, bool kmajor_b) {
    return (kmajor_a ? GBK * GLA : GBM * GLB) + (kmajor_b ? GBK * GLA : GBN * GLB);
}
template <bool TA, bool TB>
constexpr size_t big_smem() { return (size_t)GST * big_stage_doubles(!TA, TB) * sizeof(double); }

__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(bytes) : "memory");
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(GTHREADS, 1)
dgemm_big_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                 int64_t k_per_split, double* __restrict__ work, int lower_only, int bx0, int by0) {
    constexpr bool KA = !TA;  // A staged k-major ([k][m])
    constexpr bool KB = TB;   // B staged k-major ([k][n])
    constexpr int SA_D = KA ? GBK * GLA : GBM * GLB;
    constexpr int SB_D = KB ? GBK * GLA : GBN * GLB;
    // bx0: first block row of this launch (a product launched in block-row pieces, dgemm_rows)
    const int64_t m0 = ((int64_t)blockIdx.x + bx0) * GBM, n0 = ((int64_t)blockIdx.y + by0) * GBN;
    if (lower_only && n0 > m0 + GBM - 1) return;
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double gsm[];
    const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
    const int64_t kend = min(K, kbeg + k_per_split);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;
    double* As0 = gsm;
    double* Bs0 = gsm + GST * SA_D;
    // 1024 16-byte chunks per operand per stage, 4 per thread: k-major c -> (k = c / 64, pair = c % 64),
    // row-major c -> (row = c / 8, k pair = c % 8)
    auto issue = [&](int64_t k0, int stage) {
        double* As = As0 + stage * SA_D;
        double* Bs = Bs0 + stage * SB_D;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = t + GTHREADS * u;
            if (KA) {
                const int kk = c >> 6, mm = (c & 63) * 2;
                const int64_t gk = k0 + kk, gm = m0 + mm;
                int bytes = 0;
                if (gk < kend) bytes = gm + 1 < M ? 16 : (gm < M ? 8 : 0);
                cp16(As + kk * GLA + mm, bytes ? A + gm + gk * lda : A, bytes);
            } else {
                const int mm = c >> 3, kk = (c & 7) * 2;
                const int64_t gm = m0 + mm, gk = k0 + kk;
                int bytes = 0;
                if (gm < M) bytes = gk + 1 < kend ? 16 : (gk < kend ? 8 : 0);
                cp16(As + mm * GLB + kk, bytes ? A + gk + gm * lda : A, bytes);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = t + GTHREADS * u;
            if (KB) {
                const int kk = c >> 6, nn = (c & 63) * 2;
                const int64_t gk = k0 + kk, gn = n0 + nn;
                int bytes = 0;
                if (gk < kend) bytes = gn + 1 < N ? 16 : (gn < N ? 8 : 0);
                cp16(Bs + kk * GLA + nn, bytes ? B + gn + gk * ldb : B, bytes);
            } else {
                const int nn = c >> 3, kk = (c & 7) * 2;
                const int64_t gn = n0 + nn, gk = k0 + kk;
                int bytes = 0;
                if (gn < N) bytes = gk + 1 < kend ? 16 : (gk < kend ? 8 : 0);
                cp16(Bs + nn * GLB + kk, bytes ? B + gk + gn * ldb : B, bytes);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int64_t ntiles = (kend - kbeg + GBK - 1) / GBK;
#pragma unroll
    for (int s = 0; s < GST - 1; ++s) {
        if (s < ntiles) issue(kbeg + s * GBK, s);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const int fr = lane >> 2, fk = lane & 3;
    for (int64_t it = 0; it < ntiles; ++it) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(GST - 2) : "memory");
        __syncthreads();
        const int64_t nx = it + GST - 1;
        if (nx < ntiles) issue(kbeg + nx * GBK, (int)(nx % GST));
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        const int stage = (int)(it % GST);
        const double* As = As0 + stage * SA_D + (KA ? wm + fr : (wm + fr) * GLB);
        const double* Bs = Bs0 + stage * SB_D + (KB ? wn + fr : (wn + fr) * GLB);
#pragma unroll
        for (int kk = 0; kk < GBK; kk += 4) {
            double af[8], bf[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) af[i] = KA ? As[(kk + fk) * GLA + i * 8] : As[i * 8 * GLB + kk + fk];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = KB ? Bs[(kk + fk) * GLA + j * 8] : Bs[j * 8 * GLB + kk + fk];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gm = m0 + wm + i * 8 + fr;
                const int64_t gn = n0 + wn + j * 8 + 2 * fk + h;
                if (gm >= M || gn >= N) continue;
                const double v = acc[i][j][h];
                if (work) {
                    work[(int64_t)blockIdx.z * M * N + gm + gn * M] = v;
                } else {
                    double out = alpha * v;
                    if (beta != 0.0) out += beta * C[gm + gn * ldc];
                    C[gm + gn * ldc] = out;
                }
            }
}

// C = alpha * sum_z work[z] + beta * C, splits summed in fixed order
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const double* __restrict__ work, double alpha,
                                     double beta, double* __restrict__ C, int64_t ldc, int lower_only) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t total = M * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gm = e % M, gn = e / M;
        if (lower_only && (gn / BN) * BN > (gm / BM) * BM + BM - 1) continue;
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += work[(int64_t)z * total + e];
        double out = alpha * s;
        if (beta != 0.0) out += beta * C[gm + gn * ldc];
        C[gm + gn * ldc] = out;
    }
}
}  // namespace

// the 128x128 cp.async kernel: enough work per tile and even leading dimensions (16-byte chunks along the
// contiguous index of both operands; the base pointers are checked in dgemm)
bool dgemm_use_big(bool transA, bool transB, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                   bool lower_only) {
    (void)transA;
    (void)transB;
    (void)lower_only;
    return M >= 256 && N >= 128 && K >= 1024 && lda % 2 == 0 && ldb % 2 == 0;
}
// ... and its 16-byte cp.async loads need 16-byte aligned operand base pointers as well
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int dgemm_pick_splitk(int64_t M, int64_t N, int64_t K, int num_sms, bool transA, bool transB, bool lower_only) {
    if (dgemm_use_big(transA, transB, M, N, K, M + (M & 1), 2, lower_only)) {
        // one CTA per SM: the split count whose last wave is fullest (>= 1024 rows of K per split)
        const int64_t tm = ceil_div(M, GBM), tn = ceil_div(N, GBN);
        int64_t tiles = tm * tn;
        if (lower_only) {  // tiles on or below the diagonal
            tiles = 0;
            for (int64_t bm = 0; bm < tm; ++bm) tiles += std::min<int64_t>(tn, (bm * GBM + GBM - 1) / GBN + 1);
        }
        int best = 1;
        double best_eff = 0.0;
        // workspace (s partial M x N products) kept within 1 GiB
        const int smax = (int)std::max<int64_t>(1, std::min<int64_t>(32, (int64_t)(1ll << 30) / (8 * M * N)));
        for (int s = 1; s <= smax && K / s >= 1024; ++s) {
            const int64_t ctas = tiles * s;
            const double eff = (double)ctas / (double)(ceil_div(ctas, num_sms) * num_sms);
            if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
        }
        return best;
    }
    // small tile counts (the k x k products of the factor phase) split K down to IHS_SPLITK_MIN_K per split
    static const int64_t min_k = [] {
        const char* e = std::getenv("IHS_SPLITK_MIN_K");
        return e ? std::max<int64_t>(16, std::atoll(e)) : int64_t{128};
    }();
    const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
    const int64_t want = (int64_t)num_sms * 4;
    int s = 1;
    while (tiles * s < want && K / (s * 2) >= min_k) s *= 2;
    return s;
}

// C_i = alpha op(A_i) op(B_i) + beta C_i for i < batch, X_i = X + i sX (the 64x64 DMMA kernel, one launch)
void dgemm_batched(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                   int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta, double* C, int64_t ldc,
                   int64_t sC, int batch, cudaStream_t st) {
    if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) fail(IHS_INTERNAL_ERROR, "dgemm_batched: empty product");
    if (sC == 0) fail(IHS_INTERNAL_ERROR, "dgemm_batched: output stride must be nonzero");
    const dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)batch);
    const int64_t kps = ceil_div(K, BK) * BK;
#define IHS_BATCHED(TA_, TB_)                                                                                    \
    LAUNCH_PDL((dgemm_kernel<TA_, TB_>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0, kps, \
               (double*)nullptr, sA, sB, sC)
    if (!transA && !transB) IHS_BATCHED(false, false);
    else if (transA && !transB) IHS_BATCHED(true, false);
    else if (!transA && transB) IHS_BATCHED(false, true);
    else IHS_BATCHED(true, true);
#undef IHS_BATCHED
}

void dgemm(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
           const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower_only, int splitk,
           double* d_work, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) {
        // C = beta * C
        splitk = 1;
    }
    if (splitk < 1) splitk = 1;
    // the 128x128 tiles need enough CTAs to fill the GPU (the factor phase's recursive products at k/2..k/8
    // without split-K would launch 16-64 of them); small grids stay on the 64x64 kernel
    const bool big = dgemm_use_big(transA, transB, M, N, K, lda, ldb, lower_only) && aligned16(A) && aligned16(B) &&
                     ceil_div(M, GBM) * ceil_div(N, GBN) * std::max(splitk, 1) >= 96;
    int64_t kps = ceil_div(std::max<int64_t>(K, 1), splitk);
    kps = ceil_div(kps, BK) * BK;
    const int splits = (int)std::max<int64_t>(1, ceil_div(std::max<int64_t>(K, 1), kps));
    dim3 grid((unsigned)ceil_div(M, big ? GBM : BM), (unsigned)ceil_div(N, big ? GBN : BN), (unsigned)splits);
    double* work = splits > 1 ? d_work : nullptr;
    if (splits > 1 && !d_work) fail(IHS_INTERNAL_ERROR, "dgemm: split-K without workspace");
    if (K <= 0) {
        // no products: run the reduce with zero splits semantics via a 1-split pass of zeros
        const int64_t total = M * N;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 8);
        LAUNCH_PDL(splitk_reduce_kernel, blocks, 256, 0, st, M, N, 0, (const double*)nullptr, alpha, beta, C, ldc,
               (int)lower_only);
        return;
    }
#define IHS_BIG(TA_, TB_)                                                                                       \
    do {                                                                                                        \
        IHS_SMEM_ATTR((dgemm_big_kernel<TA_, TB_>), (int)(big_smem<TA_, TB_>()));                               \
        LAUNCH_PDL((dgemm_big_kernel<TA_, TB_>), grid, GTHREADS, (big_smem<TA_, TB_>()), st, M, N, K, alpha, A, lda, B,\
                   ldb, beta, C, ldc, kps, work, (int)lower_only, 0, 0);                                        \
    } while (0)
    if (big && !transA && !transB) IHS_BIG(false, false);
    else if (big && transA && !transB) IHS_BIG(true, false);
    else if (big && !transA && transB) IHS_BIG(false, true);
    else if (big) IHS_BIG(true, true);
#undef IHS_BIG
    else if (!transA && !transB)
        LAUNCH_PDL((dgemm_kernel<false, false>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work, (int64_t)0, (int64_t)0, (int64_t)0);
    else if (transA && !transB)
        LAUNCH_PDL((dgemm_kernel<true, false>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work, (int64_t)0, (int64_t)0, (int64_t)0);
    else if (!transA && transB)
        LAUNCH_PDL((dgemm_kernel<false, true>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work, (int64_t)0, (int64_t)0, (int64_t)0);
    else
        LAUNCH_PDL((dgemm_kernel<true, true>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work, (int64_t)0, (int64_t)0, (int64_t)0);
    if (work) {
        const int64_t total = M * N;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 8);
        LAUNCH_PDL(splitk_reduce_kernel, blocks, 256, 0, st, M, N, splits, work, alpha, beta, C, ldc, (int)lower_only);
    }
}

// The same product as dgemm(...) on the 128x128 kernel, launched in pieces: phase 0 runs the output block rows
// covering rows [row0, row1) (row0 a multiple of dgemm_row_block()) without the split-K reduction, phase 1 runs only
// the reduction. Every tile is computed by the same CTA code over the same K partition whatever the pieces, so
// pieces + reduction give the bytes of the single call (the sketched Gram accumulated block row by block row as
// SA's columns arrive). Returns false, doing nothing, when dgemm would not take the 128x128 kernel.
int64_t dgemm_row_block() { return GBM; }
static bool dgemm_window(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower_only,
                         int splitk, double* d_work, cudaStream_t st, int64_t row0, int64_t row1, int64_t col0,
                         int64_t col1, int phase) {
    if (M <= 0 || N <= 0 || K <= 0) return false;
    if (splitk < 1) splitk = 1;
    const bool big = dgemm_use_big(transA, transB, M, N, K, lda, ldb, lower_only) && aligned16(A) && aligned16(B) &&
                     ceil_div(M, GBM) * ceil_div(N, GBN) * std::max(splitk, 1) >= 96;
    if (!big) return false;
    int64_t kps = ceil_div(K, splitk);
    kps = ceil_div(kps, BK) * BK;
    const int splits = (int)std::max<int64_t>(1, ceil_div(K, kps));
    double* work = splits > 1 ? d_work : nullptr;
    if (splits > 1 && !d_work) fail(IHS_INTERNAL_ERROR, "dgemm_rows: split-K without workspace");
    if (phase == 1) {
        if (work) {
            const int64_t total = M * N;
            const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 8);
            LAUNCH_PDL(splitk_reduce_kernel, blocks, 256, 0, st, M, N, splits, work, alpha, beta, C, ldc,
                       (int)lower_only);
        }
        return true;
    }
    if (row0 % GBM != 0 || row1 <= row0 || row1 > M || col0 % GBN != 0 || col1 <= col0 || col1 > N)
        fail(IHS_INTERNAL_ERROR, "dgemm window: bad tile window");
    const int bx0 = (int)(row0 / GBM), by0 = (int)(col0 / GBN);
    dim3 grid((unsigned)(ceil_div(row1, GBM) - bx0), (unsigned)(ceil_div(col1, GBN) - by0), (unsigned)splits);
#define IHS_BIGW(TA_, TB_)                                                                                      \
    do {                                                                                                        \
        IHS_SMEM_ATTR((dgemm_big_kernel<TA_, TB_>), (int)(big_smem<TA_, TB_>()));                               \
        LAUNCH_PDL((dgemm_big_kernel<TA_, TB_>), grid, GTHREADS, (big_smem<TA_, TB_>()), st, M, N, K, alpha, A, lda, B,\
                   ldb, beta, C, ldc, kps, work, (int)lower_only, bx0, by0);                                    \
    } while (0)
    if (!transA && !transB) IHS_BIGW(false, false);
    else if (transA && !transB) IHS_BIGW(true, false);
    else if (!transA && transB) IHS_BIGW(false, true);
    else IHS_BIGW(true, true);
#undef IHS_BIGW
    return true;
}

bool dgemm_rows(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower_only, int splitk,
                double* d_work, cudaStream_t st, int64_t row0, int64_t row1, int phase) {
    return dgemm_window(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only, splitk, d_work, st,
                        row0, row1, 0, N, phase);
}
// ... and in block-column pieces (columns [col0, col1), col0 a multiple of dgemm_col_block()): S*A over the columns
// of an A that is still arriving
int64_t dgemm_col_block() { return GBN; }
bool dgemm_cols(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splitk, double* d_work,
                cudaStream_t st, int64_t col0, int64_t col1, int phase) {
    return dgemm_window(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, false, splitk, d_work, st, 0, M,
                        col0, col1, phase);
}

}  // namespace ihs_b200
