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
             int lower_only, int64_t k_per_split, double* __restrict__ work) {
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int64_t n0 = (int64_t)blockIdx.y * BN;
    if (lower_only && n0 > m0 + BM - 1) return;
    const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
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

// C = alpha * sum_z work[z] + beta * C, splits summed in fixed order
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const double* __restrict__ work, double alpha,
                                     double beta, double* __restrict__ C, int64_t ldc, int lower_only) {
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

int dgemm_pick_splitk(int64_t M, int64_t N, int64_t K, int num_sms) {
    const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
    const int64_t want = (int64_t)num_sms * 4;
    int s = 1;
    while (tiles * s < want && K / (s * 2) >= 512) s *= 2;
    return s;
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
    int64_t kps = ceil_div(std::max<int64_t>(K, 1), splitk);
    kps = ceil_div(kps, BK) * BK;
    const int splits = (int)std::max<int64_t>(1, ceil_div(std::max<int64_t>(K, 1), kps));
    dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)splits);
    double* work = splits > 1 ? d_work : nullptr;
    if (splits > 1 && !d_work) fail(IHS_INTERNAL_ERROR, "dgemm: split-K without workspace");
    if (K <= 0) {
        // no products: run the reduce with zero splits semantics via a 1-split pass of zeros
        const int64_t total = M * N;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 8);
        LAUNCH(splitk_reduce_kernel, blocks, 256, 0, st, M, N, 0, (const double*)nullptr, alpha, beta, C, ldc,
               (int)lower_only);
        return;
    }
    if (!transA && !transB)
        LAUNCH((dgemm_kernel<false, false>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work);
    else if (transA && !transB)
        LAUNCH((dgemm_kernel<true, false>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work);
    else if (!transA && transB)
        LAUNCH((dgemm_kernel<false, true>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work);
    else
        LAUNCH((dgemm_kernel<true, true>), grid, THREADS, 0, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
               (int)lower_only, kps, work);
    if (work) {
        const int64_t total = M * N;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 8);
        LAUNCH(splitk_reduce_kernel, blocks, 256, 0, st, M, N, splits, work, alpha, beta, C, ldc, (int)lower_only);
    }
}

}  // namespace ihs_b200
