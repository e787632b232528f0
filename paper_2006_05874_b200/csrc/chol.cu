// chol.cu — blocked Cholesky of the sketched Hessian and its triangular solves.
//
// Reference: SketchedSystem ctor (sketched_system.hpp:69-84) runs Eigen's
// LLT on the m x m Woodbury inner matrix or the d x d regularized Gram, and
// throws NumericalBreakdown when it fails (:82-83); solve (:40-49) applies
// llt.solve. Here: right-looking blocked LLT (NB = 64): a one-CTA panel
// factorization in shared memory, a row-parallel TRSM for the panel below,
// and the trailing update on the DMMA GEMM (gemm_f64.cu). The strict upper
// triangle is then overwritten with L^T so both triangular sweeps of a solve
// read their operand coalesced. A non-positive or non-finite pivot sets
// *info = column+1 (the caller raises NumericalBreakdown).
#include "common.cuh"

namespace ihs_b200 {

namespace {
constexpr int NB = 64;

// Unblocked LLT of the nb x nb diagonal block at (k,k), in shared memory.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ H, int64_t n, int64_t k, int nb,
                                                         int* __restrict__ info) {
    __shared__ double a[NB][NB + 1];
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        a[i][j] = (i >= j) ? H[(k + i) + (k + j) * n] : 0.0;
    }
    __syncthreads();
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        // pivot
        if (threadIdx.x == 0) {
            const double s = a[j][j];
            if (!(s > 0.0) || !isfinite(s)) {
                if (!bad) { bad = 1; atomicCAS(info, 0, (int)(k + j + 1)); }
                a[j][j] = 1.0;  // keep going with a harmless pivot; result is flagged
            } else {
                a[j][j] = sqrt(s);
            }
        }
        __syncthreads();
        const double ljj = a[j][j];
        for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) a[i][j] = a[i][j] / ljj;
        __syncthreads();
        // rank-1 update of the trailing lower block
        const int rem = nb - j - 1;
        for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
            const int ii = j + 1 + e % rem, jj = j + 1 + e / rem;
            if (ii >= jj) a[ii][jj] -= a[ii][j] * a[jj][j];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        if (i >= j) H[(k + i) + (k + j) * n] = a[i][j];
    }
}

// L21 = A21 * L11^{-T}: each thread solves one row x * L11^T = a.
__global__ void __launch_bounds__(128) trsm_panel_kernel(double* __restrict__ H, int64_t n, int64_t k, int nb) {
    __shared__ double l[NB][NB + 1];
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        l[i][j] = (i >= j) ? H[(k + i) + (k + j) * n] : 0.0;
    }
    __syncthreads();
    const int64_t row = k + nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = (c < nb) ? H[row + (k + c) * n] : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        if (c < nb) {
            double s = x[c];
#pragma unroll
            for (int q = 0; q < c; ++q) s -= x[q] * l[c][q];
            x[c] = s / l[c][c];
        }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
        if (c < nb) H[row + (k + c) * n] = x[c];
}

// strict upper triangle <- L^T (H[i + j n] = H[j + i n] for i < j)
__global__ void mirror_upper_kernel(double* __restrict__ H, int64_t n) {
    // 32x32 tiles through shared memory for coalescing on both sides
    __shared__ double tile[32][33];
    const int64_t bi = blockIdx.x, bj = blockIdx.y;
    if (bi > bj) return;  // upper tiles only (tile row <= tile col)
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    // tile[a][b] = L[bj*32 + a, bi*32 + b]  (coalesced over a)
    for (int r = ty; r < 32; r += 8) {
        const int64_t src_row = bj * 32 + tx, src_col = bi * 32 + r;
        tile[tx][r] = (src_row < n && src_col < n) ? H[src_row + src_col * n] : 0.0;
    }
    __syncthreads();
    // destination (i, j) = (bi*32 + tx, bj*32 + r), i < j, gets L[j, i] = tile[r][tx]
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + tx, j = bj * 32 + r;
        if (i < n && j < n && i < j) H[i + j * n] = tile[r][tx];
    }
}

// Triangular solves with the mirrored factor, single CTA, nrhs in {1, 2}.
// Forward: L y = r ; backward: L^T z = y, blocked by 32 (warp-sized diagonal solves).
__global__ void __launch_bounds__(512) chol_solve_kernel(const double* __restrict__ Lf, int64_t n,
                                                         double* __restrict__ R, int nrhs) {
    extern __shared__ double v[];  // nrhs * n
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t e = tid; e < n * nrhs; e += blockDim.x) v[e] = R[e];
    __syncthreads();
    // forward
    for (int64_t kb = 0; kb < n; kb += 32) {
        const int bs = (int)imin64(32, n - kb);
        if (warp < nrhs) {
            double* y = v + (int64_t)warp * n;
            double r = (lane < bs) ? y[kb + lane] : 0.0;
            for (int c = 0; c < bs; ++c) {
                double yc = 0.0;
                if (lane == c) yc = r / Lf[(kb + c) + (kb + c) * n];
                yc = __shfl_sync(0xffffffffu, yc, c);
                if (lane > c && lane < bs) r -= Lf[(kb + lane) + (kb + c) * n] * yc;
                if (lane == c) r = yc;
            }
            if (lane < bs) y[kb + lane] = r;
        }
        __syncthreads();
        for (int64_t i = kb + bs + tid; i < n; i += blockDim.x) {
            for (int q = 0; q < nrhs; ++q) {
                double* y = v + (int64_t)q * n;
                double s = 0.0;
                for (int c = 0; c < bs; ++c) s += Lf[i + (kb + c) * n] * y[kb + c];
                y[i] -= s;
            }
        }
        __syncthreads();
    }
    // backward with U = L^T stored in the strict upper triangle (diag from L)
    const int64_t nblk = (n + 31) / 32;
    for (int64_t b = nblk - 1; b >= 0; --b) {
        const int64_t kb = b * 32;
        const int bs = (int)imin64(32, n - kb);
        if (warp < nrhs) {
            double* y = v + (int64_t)warp * n;
            double r = (lane < bs) ? y[kb + lane] : 0.0;
            for (int c = bs - 1; c >= 0; --c) {
                double zc = 0.0;
                if (lane == c) zc = r / Lf[(kb + c) + (kb + c) * n];
                zc = __shfl_sync(0xffffffffu, zc, c);
                // U[kb+lane, kb+c] for lane < c lives in the upper triangle
                if (lane < c) r -= Lf[(kb + lane) + (kb + c) * n] * zc;
                if (lane == c) r = zc;
            }
            if (lane < bs) y[kb + lane] = r;
        }
        __syncthreads();
        for (int64_t i = tid; i < kb; i += blockDim.x) {
            for (int q = 0; q < nrhs; ++q) {
                double* y = v + (int64_t)q * n;
                double s = 0.0;
                for (int c = 0; c < bs; ++c) s += Lf[i + (kb + c) * n] * y[kb + c];
                y[i] -= s;
            }
        }
        __syncthreads();
    }
    for (int64_t e = tid; e < n * nrhs; e += blockDim.x) R[e] = v[e];
}
}  // namespace

void cholesky_factor(double* d_H, int64_t n, double* d_work, int* d_info, int num_sms, cudaStream_t st) {
    (void)d_work;
    (void)num_sms;
    CUDA_CHECK(cudaMemsetAsync(d_info, 0, sizeof(int), st));
    for (int64_t k = 0; k < n; k += NB) {
        const int nb = (int)std::min<int64_t>(NB, n - k);
        LAUNCH(potrf_diag_kernel, 1, 256, 0, st, d_H, n, k, nb, d_info);
        const int64_t rest = n - k - nb;
        if (rest > 0) {
            LAUNCH(trsm_panel_kernel, (unsigned)ceil_div(rest, 128), 128, 0, st, d_H, n, k, nb);
            // A22 -= L21 L21^T (lower)
            double* L21 = d_H + (k + nb) + k * n;
            double* A22 = d_H + (k + nb) + (k + nb) * n;
            dgemm(false, true, rest, rest, nb, -1.0, L21, n, L21, n, 1.0, A22, n, true, 1, nullptr, st);
        }
    }
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
    LAUNCH(mirror_upper_kernel, grid, dim3(32, 8), 0, st, d_H, n);
}

void cholesky_solve(const double* d_L, int64_t n, double* d_R, int nrhs, cudaStream_t st) {
    const size_t smem = (size_t)n * nrhs * sizeof(double);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    if (smem > 200 * 1024) fail(IHS_INVALID_INPUT, "cholesky_solve: system too large for the single-CTA solver");
    LAUNCH(chol_solve_kernel, 1, 512, smem, st, d_L, n, d_R, nrhs);
}

}  // namespace ihs_b200
