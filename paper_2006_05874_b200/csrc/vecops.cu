// vecops.cu — small d-vector kernels of the adaptive loop.
//
// Candidate updates follow solver.hpp:182 and :190 coefficient-wise with the
// same operation tree and no FMA contraction; the decrement dot products
// (sketched_system.hpp:95-101) use one CTA with a fixed reduction order so
// repeated solves are bit-identical.
#include "common.cuh"

#include <mutex>

namespace ihs_b200 {

namespace {
__global__ void candidates_kernel(const double* __restrict__ x, const double* __restrict__ xprev,
                                  const double* __restrict__ gt, double mu_p, double beta_p, double mu_gd, int64_t d,
                                  double* __restrict__ xp, double* __restrict__ xg) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i], gi = gt[i];
        if (xp) xp[i] = __dadd_rn(__dsub_rn(xi, __dmul_rn(mu_p, gi)), __dmul_rn(beta_p, __dsub_rn(xi, xprev[i])));
        if (xg) xg[i] = __dsub_rn(xi, __dmul_rn(mu_gd, gi));
    }
}

__global__ void fixed_step_kernel(const double* __restrict__ x, const double* __restrict__ xprev,
                                  const double* __restrict__ step, double mu, double beta, int64_t d,
                                  double* __restrict__ xn) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i];
        xn[i] = __dadd_rn(__dsub_rn(xi, __dmul_rn(mu, step[i])), __dmul_rn(beta, __dsub_rn(xi, xprev[i])));
    }
}

__global__ void __launch_bounds__(1024) decrement_dots_kernel(const double* __restrict__ g,
                                                              const double* __restrict__ gt, int64_t d, int nrhs,
                                                              double* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double s1[1024], s2[1024];
    for (int q = 0; q < nrhs; ++q) {
        double a = 0.0, c = 0.0;
        for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
            const double gi = g[q * d + i];
            a = fma(gi, gt[q * d + i], a);
            c = fma(gi, gi, c);
        }
        s1[threadIdx.x] = a;
        s2[threadIdx.x] = c;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) {
                s1[threadIdx.x] += s1[threadIdx.x + w];
                s2[threadIdx.x] += s2[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            out[2 * q] = s1[0];
            out[2 * q + 1] = s2[0];
        }
        __syncthreads();
    }
}

// y[:,q] = A (M x N, lda) x[:,q]
__global__ void gemv_n_kernel(const double* __restrict__ A, int64_t M, int64_t N, int64_t lda,
                              const double* __restrict__ x, int nrhs, int64_t ldx, double* __restrict__ y,
                              int64_t ldy) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        for (int q = 0; q < nrhs; ++q) {
            double s = 0.0;
            for (int64_t j = 0; j < N; ++j) s = fma(A[i + j * lda], x[q * ldx + j], s);
            y[q * ldy + i] = s;
        }
    }
}

// Tiled y = A x: CTA = 64 rows x 64 columns, 256 threads (64 rows x 4 column
// interleaves of 16 columns); partials per column chunk go to `part`; the last
// CTA of each row block (per-row-block arrival counter) sums the chunks in
// chunk order, so the result is deterministic and one launch suffices. The
// counters are reset by that last CTA for the next launch.
constexpr int GV_ROWS = 32, GV_COLS = 64, GV_G = 256 / GV_ROWS;  // 8 column interleaves
__global__ void __launch_bounds__(256) gemv_tiled_kernel(const double* __restrict__ A, int64_t M, int64_t N,
                                                         int64_t lda, const double* __restrict__ x, int nrhs,
                                                         int64_t ldx, double* __restrict__ part,
                                                         unsigned* __restrict__ arrivals, double* __restrict__ y,
                                                         int64_t ldy, double* __restrict__ dots) {
    pdl_wait();  // x is the previous kernel's output when launched programmatically
    const int64_t r0 = (int64_t)blockIdx.x * GV_ROWS, c0 = (int64_t)blockIdx.y * GV_COLS;
    const int64_t c1 = c0 + GV_COLS < N ? c0 + GV_COLS : N;
    __shared__ double xs[2][GV_COLS];
    __shared__ double red[GV_G][2][GV_ROWS];
    __shared__ unsigned last;
    for (int e = threadIdx.x; e < (int)(c1 - c0); e += blockDim.x)
        for (int q = 0; q < nrhs; ++q) xs[q][e] = x[q * ldx + c0 + e];
    __syncthreads();
    const int r = threadIdx.x % GV_ROWS, qg = threadIdx.x / GV_ROWS;
    const int64_t row = r0 + r;
    double acc[2] = {0.0, 0.0};
    if (row < M) {
#pragma unroll 4
        for (int64_t j = c0 + qg; j < c1; j += GV_G) {
            const double a = A[row + j * lda];
            acc[0] = fma(a, xs[0][j - c0], acc[0]);
            if (nrhs > 1) acc[1] = fma(a, xs[1][j - c0], acc[1]);
        }
    }
    red[qg][0][r] = acc[0];
    red[qg][1][r] = acc[1];
    __syncthreads();
    if (threadIdx.x < GV_ROWS && row < M)
        for (int q = 0; q < nrhs; ++q) {
            double sum = 0.0;
#pragma unroll
            for (int g = 0; g < GV_G; ++g) sum += red[g][q][r];
            part[((int64_t)blockIdx.y * nrhs + q) * M + row] = sum;
        }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(arrivals + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < GV_ROWS && row < M)
        for (int q = 0; q < nrhs; ++q) {
            double sum = 0.0;
            for (unsigned c = 0; c < gridDim.y; ++c) sum += __ldcg(part + ((int64_t)c * nrhs + q) * M + row);
            y[q * ldy + row] = sum;
        }
    if (threadIdx.x == 0) arrivals[blockIdx.x] = 0u;
    if (dots == nullptr) return;
    // decrement dots (sketched_system.hpp:95-101) by the last row block to finish: x . y and x . x per
    // right-hand side over all M = N rows, fixed-order tree -> deterministic
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(arrivals + gridDim.x, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ double s1[256], s2[256];
    for (int q = 0; q < nrhs; ++q) {
        double a = 0.0, c = 0.0;
        for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
            const double gi = x[q * ldx + i];
            a = fma(gi, __ldcg(y + q * ldy + i), a);
            c = fma(gi, gi, c);
        }
        s1[threadIdx.x] = a;
        s2[threadIdx.x] = c;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) {
                s1[threadIdx.x] += s1[threadIdx.x + w];
                s2[threadIdx.x] += s2[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            dots[2 * q] = s1[0];
            dots[2 * q + 1] = s2[0];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) arrivals[gridDim.x] = 0u;
}

// y = H x for a symmetric k x k H (column-major; H_S^{-1} of the direct-Gram system): y_i = column i . x,
// one warp per output over a contiguous column, no cross-CTA partial sums. With dots != nullptr the
// decrement dots x.y and x.x per right-hand side are finished by the last CTA from per-CTA partials in
// CTA order (deterministic). part: 4 * gridDim.x doubles; counter: zero before the launch, reset after.
// work (symv_col): gemv_tiled_work_doubles(k, k) + 8, reset by gemv_tiled_reset.
constexpr int SV_W = 8;  // outputs (warps) per CTA
__global__ void __launch_bounds__(32 * SV_W) symv_col_kernel(const double* __restrict__ H, int64_t k,
                                                             const double* __restrict__ x, int nrhs, int64_t ldx,
                                                             double* __restrict__ y, int64_t ldy,
                                                             double* __restrict__ dots, double* __restrict__ part,
                                                             unsigned* __restrict__ counter) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double xs[];  // nrhs x k
    __shared__ double pd[SV_W][4];
    __shared__ unsigned last;
    for (int64_t e = threadIdx.x; e < (int64_t)nrhs * k; e += blockDim.x) {
        const int64_t q = e / k, t = e % k;
        xs[e] = x[q * ldx + t];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * SV_W + w;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (i < k) {
        const double* col = H + i * k;
        int64_t t = lane;
        // eight column loads in flight per lane before any is consumed (one L2 round trip per 256 rows instead
        // of one per 64)
        for (; t + 224 < k; t += 256) {
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldcg(col + t + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acc[0][u & 1] = fma(a[u], xs[t + 32 * u], acc[0][u & 1]);
                if (nrhs > 1) acc[1][u & 1] = fma(a[u], xs[k + t + 32 * u], acc[1][u & 1]);
            }
        }
        for (; t + 32 < k; t += 64) {
            const double a0 = col[t], a1 = col[t + 32];
            acc[0][0] = fma(a0, xs[t], acc[0][0]);
            acc[0][1] = fma(a1, xs[t + 32], acc[0][1]);
            if (nrhs > 1) {
                acc[1][0] = fma(a0, xs[k + t], acc[1][0]);
                acc[1][1] = fma(a1, xs[k + t + 32], acc[1][1]);
            }
        }
        if (t < k) {
            const double a0 = col[t];
            acc[0][0] = fma(a0, xs[t], acc[0][0]);
            if (nrhs > 1) acc[1][0] = fma(a0, xs[k + t], acc[1][0]);
        }
    }
    double yv[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        double v = acc[q][0] + acc[q][1];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        yv[q] = v;
    }
    if (lane == 0) {
        for (int q = 0; q < 4; ++q) pd[w][q] = 0.0;
        if (i < k)
            for (int q = 0; q < nrhs; ++q) {
                y[q * ldy + i] = yv[q];
                const double xi = xs[q * k + i];
                pd[w][2 * q] = xi * yv[q];
                pd[w][2 * q + 1] = xi * xi;
            }
    }
    if (dots == nullptr) return;
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int ww = 0; ww < SV_W; ++ww) s += pd[ww][threadIdx.x];
        part[(int64_t)blockIdx.x * 4 + threadIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < 2 * nrhs) {
        double s = 0.0;
        for (unsigned c = 0; c < gridDim.x; ++c) s += __ldcg(part + (int64_t)c * 4 + threadIdx.x);
        dots[threadIdx.x] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
}

// z[:,q] = (g[:,q] - SA^T w[:,q]) / nu2 ; one warp per column of SA
__global__ void woodbury_finish_kernel(const double* __restrict__ SA, int64_t m, int64_t d,
                                       const double* __restrict__ g, const double* __restrict__ w, double nu2,
                                       int nrhs, double* __restrict__ z) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = warp; j < d; j += nwarps) {
        for (int q = 0; q < nrhs; ++q) {
            double s = 0.0;
            for (int64_t i = lane; i < m; i += 32) s = fma(SA[i + j * m], w[q * m + i], s);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) z[q * d + j] = __ddiv_rn(__dsub_rn(g[q * d + j], s), nu2);
        }
    }
}

__global__ void add_scaled_kernel(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = y[i] + a * x[i];
}

__global__ void add_diag_kernel(double* __restrict__ H, int64_t n, double v) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        H[i + i * n] += v;
}

__global__ void check_finite_kernel(const double* __restrict__ v, int64_t count, int* __restrict__ flag) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) *flag = 1;
}

int blocks_for(int64_t n, int threads, int cap = 148 * 8) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap));
}
}  // namespace

void candidates(const double* x, const double* xprev, const double* gt, double mu_p, double beta_p, double mu_gd,
                int64_t d, double* xp, double* xg, cudaStream_t st) {
    LAUNCH_PDL(candidates_kernel, blocks_for(d, 256), 256, 0, st, x, xprev, gt, mu_p, beta_p, mu_gd, d, xp, xg);
}

void fixed_step(const double* x, const double* xprev, const double* step, double mu, double beta, int64_t d,
                double* xn, cudaStream_t st) {
    LAUNCH_PDL(fixed_step_kernel, blocks_for(d, 256), 256, 0, st, x, xprev, step, mu, beta, d, xn);
}

void decrement_dots(const double* g, const double* gt, int64_t d, int nrhs, double* out, cudaStream_t st) {
    LAUNCH_PDL(decrement_dots_kernel, 1, 1024, 0, st, g, gt, d, nrhs, out);
}

void gemv_n(const double* A, int64_t M, int64_t N, int64_t lda, const double* x, int nrhs, int64_t ldx, double* y,
            int64_t ldy, cudaStream_t st) {
    LAUNCH_PDL(gemv_n_kernel, blocks_for(M, 128), 128, 0, st, A, M, N, lda, x, nrhs, ldx, y, ldy);
}

// partials (nchunks x 2 x M) followed by the per-row-block arrival counters
// (zeroed here once; the kernel leaves them zero)
size_t gemv_tiled_work_doubles(int64_t M, int64_t N) {
    return (size_t)ceil_div(N, GV_COLS) * 2 * (size_t)M + (size_t)ceil_div(M, GV_ROWS) + 8;
}

void gemv_tiled(const double* A, int64_t M, int64_t N, int64_t lda, const double* x, int nrhs, int64_t ldx, double* y,
                int64_t ldy, double* work, cudaStream_t st, double* dots) {
    dim3 grid((unsigned)ceil_div(M, GV_ROWS), (unsigned)ceil_div(N, GV_COLS));
    unsigned* arrivals = reinterpret_cast<unsigned*>(work + (size_t)grid.y * 2 * (size_t)M);
    LAUNCH_PDL(gemv_tiled_kernel, grid, dim3(256), 0, st, A, M, N, lda, x, nrhs, ldx, work, arrivals, y, ldy, dots);
}

// y = H x, H symmetric k x k (column-major); work: gemv_tiled_work_doubles(k, k) (its counter tail is
// reset by gemv_tiled_reset, and this kernel leaves it zero)
void symv_col(const double* H, int64_t k, const double* x, int nrhs, int64_t ldx, double* y, int64_t ldy,
              double* work, cudaStream_t st, double* dots) {
    // the counter sits in the zeroed tail of the gemv_tiled layout, past gemv_tiled's own arrival counters;
    // the per-CTA partials at the front (or, for k <= 2 where the front is shorter, in the 8 spare doubles
    // the factorization allocates after the tail)
    const size_t front = (size_t)ceil_div(k, GV_COLS) * 2 * (size_t)k;
    double* tail = work + front;
    unsigned* counter = reinterpret_cast<unsigned*>(tail + ceil_div(k, GV_ROWS) + 4);
    const unsigned grid = (unsigned)ceil_div(k, SV_W);
    double* part = (size_t)4 * grid <= front ? work : tail + ceil_div(k, GV_ROWS) + 8;
    const size_t smem = (size_t)nrhs * k * sizeof(double);
    if (smem > 48 * 1024) {  // opt in per device, raised to the largest request seen on that device
        static std::mutex mu;
        static int attr_bytes[64] = {};
        int dev = 0;
        CUDA_CHECK(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        if ((int)smem > attr_bytes[dev & 63]) {
            CUDA_CHECK(cudaFuncSetAttribute(symv_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_bytes[dev & 63] = (int)smem;
        }
    }
    LAUNCH_PDL(symv_col_kernel, dim3(grid), dim3(32 * SV_W), smem, st, H, k, x, nrhs, ldx, y, ldy, dots, part,
               counter);
}

void gemv_tiled_reset(double* work, int64_t M, int64_t N, cudaStream_t st) {
    const size_t off = (size_t)ceil_div(N, GV_COLS) * 2 * (size_t)M;
    CUDA_CHECK(cudaMemsetAsync(work + off, 0, ((size_t)ceil_div(M, GV_ROWS) + 8) * sizeof(double), st));
}

__global__ void tril_copy_kernel(const double* __restrict__ W, int64_t k, double* __restrict__ Wl) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t total = k * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % k, j = e / k;
        Wl[e] = i >= j ? W[e] : 0.0;
    }
}

void tril_copy(const double* W, int64_t k, double* Wl, cudaStream_t st) {
    LAUNCH_PDL(tril_copy_kernel, blocks_for(k * k, 256), 256, 0, st, W, k, Wl);
}

void woodbury_finish(const double* SA, int64_t m, int64_t d, const double* g, const double* w, double nu2, int nrhs,
                     double* z, cudaStream_t st) {
    LAUNCH_PDL(woodbury_finish_kernel, blocks_for(d * 32, 256), 256, 0, st, SA, m, d, g, w, nu2, nrhs, z);
}

void add_scaled(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
    LAUNCH_PDL(add_scaled_kernel, blocks_for(n, 256), 256, 0, st, y, x, a, n);
}

void add_diag(double* H, int64_t n, double v, cudaStream_t st) {
    LAUNCH_PDL(add_diag_kernel, blocks_for(n, 256), 256, 0, st, H, n, v);
}

void check_finite(const double* v, int64_t count, int* d_flag, cudaStream_t st) {
    LAUNCH_PDL(check_finite_kernel, blocks_for(count, 256), 256, 0, st, v, count, d_flag);
}

}  // namespace ihs_b200
