// chol.cu — blocked Cholesky of the sketched Hessian and its triangular solves.
//
// Reference: SketchedSystem ctor (sketched_system.hpp:69-84) runs Eigen's
// LLT on the m x m Woodbury inner matrix or the d x d regularized Gram, and
// throws NumericalBreakdown when it fails (:82-83); solve (:40-49) applies
// llt.solve. Here: right-looking blocked LLT (NB = 64): a one-CTA panel
// factorization in shared memory, a row-parallel TRSM for the panel below,
// and the trailing update on the DMMA GEMM (gemm_f64.cu). A non-positive or
// non-finite pivot sets *info = column+1 (the caller raises
// NumericalBreakdown). The factor is then inverted once per sketch
// (recursive 2x2 blocking, DMMA GEMMs) into W = L^{-1} with W^T mirrored into
// the strict upper triangle, so every solve of the adaptive loop is two
// fully parallel, coalesced triangular mat-vecs instead of a latency-bound
// substitution.
#include "common.cuh"

#include <cstdlib>


namespace ihs_b200 {

namespace {
constexpr int NB = 64;
constexpr int TRSM_WARPS = 8;  // rows (warps) per CTA of the panel solves

// LLT of the nb x nb diagonal block at (k,k), in shared memory, blocked by 16 columns: warp 0 factors
// each 16 x 16 diagonal sub-block in registers (lane = row; the pivot and the column broadcast by
// shuffles, reciprocal square roots instead of sqrt + division, no CTA barrier per column), one thread
// per row solves the panel below against it, and all 256 threads apply the rank-16 trailing update.
// The serial part is 16 short column steps per sub-block instead of a barrier-separated step per column
// of the whole block. A non-positive or non-finite pivot sets *info = column + 1 (a harmless pivot is
// substituted so the kernel completes).
constexpr int PD_B = 16;
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ H, int64_t n, int64_t k, int nb,
                                                         int* __restrict__ info) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double a[NB][NB + 1];
    __shared__ double rdiag[PD_B];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < NB * NB; e += 256) {
        const int i = e % NB, jj = e / NB;
        a[i][jj] = (i < nb && jj < nb && i >= jj) ? H[(k + i) + (k + jj) * n] : 0.0;
    }
    __syncthreads();
    for (int kb = 0; kb < nb; kb += PD_B) {
        const int bs = nb - kb < PD_B ? nb - kb : PD_B;
        if (warp == 0) {
            // 1. the diagonal sub-block: lane i < bs holds row kb + i
            double r[PD_B];
#pragma unroll
            for (int q = 0; q < PD_B; ++q) r[q] = (lane < bs && q <= lane) ? a[kb + lane][kb + q] : 0.0;
#pragma unroll
            for (int j = 0; j < PD_B; ++j) {
                if (j < bs) {
                    double dj = __shfl_sync(0xffffffffu, r[j], j);
                    if (!(dj > 0.0) || !isfinite(dj)) {
                        if (lane == 0) atomicCAS(info, 0, (int)(k + kb + j + 1));
                        dj = 1.0;
                    }
                    const double rs = rsqrt(dj);
                    const double l = lane == j ? dj * rs : (lane > j ? r[j] * rs : 0.0);
                    r[j] = l;
                    if (lane == j) rdiag[j] = rs;  // 1 / l_jj for the panel solve
#pragma unroll
                    for (int q = j + 1; q < PD_B; ++q) {
                        const double lq = __shfl_sync(0xffffffffu, l, q);
                        if (lane >= q) r[q] = fma(-l, lq, r[q]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < PD_B; ++q)
                if (lane < bs && q <= lane) a[kb + lane][kb + q] = r[q];
        }
        __syncthreads();
        const int rows = nb - kb - bs;
        if (rows <= 0) break;
        // 2. the panel below: row i solves l_i,kb+j = (a_i,kb+j - sum_t<j l_i,kb+t l_kb+j,kb+t) / l_jj
        if (tid < rows) {
            const int i = kb + bs + tid;
            double x[PD_B];
#pragma unroll
            for (int j = 0; j < PD_B; ++j) x[j] = j < bs ? a[i][kb + j] : 0.0;
#pragma unroll
            for (int j = 0; j < PD_B; ++j) {
                if (j < bs) {
                    double s = x[j];
#pragma unroll
                    for (int t = 0; t < j; ++t) s = fma(-x[t], a[kb + j][kb + t], s);
                    x[j] = s * rdiag[j];
                }
            }
#pragma unroll
            for (int j = 0; j < PD_B; ++j)
                if (j < bs) a[i][kb + j] = x[j];
        }
        __syncthreads();
        // 3. trailing update of the lower part: A22 -= L21 L21^T (rank bs)
        const int r0 = kb + bs;
        for (int e = tid; e < rows * rows; e += 256) {
            const int ii = e % rows, jj = e / rows;
            if (ii < jj) continue;
            double s = a[r0 + ii][r0 + jj];
#pragma unroll
            for (int t = 0; t < PD_B; ++t)
                if (t < bs) s = fma(-a[r0 + ii][kb + t], a[r0 + jj][kb + t], s);
            a[r0 + ii][r0 + jj] = s;
        }
        __syncthreads();
    }
    for (int e = tid; e < NB * NB; e += 256) {
        const int i = e % NB, jj = e / NB;
        if (i < nb && jj < nb && i >= jj) H[(k + i) + (k + jj) * n] = a[i][jj];
    }
}

// L21 = A21 * L11^{-T}: one warp per row, lane c holds columns c and c+32 of
// the row; column c is finished by its owner lane and broadcast by shuffle.
__global__ void __launch_bounds__(32 * TRSM_WARPS) trsm_panel_kernel(double* __restrict__ H, int64_t n, int64_t k,
                                                                     int nb) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double l[NB][NB + 1];
    __shared__ double rdiag[NB];
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
        const int ii = e % NB, jj = e / NB;
        l[ii][jj] = (ii < nb && jj < nb && ii >= jj) ? H[(k + ii) + (k + jj) * n] : 0.0;
    }
    if (threadIdx.x < nb) rdiag[threadIdx.x] = 1.0 / H[(k + threadIdx.x) * (n + 1)];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row = k + nb + (int64_t)blockIdx.x * TRSM_WARPS + warp;
    if (row >= n) return;
    double x0 = (lane < nb) ? H[row + (k + lane) * n] : 0.0;
    double x1 = (lane + 32 < nb) ? H[row + (k + lane + 32) * n] : 0.0;
    for (int c = 0; c < nb; ++c) {
        // finish x[c] on its owner lane, broadcast, update the columns after it
        const bool hi = c >= 32;
        double xc = 0.0;
        if (lane == (c & 31)) xc = (hi ? x1 : x0) * rdiag[c];
        xc = __shfl_sync(0xffffffffu, xc, c & 31);
        if (lane == (c & 31)) {
            if (hi) x1 = xc;
            else x0 = xc;
        }
        if (!hi && lane > c) x0 -= xc * l[lane][c];
        if (lane + 32 > c && lane + 32 < nb) x1 -= xc * l[lane + 32][c];
    }
    if (lane < nb) H[row + (k + lane) * n] = x0;
    if (lane + 32 < nb) H[row + (k + lane + 32) * n] = x1;
}

// strict upper triangle <- L^T (H[i + j n] = H[j + i n] for i < j)
__global__ void mirror_upper_kernel(double* __restrict__ H, int64_t n) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
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

// Inverse of each 64x64 lower-triangular diagonal block, latency-shaped for
// parallelism: eight 8x8 leaves
// by forward substitution in parallel (lane = column, reciprocal diagonals
// precomputed), then three 2x2 combine levels X21 = -X22 (L21 X11) as small
// shared-memory products with four independent accumulators per output.
// One CTA (8 warps) per block.
constexpr int TI = 64, TIP = TI + 1;
__device__ __forceinline__ double dot_strided4(const double* a, int as, const double* b, int bs, int q0, int q1) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    int q = q0;
    for (; q + 3 < q1; q += 4) {
        c0 = fma(a[q * as], b[q * bs], c0);
        c1 = fma(a[(q + 1) * as], b[(q + 1) * bs], c1);
        c2 = fma(a[(q + 2) * as], b[(q + 2) * bs], c2);
        c3 = fma(a[(q + 3) * as], b[(q + 3) * bs], c3);
    }
    for (; q < q1; ++q) c0 = fma(a[q * as], b[q * bs], c0);
    return (c0 + c1) + (c2 + c3);
}

__global__ void __launch_bounds__(256) tri_inv64_kernel(const double* __restrict__ L, int64_t n,
                                                        double* __restrict__ W) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ double ti_smem[];
    double(*l)[TIP] = reinterpret_cast<double(*)[TIP]>(ti_smem);
    double(*x)[TIP] = reinterpret_cast<double(*)[TIP]>(ti_smem + TI * TIP);
    double(*tt)[TIP] = reinterpret_cast<double(*)[TIP]>(ti_smem + 2 * TI * TIP);
    const int64_t k = (int64_t)blockIdx.x * TI;
    const int nb = (int)imin64(TI, n - k);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < TI * TI; e += 256) {
        const int i = e & 63, j = e >> 6;
        double v = 0.0;
        if (i < nb && j < nb) v = i >= j ? L[(k + i) + (k + j) * n] : 0.0;
        else if (i == j) v = 1.0;  // identity padding of a ragged last block
        l[i][j] = v;
        x[i][j] = 0.0;
    }
    __syncthreads();
    // ---- leaves: warp w inverts the 8x8 block at (8w, 8w); lane c < 8 owns column c
    {
        const int o = 8 * warp, c = lane;
        if (c < 8) {
            double rd[8], xr[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) rd[i] = 1.0 / l[o + i][o + i];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
                for (int q = 0; q < i; ++q) {
                    const double t = l[o + i][o + q] * xr[q];
                    if (q & 1) s1 -= t;
                    else s0 -= t;
                }
                xr[i] = i < c ? 0.0 : (s0 + s1) * rd[i];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) x[o + i][o + c] = xr[i];
        }
    }
    __syncthreads();
    // ---- combine levels h = 8, 16, 32: pairs at offsets 2h*p; X21 = -X22 (L21 X11)
    for (int h = 8; h < TI; h *= 2) {
        const int npairs = TI / (2 * h);
        // T = L21 X11 (X11 lower: q >= j) into tt at the X21 positions
        for (int e = tid; e < npairs * h * h; e += 256) {
            const int pr = e / (h * h), r = e % (h * h), i = r % h, j = r / h;
            const int o = 2 * h * pr;
            tt[o + h + i][o + j] = dot_strided4(&l[o + h + i][o], 1, &x[o][o + j], TIP, j, h);
        }
        __syncthreads();
        // X21 = -X22 T (X22 lower: q <= i)
        for (int e = tid; e < npairs * h * h; e += 256) {
            const int pr = e / (h * h), r = e % (h * h), i = r % h, j = r / h;
            const int o = 2 * h * pr;
            x[o + h + i][o + j] = -dot_strided4(&x[o + h + i][o + h], 1, &tt[o + h][o + j], TIP, 0, i + 1);
        }
        __syncthreads();
    }
    for (int e = tid; e < nb * nb; e += 256) {
        const int i = e % nb, j = e / nb;
        if (i >= j) W[(k + i) + (k + j) * n] = x[i][j];
    }
}

// y[:, q] (+)= T x[:, q] for a triangular T stored in Wf: lower (W) when
// lower != 0, else upper (W^T mirrored into the strict upper triangle, with
// the diagonal of W). CTA tile: 64 rows x 512 columns; partials per column
// chunk go to part[chunk][q][row] and are summed in fixed order afterwards.
constexpr int TR_ROWS = 64, TR_COLS = 64;  // 16 columns per thread: short, independent load chains
__global__ void __launch_bounds__(256) trmv_partial_kernel(const double* __restrict__ Wf, int64_t n, int lower,
                                                           const double* __restrict__ x, int nrhs,
                                                           double* __restrict__ part) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t r0 = (int64_t)blockIdx.x * TR_ROWS;
    const int64_t c0 = (int64_t)blockIdx.y * TR_COLS;
    const int64_t c1 = imin64(n, c0 + TR_COLS);
    __shared__ double xs[2][TR_COLS];
    __shared__ double red[4][2][TR_ROWS];
    const bool skip = lower ? (c0 > r0 + TR_ROWS - 1) : (c1 - 1 < r0);
    const int r = threadIdx.x % TR_ROWS, qg = threadIdx.x / TR_ROWS;  // 4 column interleaves
    const int64_t row = r0 + r;
    double acc[2] = {0.0, 0.0};
    if (!skip) {
        for (int e = threadIdx.x; e < (int)(c1 - c0); e += blockDim.x)
            for (int q = 0; q < nrhs; ++q) xs[q][e] = x[q * n + c0 + e];
        __syncthreads();
        if (row < n) {
            int64_t jb = c0 + qg, je = c1;
            if (lower) je = imin64(je, row + 1);        // j <= row
            else if (jb < row) jb += ((row - jb + 3) / 4) * 4;  // j >= row, same interleave class
            for (int64_t j = jb; j < je; j += 4) {
                const double w = Wf[row + j * n];
                acc[0] = fma(w, xs[0][j - c0], acc[0]);
                if (nrhs > 1) acc[1] = fma(w, xs[1][j - c0], acc[1]);
            }
        }
    }
    red[qg][0][r] = acc[0];
    red[qg][1][r] = acc[1];
    __syncthreads();
    if (threadIdx.x < TR_ROWS && row < n) {
        for (int q = 0; q < nrhs; ++q)
            part[((int64_t)blockIdx.y * nrhs + q) * n + row] =
                (red[0][q][r] + red[1][q][r]) + (red[2][q][r] + red[3][q][r]);
    }
}

__global__ void trmv_reduce_kernel(const double* __restrict__ part, int64_t n, int nrhs, int nchunks, int lower,
                                   double* __restrict__ y) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    const int64_t total = (int64_t)nrhs * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / n, row = e % n;
        // chunks that touch this row: lower -> chunks with c0 <= row, upper -> c1 > row
        double s = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const int64_t c0 = (int64_t)c * TR_COLS, c1 = imin64(n, c0 + TR_COLS);
            const int64_t r0 = (row / TR_ROWS) * TR_ROWS;
            const bool skip = lower ? (c0 > r0 + TR_ROWS - 1) : (c1 - 1 < r0);
            if (!skip) s += part[((int64_t)c * nrhs + q) * n + row];
        }
        y[e] = s;
    }
}

void trmv(const double* Wf, int64_t n, bool lower, const double* x, int nrhs, double* y, double* part, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(n, TR_ROWS), (unsigned)ceil_div(n, TR_COLS));
    LAUNCH_PDL(trmv_partial_kernel, grid, 256, 0, st, Wf, n, (int)lower, x, nrhs, part);
    const int64_t total = (int64_t)nrhs * n;
    LAUNCH_PDL(trmv_reduce_kernel, (unsigned)std::min<int64_t>(ceil_div(total, 256), 1024), 256, 0, st, part, n, nrhs,
           (int)grid.y, (int)lower, y);
}

// W[n0:n0+size, n0:n0+size] <- L^{-1} of the same diagonal block (lower), with
// the diagonal 64-blocks already inverted and the strict upper part zero.
void tri_inv_rec(const double* L, double* W, int64_t n, int64_t n0, int64_t size, double* tmp, cudaStream_t st,
                 int base = NB) {
    if (size <= base) return;
    const int64_t h = ((size / 2 + base - 1) / base) * base;  // split on a block boundary
    tri_inv_rec(L, W, n, n0, h, tmp, st, base);
    tri_inv_rec(L, W, n, n0 + h, size - h, tmp, st, base);
    const int64_t m2 = size - h;
    // tmp (m2 x h, ld m2) = L21 * W11
    dgemm(false, false, m2, h, h, 1.0, L + (n0 + h) + n0 * n, n, W + n0 + n0 * n, n, 0.0, tmp, m2, false, 1, nullptr,
          st);
    // W21 = -W22 * tmp
    dgemm(false, false, m2, h, m2, -1.0, W + (n0 + h) + (n0 + h) * n, n, tmp, m2, 0.0, W + (n0 + h) + n0 * n, n, false,
          1, nullptr, st);
}
}  // namespace

void cholesky_invert(const double* d_L, int64_t n, double* d_W, double* d_tmp, cudaStream_t st) {
    CUDA_CHECK(cudaMemsetAsync(d_W, 0, (size_t)n * n * sizeof(double), st));
    const int base = NB;
    const size_t ti_smem = (size_t)3 * TI * TIP * sizeof(double);
    IHS_SMEM_ATTR(tri_inv64_kernel, (int)ti_smem);
    LAUNCH_PDL(tri_inv64_kernel, (unsigned)ceil_div(n, NB), 256, ti_smem, st, d_L, n, d_W);
    // n = base * 2^L: the recursion's nodes of one size are independent and equally shaped, so each level is
    // two strided-batched products (2 L launches instead of 2 (2^L - 1)); otherwise the recursion itself
    static const bool rec_only = [] {  // IHS_TRI_INV_REC=1: the depth-first recursion (A/B)
        const char* e = std::getenv("IHS_TRI_INV_REC");
        return e && e[0] == '1';
    }();
    int64_t blocks = n / base;
    if (!rec_only && n % base == 0 && blocks > 1 && (blocks & (blocks - 1)) == 0) {
        for (int64_t h = base; h < n; h *= 2) {
            const int64_t s = 2 * h, nodes = n / s, diag = s * (n + 1);  // node i: rows/cols [i s, i s + s)
            // tmp_i (h x h) = L21_i W11_i;  W21_i = -W22_i tmp_i
            if (nodes == 1) {  // the top level: one product, on whichever kernel suits its size
                dgemm(false, false, h, h, h, 1.0, d_L + h, n, d_W, n, 0.0, d_tmp, h, false, 1, nullptr, st);
                dgemm(false, false, h, h, h, -1.0, d_W + h + h * n, n, d_tmp, h, 0.0, d_W + h, n, false, 1, nullptr, st);
                continue;
            }
            dgemm_batched(false, false, h, h, h, 1.0, d_L + h, n, diag, d_W, n, diag, 0.0, d_tmp, h, h * h,
                          (int)nodes, st);
            dgemm_batched(false, false, h, h, h, -1.0, d_W + h + h * n, n, diag, d_tmp, h, h * h, 0.0, d_W + h, n, diag,
                          (int)nodes, st);
        }
    } else {
        tri_inv_rec(d_L, d_W, n, 0, n, d_tmp, st, base);
    }
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
    LAUNCH_PDL(mirror_upper_kernel, grid, dim3(32, 8), 0, st, d_W, n);
}

size_t cholesky_solve_work_doubles(int64_t n) { return (size_t)ceil_div(n, TR_COLS) * 2 * n + 2 * n; }

void cholesky_solve_inv(const double* d_W, int64_t n, const double* d_R, double* d_Z, int nrhs, double* d_work,
                        cudaStream_t st) {
    double* part = d_work;
    double* y = d_work + (size_t)ceil_div(n, TR_COLS) * 2 * n;
    trmv(d_W, n, true, d_R, nrhs, y, part, st);    // y = L^{-1} r
    trmv(d_W, n, false, y, nrhs, d_Z, part, st);   // z = L^{-T} y
}

void cholesky_factor(double* d_H, int64_t n, int* d_info, cudaStream_t st) {
    CUDA_CHECK(cudaMemsetAsync(d_info, 0, sizeof(int), st));
    for (int64_t k = 0; k < n; k += NB) {
        const int nb = (int)std::min<int64_t>(NB, n - k);
        LAUNCH_PDL(potrf_diag_kernel, 1, 256, 0, st, d_H, n, k, nb, d_info);
        const int64_t rest = n - k - nb;
        if (rest > 0) {
            LAUNCH_PDL(trsm_panel_kernel, (unsigned)ceil_div(rest, TRSM_WARPS), 32 * TRSM_WARPS, 0, st, d_H, n, k, nb);
            // A22 -= L21 L21^T (lower)
            double* L21 = d_H + (k + nb) + k * n;
            double* A22 = d_H + (k + nb) + (k + nb) * n;
            dgemm(false, true, rest, rest, nb, -1.0, L21, n, L21, n, 1.0, A22, n, true, 1, nullptr, st);
        }
    }
}

}  // namespace ihs_b200
