// chol_micro.cu — isolated timings of the Cholesky diagonal-block kernels
// (CUDA events, warm, averaged). Builds against the library for LAUNCH's
// launch counter and the DMMA GEMM:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2006_05874_b200/csrc tools/chol_micro.cu -Lpaper_2006_05874_b200 -lihs_b200 \
//        -Xlinker -rpath -Xlinker $PWD/paper_2006_05874_b200 -o tools/chol_micro
#include "../paper_2006_05874_b200/csrc/chol.cu"

#include <cstdio>
#include <vector>

using namespace ihs_b200;

__global__ void only_potrf32(double* H, int* info) {
    __shared__ double a[64][PB];
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) a[e & 63][e >> 6] = H[e];
    __syncthreads();
    if (threadIdx.x < 32) potrf32_warp(a, 0, info, 0, 64);
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) H[64 * 64 + e] = a[e & 63][e >> 6];
}

__global__ void only_trtri32(double* H) {
    __shared__ double a[32][PB], x[32][PB];
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) a[e & 31][e >> 5] = (e & 31) == (e >> 5) ? 2.0 : 0.01;
    __syncthreads();
    if (threadIdx.x < 32) trtri32_warp(a, x, 0);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) H[64 * 64 + e] = x[e & 31][e >> 5];
}


// candidate: register-resident right-looking LLT of a 64x64 block, one barrier per column.
// 256 threads; thread t owns lower elements e = t + 256u (u < 9) of the column-major
// enumeration of the lower triangle; column j's current values are published into a
// ping-pong shared column; the L column j = col * rsqrt(pivot) is written by 64 threads.
__device__ __forceinline__ void tri_index(int e, int& i, int& j) {
    // column-major lower triangle of 64: column j holds 64 - j entries
    int c = 0, base = 0;
    while (base + (64 - c) <= e) { base += 64 - c; ++c; }
    j = c;
    i = c + (e - base);
}
__global__ void __launch_bounds__(256) potrf64_reg(double* __restrict__ H, int64_t n, int* __restrict__ info) {
    __shared__ double col[2][64];
    __shared__ double L[64][PB];
    constexpr int NE = 9;  // ceil(2080 / 256)
    double v[NE];
    int ei[NE], ej[NE];
    const int t = threadIdx.x;
#pragma unroll
    for (int u = 0; u < NE; ++u) {
        const int e = t + 256 * u;
        if (e < 2080) {
            tri_index(e, ei[u], ej[u]);
            v[u] = H[ei[u] + ej[u] * n];
            if (ej[u] == 0) col[0][ei[u]] = v[u];
        } else {
            ei[u] = 0; ej[u] = 64; v[u] = 0.0;
        }
    }
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
        const double* cj = col[j & 1];
        double* cn = col[(j + 1) & 1];
        double d = cj[j];
        if (!(d > 0.0) || !isfinite(d)) { if (t == 0) atomicCAS(info, 0, j + 1); d = 1.0; }
        const double rs = rsqrt(d);
        const double rd = rs * rs;
        if (t < 64 && t >= j) L[t][j] = cj[t] * rs;
#pragma unroll
        for (int u = 0; u < NE; ++u) {
            if (ej[u] > j) {
                v[u] = fma(-cj[ei[u]] * rd, cj[ej[u]], v[u]);
                if (ej[u] == j + 1) cn[ei[u]] = v[u];
            }
        }
        __syncthreads();
    }
    for (int e = t; e < 64 * 64; e += 256) {
        const int i = e & 63, jj = e >> 6;
        if (i >= jj) H[i + jj * n] = L[i][jj];
    }
}

__global__ void __launch_bounds__(1024) potrf64_reg1k(double* __restrict__ H, int64_t n, int* __restrict__ info) {
    __shared__ double col[2][64];
    __shared__ double L[64][PB];
    constexpr int NE = 3;  // ceil(2080 / 1024)
    double v[NE];
    int ei[NE], ej[NE];
    const int t = threadIdx.x;
#pragma unroll
    for (int u = 0; u < NE; ++u) {
        const int e = t + 1024 * u;
        if (e < 2080) {
            tri_index(e, ei[u], ej[u]);
            v[u] = H[ei[u] + ej[u] * n];
            if (ej[u] == 0) col[0][ei[u]] = v[u];
        } else {
            ei[u] = 0; ej[u] = 64; v[u] = 0.0;
        }
    }
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
        const double* cj = col[j & 1];
        double* cn = col[(j + 1) & 1];
        double d = cj[j];
        if (!(d > 0.0) || !isfinite(d)) { if (t == 0) atomicCAS(info, 0, j + 1); d = 1.0; }
        const double rs = rsqrt(d);
        const double rd = rs * rs;
        if (t < 64 && t >= j) L[t][j] = cj[t] * rs;
#pragma unroll
        for (int u = 0; u < NE; ++u) {
            if (ej[u] > j) {
                v[u] = fma(-cj[ei[u]] * rd, cj[ej[u]], v[u]);
                if (ej[u] == j + 1) cn[ei[u]] = v[u];
            }
        }
        __syncthreads();
    }
    for (int e = t; e < 64 * 64; e += 1024) {
        const int i = e & 63, jj = e >> 6;
        if (i >= jj) H[i + jj * n] = L[i][jj];
    }
}


__global__ void loop_sync(double* out, int mode) {
    __shared__ double c[2][64];
    const int t = threadIdx.x;
    if (t < 64) c[0][t] = 1.0 + t;
    __syncthreads();
    double acc = 0.0;
    for (int j = 0; j < 64; ++j) {
        double dj = c[j & 1][j];
        if (mode >= 1) dj = rsqrt(dj);
        if (mode >= 2) acc = fma(dj, c[j & 1][t & 63], acc);
        if (t < 64) c[(j + 1) & 1][t] = dj + acc;
        __syncthreads();
    }
    if (t == 0) out[0] = acc;
}


// 1024 threads, thread t owns row i = t & 63, columns c0 + 16u (c0 = t >> 6, u < 4)
__global__ void __launch_bounds__(1024) potrf64_grid(double* __restrict__ H, int64_t n, int* __restrict__ info) {
    __shared__ double col[2][64];
    __shared__ double L[64][PB];
    const int t = threadIdx.x, i = t & 63, c0 = t >> 6;
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int jj = c0 + 16 * u;
        v[u] = i >= jj ? H[i + jj * n] : 0.0;
        if (jj == 0) col[0][i] = v[u];
    }
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < 64; ++j) {
        const double* cj = col[j & 1];
        double* cn = col[(j + 1) & 1];
        double d = cj[j];
        if (!(d > 0.0) || !isfinite(d)) { if (t == 0) atomicCAS(info, 0, j + 1); d = 1.0; }
        const double rs = rsqrt(d);
        if (t < 64 && t >= j) L[t][j] = cj[t] * rs;
        const double li = cj[i] * (rs * rs);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int jj = c0 + 16 * u;
            const bool act = jj > j && i >= jj;
            const double nv = fma(-li, cj[jj], v[u]);
            v[u] = act ? nv : v[u];
            if (act && jj == j + 1) cn[i] = v[u];
        }
        __syncthreads();
    }
    for (int e = t; e < 64 * 64; e += 1024) {
        const int r = e & 63, c = e >> 6;
        if (r >= c) H[r + c * n] = L[r][c];
    }
}

__global__ void empty_kernel(double*) {}

template <class F>
float time_it(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return 1e3f * ms / reps;
}

int main() {
    const int n = 64;
    std::vector<double> h(2 * n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[i + n * j] = (i == j ? n : 0.0) + 1.0 / (1.0 + i + j);
    double *d, *xd;
    int* info;
    cudaMalloc(&d, 2 * n * n * 8);
    cudaMalloc(&xd, n * n * 8);
    cudaMalloc(&info, 4);
    cudaMemset(info, 0, 4);
    cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d + n * n, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    const size_t pi_smem = (size_t)(64 + 64 + 32) * PB * sizeof(double);
    cudaFuncSetAttribute(potrf_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pi_smem);
    const int reps = 200;
    printf("{\"empty_us\": %.2f", time_it([&] { empty_kernel<<<1, 128>>>(d); }, reps));
    auto restore = [&] { cudaMemcpyAsync(d + n * n, d, n * n * 8, cudaMemcpyDeviceToDevice); };
    printf(", \"restore_only_us\": %.2f", time_it([&] { restore(); }, reps));
    printf(", \"potrf_diag_us\": %.2f", time_it([&] {
        restore();
        potrf_diag_kernel<<<1, 256>>>(d + n * n, n, 0, 64, info);
    }, reps));
    printf(", \"tri_inv_diag_us\": %.2f", time_it([&] {
        cudaFuncSetAttribute(tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * (NB + 1) * 8);
        tri_inv_diag_kernel<<<1, 64, 2 * NB * (NB + 1) * 8>>>(d, n, d + n * n);
    }, reps));
    cudaFuncSetAttribute(tri_inv64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TI * TIP * 8);
    printf(", \"tri_inv64_us\": %.2f", time_it([&] {
        tri_inv64_kernel<<<1, 256, 3 * TI * TIP * 8>>>(d, n, d + n * n);
    }, reps));
    printf(", \"potrf_inv_diag_us\": %.2f", time_it([&] { restore(); potrf_inv_diag_kernel<<<1, 128, pi_smem>>>(d + n * n, n, 0, 64, xd, info); }, reps));
    printf(", \"only_potrf32_us\": %.2f", time_it([&] { restore(); only_potrf32<<<1, 128>>>(d + n * n, info); }, reps));
    printf(", \"only_trtri32_us\": %.2f", time_it([&] { only_trtri32<<<1, 128>>>(d); }, reps));
    for (int mode = 0; mode < 3; ++mode)
        printf(", \"loop_sync%d_us\": %.2f", mode, time_it([&] { loop_sync<<<1, 256>>>(d, mode); }, reps));
    printf(", \"potrf64_reg1k_us\": %.2f", time_it([&] { restore(); potrf64_reg1k<<<1, 1024>>>(d + n * n, n, info); }, reps));
    printf(", \"potrf64_grid_us\": %.2f", time_it([&] { restore(); potrf64_grid<<<1, 1024>>>(d + n * n, n, info); }, reps));
    printf(", \"potrf64_reg_us\": %.2f", time_it([&] { restore(); potrf64_reg<<<1, 256>>>(d + n * n, n, info); }, reps));
    // accuracy of potrf64_reg against potrf_diag on the same SPD input
    {
        double *d1, *d2;
        cudaMalloc(&d1, n * n * 8);
        cudaMalloc(&d2, n * n * 8);
        cudaMemcpy(d1, h.data(), n * n * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(d2, h.data(), n * n * 8, cudaMemcpyHostToDevice);
        potrf_diag_kernel<<<1, 256>>>(d1, n, 0, 64, info);
        potrf64_grid<<<1, 1024>>>(d2, n, info);
        std::vector<double> a1(n * n), a2(n * n);
        cudaMemcpy(a1.data(), d1, n * n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(a2.data(), d2, n * n * 8, cudaMemcpyDeviceToHost);
        double md = 0, ma = 0;
        for (int j = 0; j < n; ++j)
            for (int i = j; i < n; ++i) { md = fmax(md, fabs(a1[i + n * j] - a2[i + n * j])); ma = fmax(ma, fabs(a1[i + n * j])); }
        printf(", \"potrf64_reg_maxdiff_rel\": %.3e", md / ma);
    }
    // whole factorizations: per-panel kernels vs one cooperative launch
    for (int K : {64, 256, 512, 1024}) {
        std::vector<double> hk((size_t)K * K);
        for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j) hk[i + (size_t)K * j] = (i == j ? K : 0.0) + 1.0 / (1.0 + i + j);
        double *src, *dst, *xk;
        cudaMalloc(&src, (size_t)K * K * 8);
        cudaMalloc(&dst, (size_t)K * K * 8);
        cudaMalloc(&xk, cholesky_diag_inv_doubles(K) * 8);
        cudaMemcpy(src, hk.data(), (size_t)K * K * 8, cudaMemcpyHostToDevice);
        auto rs = [&] { cudaMemcpyAsync(dst, src, (size_t)K * K * 8, cudaMemcpyDeviceToDevice); };
        const float t_copy = time_it(rs, 50);
        const float t_panel = time_it([&] { rs(); cholesky_factor(dst, K, nullptr, info, 148, 0); }, 50);
        const float t_coop = time_it([&] { rs(); cholesky_factor_coop(dst, K, xk, info, 148, 0); }, 50);
        printf(", \"k%d\": {\"copy_us\": %.1f, \"panel_us\": %.1f, \"coop_us\": %.1f}", K, t_copy, t_panel, t_coop);
        cudaFree(src);
        cudaFree(dst);
        cudaFree(xk);
    }
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
