#include <cstdio>
#include <cuda_runtime.h>
// per-step latency of the potrf column chain: shfl -> rsqrt -> mul -> shfl -> fma (one warp)
__global__ void chain_rsqrt(double* out, int steps) {
    const int lane = threadIdx.x & 31;
    double r = 2.0 + lane * 1e-3, acc = 0.0;
    for (int j = 0; j < steps; ++j) {
        double d = __shfl_sync(0xffffffffu, r, j & 31);
        const double rs = rsqrt(d);
        const double l = r * rs;
        const double lq = __shfl_sync(0xffffffffu, l, (j + 1) & 31);
        r = fma(-l, lq * 1e-3, r) + 1.0;
        acc += l;
    }
    out[threadIdx.x] = r + acc;
}
__global__ void chain_sqrtdiv(double* out, int steps) {
    const int lane = threadIdx.x & 31;
    double r = 2.0 + lane * 1e-3, acc = 0.0;
    for (int j = 0; j < steps; ++j) {
        double d = __shfl_sync(0xffffffffu, r, j & 31);
        const double sq = sqrt(d);
        const double l = r / sq;
        const double lq = __shfl_sync(0xffffffffu, l, (j + 1) & 31);
        r = fma(-l, lq * 1e-3, r) + 1.0;
        acc += l;
    }
    out[threadIdx.x] = r + acc;
}
__global__ void chain_shfl(double* out, int steps) {
    const int lane = threadIdx.x & 31;
    double r = 2.0 + lane * 1e-3;
    for (int j = 0; j < steps; ++j) {
        double d = __shfl_sync(0xffffffffu, r, j & 31);
        r = fma(d, 1e-3, r);
    }
    out[threadIdx.x] = r;
}
__global__ void chain_rsqrt_only(double* out, int steps) {
    double r = 2.0 + threadIdx.x * 1e-3;
    for (int j = 0; j < steps; ++j) r = rsqrt(r) + 1.5;
    out[threadIdx.x] = r;
}
template <class K> float time_it(K k, double* d, int steps) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<1, 32>>>(d, steps); cudaDeviceSynchronize();
    cudaEventRecord(a); k<<<1, 32>>>(d, steps); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
    double* d; cudaMalloc(&d, 1024);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int steps = 100000;
    auto cyc = [&](float ms) { return ms * 1e-3 * clk * 1e3 / steps; };
    printf("{\"rsqrt_chain_cyc\": %.1f, \"sqrtdiv_chain_cyc\": %.1f, \"shfl_fma_cyc\": %.1f, \"rsqrt_only_cyc\": %.1f}\n",
           cyc(time_it(chain_rsqrt, d, steps)), cyc(time_it(chain_sqrtdiv, d, steps)), cyc(time_it(chain_shfl, d, steps)),
           cyc(time_it(chain_rsqrt_only, d, steps)));
}
