// lat_micro.cu — dependent-chain latencies (SM cycles per op) of fp64/fp32 primitives on one warp,
// one kernel per operation (no branches in the loop):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(double* out, long long* cyc, double seed) {
    double x = seed + threadIdx.x * 1e-9;
    const double y = 1.0000001;
    const int N = 4096;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (OP == 0) x = fma(x, y, 1e-300);
        if (OP == 1) x = x + y;
        if (OP == 2) x = x * y;
        if (OP == 3) x = sqrt(x);
        if (OP == 4) x = 1.5 / x;
        if (OP == 5) x = rsqrt(x);
        if (OP == 6) x = __drcp_rn(x);
        if (OP == 7) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
        if (OP == 8) {
            double c0 = x, c1 = 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0), "+d"(c1) : "d"(y), "d"(y));
            x = c0;
        }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / N;
}

__global__ void latf(float* out, long long* cyc, float seed) {
    float x = seed + threadIdx.x * 1e-9f;
    const float y = 1.0000001f;
    const int N = 4096;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fmaf(x, y, 1e-30f);
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[15] = (t1 - t0) / N;
}

int main() {
    double* out;
    float* fo;
    long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMalloc(&fo, 32 * 4);
    cudaMallocManaged(&cyc, 16 * 8);
    for (int r = 0; r < 2; ++r) {
        lat<0><<<1, 32>>>(out, cyc, 2.0);
        lat<1><<<1, 32>>>(out, cyc, 2.0);
        lat<2><<<1, 32>>>(out, cyc, 2.0);
        lat<3><<<1, 32>>>(out, cyc, 2.0);
        lat<4><<<1, 32>>>(out, cyc, 2.0);
        lat<5><<<1, 32>>>(out, cyc, 2.0);
        lat<6><<<1, 32>>>(out, cyc, 2.0);
        lat<7><<<1, 32>>>(out, cyc, 2.0);
        lat<8><<<1, 32>>>(out, cyc, 2.0);
        latf<<<1, 32>>>(fo, cyc, 2.0f);
    }
    cudaDeviceSynchronize();
    const char* names[] = {"dfma", "dadd", "dmul", "sqrt", "div", "rsqrt", "drcp_rn", "shfl_f64", "dmma"};
    printf("{");
    for (int m = 0; m < 9; ++m) printf("\"%s_cycles\": %lld, ", names[m], cyc[m]);
    printf("\"ffma32_cycles\": %lld}\n", cyc[15]);
    return 0;
}
