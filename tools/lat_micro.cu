// lat_micro.cu — dependent-chain latencies (cycles/op) of fp64 primitives on one warp:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void latf(float* out, long long* cyc, float seed) {
    float x = seed + threadIdx.x * 1e-9f, y = 1.0000001f;
    const int N = 1024;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = fmaf(x, y, 1e-30f);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[15] = (t1 - t0) / N;
}

__global__ void lat(double* out, long long* cyc, double seed, int mode) {
    double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
    const int N = 1024;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        switch (mode) {
            case 0: x = fma(x, y, 1e-300); break;
            case 1: x = sqrt(x) + 1.0; break;
            case 2: x = 1.5 / x + 0.5; break;
            case 3: x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * y; break;
            case 4: x = rsqrt(x) + 1.0; break;
            case 5: x = __drcp_rn(x) + 0.5; break;
            case 6: x = x + y; break;
            case 7: x = x * y; break;
            case 8: {
                double c0 = x, c1 = 0.0;
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c0), "+d"(c1) : "d"(y), "d"(y));
                x = c0 * 1e-3;
                break;
            }
            case 9: { float f = (float)x; f = fmaf(f, 1.0001f, 1e-30f); x = f; break; }
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[mode] = (t1 - t0) / N;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 16 * 8);
    const char* names[] = {"dfma", "sqrt", "div", "shfl_f64", "rsqrt", "drcp_rn", "dadd", "dmul", "dmma_plus_dmul",
                           "ffma_plus_cvt"};
    printf("{");
    for (int m = 0; m < 10; ++m) {
        lat<<<1, 32>>>(out, cyc, 2.0, m);
        lat<<<1, 32>>>(out, cyc, 2.0, m);
        cudaDeviceSynchronize();
        printf("%s\"%s_cycles\": %lld", m ? ", " : "", names[m], cyc[m]);
    }
    float* fo;
    cudaMalloc(&fo, 32 * 4);
    latf<<<1, 32>>>(fo, cyc, 2.0f);
    latf<<<1, 32>>>(fo, cyc, 2.0f);
    cudaDeviceSynchronize();
    printf(", \"ffma32_cycles\": %lld", cyc[15]);
    printf("}\n");
    return 0;
}
