// lat_micro.cu — dependent-chain latencies (cycles/op) of fp64 primitives on one warp:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

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
    cudaMallocManaged(&cyc, 8 * 8);
    const char* names[] = {"dfma", "sqrt", "div", "shfl_f64", "rsqrt", "drcp_rn"};
    printf("{");
    for (int m = 0; m < 6; ++m) {
        lat<<<1, 32>>>(out, cyc, 2.0, m);
        lat<<<1, 32>>>(out, cyc, 2.0, m);
        cudaDeviceSynchronize();
        printf("%s\"%s_cycles\": %lld", m ? ", " : "", names[m], cyc[m]);
    }
    printf("}\n");
    return 0;
}
