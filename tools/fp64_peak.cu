// fp64_peak.cu — measured fp64 peaks of this B200: DMMA (mma.sync m8n8k4 f64)
// and DFMA, sustained over ~2 s each, CUDA-event timed. Prints one JSON line.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
    const double a = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // DMMA: per warp per iteration 8 mma of 8x8x4 = 8*256 MAC = 4096 flop
    const int blocks = sms * 4, threads = 256;
    int iters = 20000;
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // scale iterations to ~2 s
    iters = (int)(iters * (2000.0 / ms));
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_flops = (double)blocks * (threads / 32) * (double)iters * 8 * 512.0;
    const double dmma_tf = dmma_flops / (ms * 1e-3) / 1e12;
    // DFMA: per thread per iteration 8 FMA = 16 flop
    int it2 = 200000;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, it2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    it2 = (int)(it2 * (2000.0 / ms));
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, it2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma_tf = (double)blocks * threads * (double)it2 * 16.0 / (ms * 1e-3) / 1e12;
    cudaError_t err = cudaGetLastError();
    std::printf("{\"fp64_dmma_tflops\": %.3f, \"fp64_dfma_tflops\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n", dmma_tf,
                dfma_tf, sms, cudaGetErrorString(err));
    return err != cudaSuccess;
}
