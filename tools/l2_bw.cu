// l2_bw.cu — measured L2-resident bandwidth of this B200 for the access patterns of the L2-resident SRHT's
// T ring (srht.cu, srht_l2_kernel): a buffer of B MiB (default 32, 64, 96: the ring depths 1-3 of C4's 32 MiB
// columns) is first touched, then repeatedly
//   read    — 16-byte coalesced loads (ld.global.cg), as the emitting groups read their tiles;
//   write   — 16-byte coalesced stores of whole lines, as the item stores;
//   strided — 128-byte line writes 64 KiB apart (one line per tile per item: the c-major T layout's pattern);
// each as one persistent launch of 148 x 8 CTAs, CUDA-event timed, best of R. Prints one JSON line.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) l2_read(const double2* __restrict__ src, size_t n16, int passes, double* out) {
    double acc = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n16; i += 4 * stride) {
            const double2 a = __ldcg(src + i), b = __ldcg(src + i + stride), c = __ldcg(src + i + 2 * stride),
                          d = __ldcg(src + i + 3 * stride);
            acc += (a.x + b.y) + (c.x + d.y);
        }
        for (; i < n16; i += stride) acc += __ldcg(src + i).x;
    }
    if (acc == 1234.5) out[0] = acc;
}

__global__ void __launch_bounds__(512) l2_write(double2* __restrict__ dst, size_t n16, int passes) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
            __stcg(dst + i, make_double2((double)p, (double)i));
}

// 8 lanes write one 128-byte line; consecutive line groups are 64 KiB apart (wrapping inside the buffer)
__global__ void __launch_bounds__(512) l2_write_strided(double2* __restrict__ dst, size_t n16, int passes) {
    const size_t lines = n16 / 8, per_row = 65536 / 128;  // lines per 64 KiB row
    const size_t rows = lines / per_row;
    const size_t gstride = (size_t)gridDim.x * (blockDim.x / 8);
    for (int p = 0; p < passes; ++p)
        for (size_t l = (size_t)blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8; l < lines; l += gstride) {
            const size_t row = l % rows, col = l / rows;  // successive l: successive 64 KiB rows, same column
            __stcg(dst + (row * per_row + col) * 8 + (threadIdx.x & 7), make_double2((double)p, (double)l));
        }
}

// half the CTAs stream a large buffer from HBM (read once per pass, 16-byte loads), the other half store into an
// L2-resident buffer: do A's fill and T's store share one L2 write budget (the SRHT's two streams)?
__global__ void __launch_bounds__(512) mixed(const double2* __restrict__ big, size_t nbig16, double2* __restrict__ l2buf,
                                             size_t nl2_16, int passes, double* out, unsigned long long* cyc) {
    const int half = gridDim.x / 2;
    const bool reader = blockIdx.x < half;
    const int b = reader ? blockIdx.x : blockIdx.x - half;
    const size_t stride = (size_t)half * blockDim.x;
    const long long t0 = clock64();
    if (reader) {
        double acc = 0.0;
        for (size_t i = (size_t)b * blockDim.x + threadIdx.x; i + 3 * stride < nbig16; i += 4 * stride) {
            const double2 a = __ldcs(big + i), c = __ldcs(big + i + stride), e = __ldcs(big + i + 2 * stride),
                          f = __ldcs(big + i + 3 * stride);
            acc += (a.x + c.y) + (e.x + f.y);
        }
        if (acc == 1234.5) out[0] = acc;
    } else {
        for (int p = 0; p < passes; ++p)
            for (size_t i = (size_t)b * blockDim.x + threadIdx.x; i < nl2_16; i += stride)
                __stcg(l2buf + i, make_double2((double)p, (double)i));
    }
    if (threadIdx.x == 0) atomicMax(cyc + (reader ? 0 : 1), (unsigned long long)(clock64() - t0));
}

int main(int argc, char** argv) {
    const int reps = 5, passes = 20;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out = nullptr;
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"sms\": %d, \"passes\": %d", sms, passes);
    const int mib_list[3] = {32, 64, 96};
    for (int mi = 0; mi < 3; ++mi) {
        const size_t mib = argc > 1 ? strtoull(argv[1], nullptr, 10) : (size_t)mib_list[mi];
        const size_t bytes = mib << 20, n16 = bytes / 16;
        double2* buf = nullptr;
        if (cudaMalloc(&buf, bytes) != cudaSuccess) {
            printf(", \"err\": \"alloc\"}\n");
            return 1;
        }
        cudaMemset(buf, 0, bytes);
        float best[3] = {1e30f, 1e30f, 1e30f};
        for (int r = 0; r < reps; ++r)
            for (int k = 0; k < 3; ++k) {
                cudaEventRecord(e0);
                if (k == 0) l2_read<<<sms * 4, 512>>>(buf, n16, passes, out);
                else if (k == 1) l2_write<<<sms * 4, 512>>>(buf, n16, passes);
                else l2_write_strided<<<sms * 4, 512>>>(buf, n16, passes);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best[k]) best[k] = ms;
            }
        const double gb = (double)bytes * passes / 1e9;
        printf(", \"%zu_MiB\": {\"read_GBps\": %.0f, \"write_GBps\": %.0f, \"strided_write_GBps\": %.0f}", mib,
               gb / (best[0] * 1e-3), gb / (best[1] * 1e-3), gb / (best[2] * 1e-3));
        cudaFree(buf);
        if (argc > 1) break;
    }
    {  // mixed: 8 GiB streamed from HBM by half the CTAs while the other half store into a 64 MiB L2 buffer
        const size_t big_b = 8ull << 30, l2_b = 64ull << 20;
        double2 *big = nullptr, *l2 = nullptr;
        unsigned long long* cyc = nullptr;
        if (cudaMalloc(&big, big_b) == cudaSuccess && cudaMalloc(&l2, l2_b) == cudaSuccess &&
            cudaMalloc(&cyc, 16) == cudaSuccess) {
            cudaMemset(big, 0, big_b);
            cudaMemset(l2, 0, l2_b);
            int clk_khz = 0;
            cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
            // passes chosen so the store half moves about as many bytes as the read half
            const int mpasses = (int)(big_b / l2_b);
            float best = 1e30f;
            for (int r = 0; r < 3; ++r) {
                cudaMemset(cyc, 0, 16);
                cudaEventRecord(e0);
                mixed<<<sms * 4, 512>>>(big, big_b / 16, l2, l2_b / 16, mpasses, out, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            unsigned long long hc[2] = {0, 0};
            cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
            printf(", \"mixed\": {\"ms\": %.3f, \"hbm_read_GB\": %.2f, \"l2_write_GB\": %.2f, \"aggregate_GBps\": %.0f, "
                   "\"reader_cycles\": %llu, \"writer_cycles\": %llu}",
                   best, big_b / 1e9, (double)l2_b * mpasses / 1e9, (big_b + (double)l2_b * mpasses) / 1e9 / (best * 1e-3),
                   hc[0], hc[1]);
        }
        cudaFree(big);
        cudaFree(l2);
        cudaFree(cyc);
    }
    const cudaError_t err = cudaGetLastError();
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
