// grad_tma.cu — fused gradient with TMA-fed panels (sm_100a).
//
// Same math and reduction order as grad_smem_kernel (gradient.cu): per R-row
// panel, sweep 1 forms r = A_p x - b_p from shared memory and sweep 2
// accumulates A_p^T r into register column partials. The difference is the
// copy engine: one elected thread issues 2D TMA boxes (cp.async.bulk.tensor)
// of R rows x BOXC columns per stage, completion is tracked by an mbarrier
// per stage (expect_tx), so the LSU/MIO queue only carries the sweeps' shared
// loads. Stages are released by the CTA barrier that ends each panel.
#include "common.cuh"
#include "tma.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace ihs_b200 {

namespace {
constexpr int TT = 512;  // threads
constexpr int TW = TT / 32;
constexpr int BOXC = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Offset (in doubles) of row pair h of panel column j under the TMA swizzle
// of RR-row (RR*8-byte) box rows: 16-byte chunk h is stored at h ^ f(j),
// f(j) = address bits [7, 7+log2(RR/2)) of j*RR*8 (SWIZZLE_32B/64B/128B).
template <int RR>
__device__ __forceinline__ int64_t swz(int64_t j, int h) {
    constexpr int HP = RR / 2;
    const int f = (int)((j * RR / 16) & (HP - 1));
    return j * RR + 2 * (h ^ f);
}

template <int NRHS, int RR, int MAXC, int NS>
__global__ void __launch_bounds__(TT, 1)
grad_tma_kernel(const __grid_constant__ CUtensorMap tmap, int64_t d, int64_t npanels, const double* __restrict__ b,
                const double* __restrict__ X, double* __restrict__ work) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    extern __shared__ __align__(1024) double sm_raw[];
    // swizzled TMA destinations need 1024-byte aligned stages
    double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int nbox = (int)((d + BOXC - 1) / BOXC);
    const int64_t stage = (int64_t)nbox * BOXC * RR;  // doubles per stage (box-padded, multiple of 1024 B)
    double* panel = sm;
    double* xs = panel + NS * stage;
    double* red = xs + NRHS * d;
    double* rv = red + TW * NRHS * RR;
    uint64_t* full = reinterpret_cast<uint64_t*>(rv + NRHS * RR + 8);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t stage_bytes = (uint32_t)(stage * sizeof(double));

    if (t == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // x interleaved by right-hand side: xs[j * NRHS + q] (one 128-bit load feeds both)
    for (int64_t e = t; e < NRHS * d; e += TT) {
        const int64_t q = e / d, j = e % d;
        xs[j * NRHS + q] = X[e];
    }
    __syncthreads();

    auto issue = [&](int64_t p, int s) {  // thread 0 only
        if (p >= npanels) return;
        mbar_expect_tx(&full[s], stage_bytes);
        for (int bx = 0; bx < nbox; ++bx)
            tma_load_2d(panel + s * stage + (int64_t)bx * BOXC * RR, &tmap, (int)(p * RR), bx * BOXC, &full[s]);
    };
    int64_t p = blockIdx.x;
    if (t == 0)
        for (int k = 0; k < NS; ++k) issue(p + (int64_t)k * gridDim.x, k);

    double gacc[NRHS][MAXC];
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) gacc[q][c] = 0.0;

    int s = 0;
    uint32_t phase = 0;
    for (; p < npanels; p += gridDim.x) {
        mbar_wait(&full[s], phase);
        const double* P = panel + s * stage;
        // ---- sweep 1: r = A_p x - b_p ; thread = (row pair h, column group jg)
        {
            constexpr int HP = RR / 2;  // row pairs per panel
            const int h = t % HP;
            const int jg = t / HP;
            constexpr int G = TT / HP;
            double acc[2][NRHS];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int q = 0; q < NRHS; ++q) acc[u][q] = 0.0;
#pragma unroll 4
            for (int64_t j = jg; j < d; j += G) {
                const double2 a = *reinterpret_cast<const double2*>(P + swz<RR>(j, h));
                if constexpr (NRHS == 2) {
                    const double2 xv = *reinterpret_cast<const double2*>(xs + 2 * j);
                    acc[0][0] = fma(a.x, xv.x, acc[0][0]);
                    acc[0][1] = fma(a.x, xv.y, acc[0][1]);
                    acc[1][0] = fma(a.y, xv.x, acc[1][0]);
                    acc[1][1] = fma(a.y, xv.y, acc[1][1]);
                } else {
                    const double xv = xs[j];
                    acc[0][0] = fma(a.x, xv, acc[0][0]);
                    acc[1][0] = fma(a.y, xv, acc[1][0]);
                }
            }
#pragma unroll
            for (int off = HP; off < 32; off <<= 1)
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) acc[u][q] += __shfl_xor_sync(0xffffffffu, acc[u][q], off);
            if (lane < HP)
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) red[(warp * NRHS + q) * RR + 2 * lane + u] = acc[u][q];
        }
        __syncthreads();
        if (t < NRHS * RR) {
            const int q = t / RR, i = t % RR;
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < TW; ++w) sum += red[(w * NRHS + q) * RR + i];
            rv[q * RR + i] = sum - b[p * RR + i];
        }
        __syncthreads();
        // ---- sweep 2: g += A_p^T r ; r in registers, 128-bit row-pair loads
        // (TMA swizzle: the 8 lanes of a 128-bit phase hit distinct chunks)
        {
            double r[NRHS][RR];
#pragma unroll
            for (int q = 0; q < NRHS; ++q)
#pragma unroll
                for (int i = 0; i < RR; ++i) r[q][i] = rv[q * RR + i];
            constexpr int HP = RR / 2;
#pragma unroll
            for (int c = 0; c < MAXC; ++c) {
                const int64_t j = t + (int64_t)c * TT;
                if (j < d) {
                    double sum[NRHS];
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) sum[q] = 0.0;
#pragma unroll
                    for (int hh = 0; hh < HP; ++hh) {
                        const double2 a = *reinterpret_cast<const double2*>(P + swz<RR>(j, hh));
#pragma unroll
                        for (int q = 0; q < NRHS; ++q) {
                            sum[q] = fma(a.x, r[q][2 * hh], sum[q]);
                            sum[q] = fma(a.y, r[q][2 * hh + 1], sum[q]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) gacc[q][c] += sum[q];
                }
            }
        }
        __syncthreads();  // stage s fully consumed: refill it
        if (t == 0) issue(p + (int64_t)NS * gridDim.x, s);
        if (++s == NS) {
            s = 0;
            phase ^= 1;
        }
    }
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int64_t j = t + (int64_t)c * TT;
            if (j < d) work[((int64_t)blockIdx.x * NRHS + q) * d + j] = gacc[q][c];
        }
}

}  // namespace

PFN_cuTensorMapEncodeTiled tma_encode_fn() {
    static PFN_cuTensorMapEncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) fail(IHS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
    }();
    return fn;
}

size_t grad_tma_smem(int64_t d, int R, int nrhs, int ns) {
    const int64_t nbox = (d + BOXC - 1) / BOXC;
    return sizeof(double) * ((size_t)ns * nbox * BOXC * R + (size_t)nrhs * d + (size_t)TW * nrhs * R + (size_t)nrhs * R +
                             8) +
           (size_t)ns * 8 + 1024 + 128;
}

bool grad_tma_make_map(const double* A, int64_t lda, int64_t d, int R, void* map_out /* CUtensorMap, 128 B */) {
    CUtensorMap* m = static_cast<CUtensorMap*>(map_out);
    const cuuint64_t dims[2] = {(cuuint64_t)lda, (cuuint64_t)d};
    const cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)BOXC};
    const cuuint32_t estr[2] = {1, 1};
    // a box row is R doubles (one panel column): swizzle span = R*8 bytes
    const CUtensorMapSwizzle sw = R == 16 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : R == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : R == 4 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (sw == CU_TENSOR_MAP_SWIZZLE_NONE) return false;
    const CUresult r = tma_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int NRHS, int RR, int NS>
void launch_tma(const GradPlan& p, const double* b, const double* X, double* work, cudaStream_t st) {
    const size_t smem = grad_tma_smem(p.d, RR, NRHS, NS);
    const int maxc = (int)ceil_div(p.d, TT);
    const CUtensorMap* map = reinterpret_cast<const CUtensorMap*>(p.tmap);
#define IHS_TMA(MC)                                                                                                 \
    do {                                                                                                            \
        IHS_SMEM_ATTR((grad_tma_kernel<NRHS, RR, MC, NS>), 227 * 1024);                                                                                                           \
        LAUNCH_PDL((grad_tma_kernel<NRHS, RR, MC, NS>), p.grid, TT, smem, st, *map, p.d, p.lda / RR, b, X, work);       \
    } while (0)
    if (maxc <= 1) IHS_TMA(1);
    else if (maxc <= 2) IHS_TMA(2);
    else IHS_TMA(4);
#undef IHS_TMA
}

void grad_tma_run(const GradPlan& p, const double* b, const double* X, int nrhs, double* work, cudaStream_t st) {
    const int key = p.R * 10 + p.stages;
    if (nrhs == 1) {
        switch (key) {
            case 163: launch_tma<1, 16, 3>(p, b, X, work, st); return;
            case 164: launch_tma<1, 16, 4>(p, b, X, work, st); return;
            case 83: launch_tma<1, 8, 3>(p, b, X, work, st); return;
            case 84: launch_tma<1, 8, 4>(p, b, X, work, st); return;
            case 43: launch_tma<1, 4, 3>(p, b, X, work, st); return;
            case 42: launch_tma<1, 4, 2>(p, b, X, work, st); return;
        }
    } else {
        switch (key) {
            case 163: launch_tma<2, 16, 3>(p, b, X, work, st); return;
            case 164: launch_tma<2, 16, 4>(p, b, X, work, st); return;
            case 83: launch_tma<2, 8, 3>(p, b, X, work, st); return;
            case 84: launch_tma<2, 8, 4>(p, b, X, work, st); return;
            case 43: launch_tma<2, 4, 3>(p, b, X, work, st); return;
            case 42: launch_tma<2, 4, 2>(p, b, X, work, st); return;
        }
    }
    fail(IHS_INTERNAL_ERROR, "gradient (TMA): no kernel for the chosen panel geometry");
}

}  // namespace ihs_b200
