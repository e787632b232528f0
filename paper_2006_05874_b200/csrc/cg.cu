// cg.cu — device side of the CG / sketch-preconditioned CG baselines
// (proj/include/ihs/baselines.hpp:40-200).
//
// The H p products are the gradient pass over A with a zero observation vector
// (A^T(A p - 0) + nu^2 p, one HBM pass, grad_run); everything else on the
// d-vectors runs in single-CTA kernels that keep the recurrence scalars (rz,
// the stopping target, the iteration count, a done flag) in a device-resident
// CgState, so the host enqueues batches of iterations without reading any
// scalar back. Once an iteration meets the stopping rule the flag turns every
// later step of the batch into a no-op, so x, r and the residual trace are
// exactly those of the iteration count the reference would stop at.
// Reductions are fixed-order (thread -> element map, warp butterflies, one
// warp over the 32 partials): deterministic run to run.
#include "common.cuh"

namespace ihs_b200 {
namespace {

constexpr int CG_T = 1024;

struct CgState {
    double rz;      // r.r (CG) or r.z (PCG) of the current direction
    double target;  // tol * ||A^T b||
    int64_t iter;   // iterations taken
    int32_t done;   // stopping rule met
    int32_t pad;
};

// block-wide sum; every thread returns the same value
__device__ double cg_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();  // red[] of the previous reduction has been read
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

// atb = -g0 (g0 = A^T(A 0 - b) + nu^2 0 = -A^T b exactly); r = atb - H x0 (or atb for a zero start);
// residual[0] = ||r||, target = tol ||atb|| (baselines.hpp:55-66, :126-137); CG: p = r, rz = r.r
__global__ void __launch_bounds__(CG_T) cg_begin_kernel(const double* __restrict__ g0, const double* __restrict__ hx,
                                                        double* __restrict__ r, double* __restrict__ p, double tol,
                                                        int64_t d, CgState* __restrict__ s, double* __restrict__ resid,
                                                        int pcg) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double red[32];
    double sa = 0.0, sr = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
        const double atb = -g0[i];
        const double ri = hx ? atb - hx[i] : atb;
        r[i] = ri;
        if (!pcg) p[i] = ri;
        sa = fma(atb, atb, sa);
        sr = fma(ri, ri, sr);
    }
    const double na = cg_block_sum(sa, red);
    const double nr = cg_block_sum(sr, red);
    if (threadIdx.x == 0) {
        const double rn = sqrt(nr);
        s->target = tol * sqrt(na);
        s->iter = 0;
        s->done = rn <= s->target;
        s->rz = nr;
        resid[0] = rn;
    }
}

// one iteration after hp = H p (baselines.hpp:71-87 / :140-156): alpha = rz/(p.hp), x += alpha p,
// r -= alpha hp, residual, stopping rule; CG also forms the next direction p = r + (r.r/rz) p
__global__ void __launch_bounds__(CG_T) cg_step_kernel(CgState* __restrict__ s, double* __restrict__ p,
                                                       const double* __restrict__ hp, double* __restrict__ x,
                                                       double* __restrict__ r, double* __restrict__ resid,
                                                       int64_t base, int64_t d, int pcg) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    __shared__ double red[32];
    if (s->done) return;
    const double rz = s->rz, target = s->target;
    const int64_t it = s->iter + 1;
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) a = fma(p[i], hp[i], a);
    const double alpha = rz / cg_block_sum(a, red);
    double q = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
        x[i] = x[i] + alpha * p[i];
        const double ri = r[i] - alpha * hp[i];
        r[i] = ri;
        q = fma(ri, ri, q);
    }
    const double ss = cg_block_sum(q, red);  // its barriers order every read of *s before the writes below
    const double rn = sqrt(ss);
    if (threadIdx.x == 0) {
        resid[it - base] = rn;
        s->iter = it;
        if (rn <= target) s->done = 1;
    }
    if (rn <= target || pcg) return;
    const double beta = ss / rz;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) p[i] = r[i] + beta * p[i];
    if (threadIdx.x == 0) s->rz = ss;
}

// PCG direction after z = M^{-1} r (dots[0] = r.z from the mat-vec's fused dot):
// p = z (first) or z + (rz_new/rz) p (baselines.hpp:133-135, :160-163)
__global__ void __launch_bounds__(CG_T) cg_dir_kernel(CgState* __restrict__ s, const double* __restrict__ z,
                                                      const double* __restrict__ dots, double* __restrict__ p,
                                                      int64_t d, int first) {
    pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible after this
    if (s->done) return;
    const double rz_new = dots[0];
    const double beta = first ? 0.0 : rz_new / s->rz;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) p[i] = first ? z[i] : z[i] + beta * p[i];
    __syncthreads();  // every thread has read s->rz
    if (threadIdx.x == 0) s->rz = rz_new;
}

}  // namespace

size_t cg_state_bytes() { return sizeof(CgState); }
int64_t cg_state_iter(const void* h_state) { return static_cast<const CgState*>(h_state)->iter; }
bool cg_state_done(const void* h_state) { return static_cast<const CgState*>(h_state)->done != 0; }

void cg_begin(const double* g0, const double* hx, double* r, double* p, double tol, int64_t d, void* state,
              double* resid, bool pcg, cudaStream_t st) {
    LAUNCH_PDL(cg_begin_kernel, 1, CG_T, 0, st, g0, hx, r, p, tol, d, static_cast<CgState*>(state), resid, (int)pcg);
}

void cg_step(void* state, double* p, const double* hp, double* x, double* r, double* resid, int64_t base, int64_t d,
             bool pcg, cudaStream_t st) {
    LAUNCH_PDL(cg_step_kernel, 1, CG_T, 0, st, static_cast<CgState*>(state), p, hp, x, r, resid, base, d, (int)pcg);
}

void cg_dir(void* state, const double* z, const double* dots, double* p, int64_t d, bool first, cudaStream_t st) {
    LAUNCH_PDL(cg_dir_kernel, 1, CG_T, 0, st, static_cast<CgState*>(state), z, dots, p, d, (int)first);
}

}  // namespace ihs_b200
