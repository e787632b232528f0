// common.cuh — shared helpers for the sm_100a kernels and the host runtime.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ihs_gpu.h"

namespace ihs_b200 {

// Exception carrying an ihs_status; converted to a status code at the C-ABI.
struct Status : std::runtime_error {
    ihs_status code;
    Status(ihs_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(ihs_status c, const std::string& m) { throw Status(c, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear a non-sticky error so later calls are not blamed for it
        fail(IHS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
    }
}
#define CUDA_CHECK(x) ::ihs_b200::cuda_check((x), #x, __FILE__, __LINE__)

// Every kernel launch of this library goes through LAUNCH so the count of
// native launches is observable (ihs_gpu_kernel_launch_count).
void note_launch();
// Programmatic dependent launch: the kernel may be scheduled while the previous kernel on the stream
// drains; it must execute griddepcontrol.wait (pdl_wait) before touching that kernel's results.
#define LAUNCH_PDL(kernel, grid, block, smem, strm_, ...)                                  \
    do {                                                                                 \
        cudaLaunchConfig_t cfg_{};                                                       \
        cfg_.gridDim = (grid);                                                           \
        cfg_.blockDim = (block);                                                         \
        cfg_.dynamicSmemBytes = (smem);                                                  \
        cfg_.stream = (strm_);                                                          \
        cudaLaunchAttribute at_[1];                                                      \
        at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                  \
        at_[0].val.programmaticStreamSerializationAllowed = 1;                           \
        cfg_.attrs = at_;                                                                \
        cfg_.numAttrs = 1;                                                               \
        CUDA_CHECK(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__));                      \
        ::ihs_b200::note_launch();                                                       \
    } while (0)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#define LAUNCH(kernel, grid, block, smem, stream, ...)                                   \
    do {                                                                                 \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                     \
        ::ihs_b200::note_launch();                                                       \
        CUDA_CHECK(cudaGetLastError());                                                  \
    } while (0)

// Opt a kernel into more than 48 KiB of dynamic shared memory. The attribute is per device, so the
// "already set" flag is a per-call-site bit mask over device ordinals (atomic: concurrent first calls from
// two threads both set it, which is harmless); a process that uses several devices sets it on each.
#define IHS_SMEM_ATTR(kernel, bytes)                                                                      \
    do {                                                                                                  \
        static std::atomic<uint64_t> ihs_attr_mask_{0};                                                   \
        int ihs_dev_ = 0;                                                                                 \
        CUDA_CHECK(cudaGetDevice(&ihs_dev_));                                                             \
        const uint64_t ihs_bit_ = 1ull << (ihs_dev_ & 63);                                                \
        if (!(ihs_attr_mask_.load(std::memory_order_acquire) & ihs_bit_)) {                               \
            CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))); \
            ihs_attr_mask_.fetch_or(ihs_bit_, std::memory_order_release);                                 \
        }                                                                                                 \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------ kernels API
// (implemented in the .cu files; all asynchronous on `st`)

// mt19937.cu — the reference RNG (rng.hpp:30-66) on the device
struct MTState { uint64_t mt[312]; };
void mt_seed_host(uint64_t seed, MTState& s);  // std::mt19937_64(seed) initial array
// raw draws [0, count) of mt19937_64(seed) (sequential single-CTA generator)
void mt_generate_raw(uint64_t seed, int64_t count, uint64_t* d_out, cudaStream_t st);
// rademacher sign bits: bit i = (draw_i & 1), 32-bit words LSB first; long
// vectors run as jump-ahead substreams (d_scratch: rademacher_scratch_bytes(n))
size_t rademacher_scratch_bytes(int64_t n);
void mt_rademacher_bits(uint64_t seed, int64_t n, uint32_t* d_bits, void* d_scratch, cudaStream_t st);
// polar.cu — the normal stream in two passes over jump-ahead substreams (count accepted attempts, scan, emit a
// window); any substream range, so a row shard generates only its share.
struct GaussPlan {
    int64_t draws;       // draws covering the stream
    int64_t big, fine;   // draws per jump-ahead (counting) substream, per emitting substream (fine divides big)
    int64_t nbig, nsub;  // counting substreams, emitting substreams
};
struct GaussScratch {
    uint64_t* jwin;      // start windows of jump substreams [j0, ...)
    uint64_t* fwin;      // start windows of emitting substreams [f0, ...) (= jwin when big == fine)
    uint64_t* xseq;
    long long* base;     // nsub + 1: first accepted attempt of each emitting substream (exclusive prefix)
    int* cnt;            // nsub accepted-attempt counts
    int64_t j0, f0;
};
GaussPlan gauss_plan(int64_t total_normals);
size_t gauss_scratch_bytes(const GaussPlan& g, int64_t nbig_win, int64_t nfine_win);
GaussScratch gauss_scratch(const GaussPlan& g, int64_t nbig_win, int64_t nfine_win, void* d_scratch);
void gauss_jump(uint64_t seed, const GaussPlan& g, int64_t bq0, int64_t bnq, GaussScratch& s, cudaStream_t st);
// counts of the emitting substreams inside jump substreams [bq0, bq0 + bnq); dump: also their start windows
void gauss_count(const GaussPlan& g, int64_t bq0, int64_t bnq, GaussScratch& s, bool dump, cudaStream_t st);
void gauss_scan(const GaussPlan& g, const GaussScratch& s, cudaStream_t st);
// start windows of emitting substreams [fq0, fq0 + fnq) (jump, plus a dump pass when big > fine)
void gauss_fine_windows(uint64_t seed, const GaussPlan& g, int64_t fq0, int64_t fnq, GaussScratch& s, cudaStream_t st);
void gauss_emit(const GaussPlan& g, int64_t fq0, int64_t fnq, const GaussScratch& s, int64_t first, int64_t count,
                double stddev, double* d_out, cudaStream_t st);
void gauss_window_range(const std::vector<long long>& h_base, int64_t first, int64_t count, int64_t* q0, int64_t* nq);
void gauss_counts_to_double(const GaussScratch& s, int64_t f0, int64_t nf, int64_t len, double* d_out, cudaStream_t st);
void gauss_counts_from_double(const double* d_in, const GaussPlan& g, const GaussScratch& s, cudaStream_t st);

// srht.cu — SRHT sketch SA = sqrt(n_pad/m) R H D A (sketch.hpp:77-108)
struct SrhtPlan {
    int64_t n, d, lda, n_pad, m;
    int64_t sa_ld;           // stride between SA columns (m; rows-per-owner for the sharded owner-block layout)
    int logn, L, H;          // n_pad = 2^logn, low bits L done in phase 1, H = logn - L
    int npass;               // phase-2 passes over the H high bits (<= 10 bits each)
    int pass_lo[3], pass_hb[3];
    double scale1, scale2;   // 1/sqrt(n_pad), sqrt(n_pad/m) (host-computed, :47 and :95)
    int p2t;                 // threads per phase-2 tile (128; 256 for the 64 KiB-tile variant)
    int compact;             // 1: compact T (only the sampled low indices; srht_plan_compact)
    int l2;                  // 1: L2-resident single launch (srht_plan_l2): T is a ring of l2_ns column slots
    int l2_ns;               // ring depth (column slots)
};
SrhtPlan srht_plan(int64_t n, int64_t d, int64_t lda, int64_t m);
// switch the plan to the streamed single-launch kernel when it applies (sets
// p2t before the entries are built); false = two-kernel path
// switch a two-kernel plan with 10 high bits (n_pad = 2^20) to compact T when the sample has few distinct
// low indices (U <= 640): phase 1 stores, per chunk, only the low indices some sampled row has
// (T[j][h][u]) and the emitting pass runs one warp per (u, column). Set before the entries are built (they then carry U tiles followed by the 1024-entry
// low-index -> u map).
bool srht_plan_compact(SrhtPlan& p, const int64_t* rows);
size_t srht_scratch_bytes(const SrhtPlan& p);  // T buffer (phase-1 output) when H > 0
// switch a single-pass plan with 8..12 high bits to the L2-resident single launch (sets p2t before the entries
// are built; the tiles then carry 4 trailing int4 of tile-occupancy bits); false = keep the plan
bool srht_plan_l2(SrhtPlan& p);
// T ring + control block of the L2-resident launch
size_t srht_l2_scratch_bytes(const SrhtPlan& p);
size_t srht_l2_ctl_bytes(const SrhtPlan& p);
// Host: bucket the sampled rows (draw order k -> row rows[k]) by phase-2
// tile. entries = (row, k) pairs grouped by tile; tiles = (rlo0, begin, end).
void srht_build_entries(const SrhtPlan& p, const int64_t* rows, std::vector<int2>& entries,
                        std::vector<int4>& tiles);
// p.l2 (srht_plan_l2) selects the L2-resident single launch: T is then a ring of srht_l2_scratch_bytes() and
// d_ctl its control block of srht_l2_ctl_bytes().
// d_mask (8 words, from srht_build_mask): phase 1 stores only the low-index
// groups the single emitting pass reads.
void srht_run_device(const SrhtPlan& p, const double* d_A, const uint32_t* d_signbits, const int2* d_entries,
                     const int4* d_tiles, int n_tiles, double* d_T, double* d_SA, cudaStream_t st,
                     unsigned long long* d_ctl = nullptr, int num_sms = 148, const uint32_t* d_mask = nullptr);
bool srht_build_mask(const SrhtPlan& p, const std::vector<int4>& tiles, uint32_t mask[8]);
// Row-sharded SRHT: plan of one shard (n_loc = n_pad / P rows, n_real of them
// real) that emits unscaled partials at r_lo(k) for all m sampled rows, and the
// combine of the P gathered partials ([P][m][d]) into SA (d_hi[k] = r_hi(k)).
SrhtPlan srht_plan_shard(int64_t n_real, int64_t n_loc, int64_t d, int64_t lda, int64_t m);
void srht_combine(const double* d_U, int P, int64_t m, int64_t d, const uint8_t* d_hi, double s1, double s2,
                  double* d_SA, cudaStream_t st);
// owner-block layout G[q][kk + j mq] (rows k = q mq + kk of owner q) -> SA[k + j m], k < m
void srht_unpack_blocks(const double* d_G, int P, int64_t mq, int64_t m, int64_t d, double* d_SA, cudaStream_t st);

// nccl_comm.cpp — collectives of the row-sharded path (NCCL loaded at run time)
void nccl_unique_id(uint8_t out[128]);
void* nccl_comm_create(const uint8_t id[128], int world, int rank);
void nccl_comm_destroy(void* comm);
// world_size emulated ranks of this process (out[r] = rank r's communicator; host threads drive the ranks)
void emu_comm_create(int world, void** out);
int comm_world(const void* comm);
int comm_rank(const void* comm);
void nccl_allreduce_sum(double* buf, size_t count, void* comm, cudaStream_t st);
void nccl_allgather(const double* send, double* recv, size_t count_per_rank, void* comm, cudaStream_t st);
// all-to-all: block p of send (count doubles) goes to rank p, block p of recv comes from rank p
void nccl_alltoall(const double* send, double* recv, size_t count_per_rank, void* comm, cudaStream_t st);

// gemm_f64.cu — DMMA (mma.sync m8n8k4 f64) GEMM
// C[M x N] (ldc) = alpha * op(A) * op(B) + beta * C ; op(A) is M x K, op(B) K x N.
// transA: A stored K x M col-major (lda); else M x K col-major. transB: B
// stored N x K; else K x N. lower_only: skip tiles strictly above diagonal.
// splitk > 1: deterministic split-K through d_work (splitk*M*N doubles).
void dgemm_batched(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                   int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta, double* C, int64_t ldc,
                   int64_t sC, int batch, cudaStream_t st);
void dgemm(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
           const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower_only, int splitk,
           double* d_work, cudaStream_t st);
// dgemm launched in block-row pieces (phase 0: the block rows of rows [row0, row1), no split-K reduction; phase 1:
// the reduction only); false when dgemm would not take the 128x128 kernel for this product
int64_t dgemm_row_block();
bool dgemm_rows(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower_only, int splitk,
                double* d_work, cudaStream_t st, int64_t row0, int64_t row1, int phase);
int64_t dgemm_col_block();
bool dgemm_cols(bool transA, bool transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splitk, double* d_work,
                cudaStream_t st, int64_t col0, int64_t col1, int phase);
int dgemm_pick_splitk(int64_t M, int64_t N, int64_t K, int num_sms, bool transA = false, bool transB = false,
                      bool lower_only = false);

// chol.cu — blocked Cholesky (lower, in place). d_info: int (0 ok, j+1 = failed pivot).
void cholesky_factor(double* d_H, int64_t n, int* d_info, cudaStream_t st);
// W = L^{-1} (lower) with W^T mirrored into the strict upper triangle; d_tmp holds (ceil(n/2) + 64)^2 doubles
void cholesky_invert(const double* d_L, int64_t n, double* d_W, double* d_tmp, cudaStream_t st);
size_t cholesky_solve_work_doubles(int64_t n);
// Z = L^{-T} L^{-1} R for nrhs columns (ld = n), two parallel triangular mat-vecs
void cholesky_solve_inv(const double* d_W, int64_t n, const double* d_R, double* d_Z, int nrhs, double* d_work,
                        cudaStream_t st);

// gradient.cu — fused g = A^T(Ax - b) + nu^2 x for 1 or 2 right-hand sides
struct GradPlan {
    int64_t n, d, lda;
    int R;          // rows per panel
    int grid;       // persistent CTAs
    size_t smem;
    int version;    // 5: register rows (row-major); 4: row-major panels; 3: TMA panels; 2: cp.async ring; 1: L2 re-read
    int stages;     // ring depth (v2/v3/v4)
    int grid_sms;   // SM count the plan was made for
    alignas(64) unsigned char tmap[128];  // CUtensorMap of A (v3)
};
GradPlan grad_plan(int64_t n, int64_t d, int64_t lda, int num_sms);
// upgrade a v2 plan to TMA panels over device matrix A (no-op when unavailable)
void grad_plan_attach_tma(GradPlan& p, const double* d_A);
// v4: row-major copy of A (contiguous panels, 1D bulk TMA); switches the plan
// to v4 when the geometry fits (the caller then keeps a row-major A)
bool grad_plan_use_rowmajor(GradPlan& p);
size_t grad_rm_smem(int64_t d, int R, int nrhs, int ns);
// Heavy-ball candidates formed inside the gradient pass (solver.hpp:182,190):
// nrhs 2 -> [x_polyak; x_gd], nrhs 1 -> x_gd; written to out (nrhs x d).
struct CandSpec {
    const double* x = nullptr;
    const double* xprev = nullptr;
    const double* gt = nullptr;
    double mu_p = 0.0, beta_p = 0.0, mu_gd = 0.0;
    double* out = nullptr;
};
// v5: register-resident rows for d <= 512 (row-major copy as well)
size_t grad_rr_smem(int64_t d, int R, int ns);
bool grad_rr_geometry(int64_t d, int64_t lda, int* R, int* ns);
void grad_rr_run(const GradPlan& p, const double* Arm, const double* b, const double* X, int nrhs, double* work,
                 cudaStream_t st, const CandSpec* cs = nullptr);
bool grad_rm_geometry(int64_t d, int64_t lda, int* R, int* ns);
// Arm[i * ldo + j] = A[i + j * lda] (i < rows, j < d); ldo = 0 means d
void transpose_to_rowmajor(const double* A, int64_t lda, int64_t rows, int64_t d, double* Arm, cudaStream_t st,
                           int64_t ldo = 0);
void grad_rm_run(const GradPlan& p, const double* Arm, const double* b, const double* X, int nrhs, double* work,
                 cudaStream_t st);
size_t grad_tma_smem(int64_t d, int R, int nrhs, int ns);
bool grad_tma_make_map(const double* A, int64_t lda, int64_t d, int R, void* map_out);
void grad_tma_run(const GradPlan& p, const double* b, const double* X, int nrhs, double* work, cudaStream_t st);
size_t grad_work_doubles(const GradPlan& p);
// X: nrhs vectors of d (ld = d); G out: nrhs vectors of d. cs != nullptr: X = cs->out is formed from the
// heavy-ball state first (inside the pass on the v5 kernel, else by candidates()).
void grad_run(const GradPlan& p, const double* d_A, const double* d_b, double nu2, const double* d_X, int nrhs,
              double* d_G, double* d_work, cudaStream_t st, const double* d_Arm = nullptr,
              const CandSpec* cs = nullptr);

// vecops.cu
// out[k*d..] for the heavy-ball candidates (solver.hpp:182,190), no FMA contraction:
//   xp = (x - mu_p*gt) + beta_p*(x - xprev) ;  xg = x - mu_gd*gt
void candidates(const double* x, const double* xprev, const double* gt, double mu_p, double beta_p, double mu_gd,
                int64_t d, double* xp, double* xg, cudaStream_t st);
void fixed_step(const double* x, const double* xprev, const double* step, double mu, double beta, int64_t d,
                double* xn, cudaStream_t st);
// deterministic dots: out[2*k] = g_k . gt_k, out[2*k+1] = g_k . g_k
void decrement_dots(const double* g, const double* gt, int64_t d, int nrhs, double* out, cudaStream_t st);

// cg.cu: CG / PCG recurrences (baselines.hpp:40-200) with a device-resident state
size_t cg_state_bytes();
int64_t cg_state_iter(const void* h_state);
bool cg_state_done(const void* h_state);
void cg_begin(const double* g0, const double* hx, double* r, double* p, double tol, int64_t d, void* state,
              double* resid, bool pcg, cudaStream_t st);
void cg_step(void* state, double* p, const double* hp, double* x, double* r, double* resid, int64_t base, int64_t d,
             bool pcg, cudaStream_t st);
void cg_dir(void* state, const double* z, const double* dots, double* p, int64_t d, bool first, cudaStream_t st);
// Woodbury pieces: u = SA g (m), z = (g - SA^T w) / nu2
void gemv_n(const double* A, int64_t M, int64_t N, int64_t lda, const double* x, int nrhs, int64_t ldx, double* y,
            int64_t ldy, cudaStream_t st);
void woodbury_finish(const double* SA, int64_t m, int64_t d, const double* g, const double* w, double nu2, int nrhs,
                     double* z, cudaStream_t st);
// tiled y = A x (64x64 CTA tiles, fixed-order chunk reduction by the last CTA
// of each row block, one launch); work: gemv_tiled_work_doubles, whose counter
// tail must be zeroed once by gemv_tiled_reset before the first use
size_t gemv_tiled_work_doubles(int64_t M, int64_t N);
// dots != nullptr (requires M == N): also the decrement dots x.y, x.x per RHS (like decrement_dots)
void gemv_tiled(const double* A, int64_t M, int64_t N, int64_t lda, const double* x, int nrhs, int64_t ldx, double* y,
                int64_t ldy, double* work, cudaStream_t st, double* dots = nullptr);
void gemv_tiled_reset(double* work, int64_t M, int64_t N, cudaStream_t st);
// y = H x for a symmetric k x k column-major H (one warp per output column), optional fused decrement dots
// (as gemv_tiled); work as gemv_tiled(k, k)
void symv_col(const double* H, int64_t k, const double* x, int nrhs, int64_t ldx, double* y, int64_t ldy,
              double* work, cudaStream_t st, double* dots = nullptr);
// Wl = lower triangle of W (upper zeroed), k x k
void tril_copy(const double* W, int64_t k, double* Wl, cudaStream_t st);
void add_diag(double* H, int64_t n, double v, cudaStream_t st);
void add_scaled(double* y, const double* x, double a, int64_t n, cudaStream_t st);  // y = y + a x
void check_finite(const double* v, int64_t count, int* d_flag, cudaStream_t st);

}  // namespace ihs_b200
