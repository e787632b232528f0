/*
 * ihs_gpu.h — C-ABI of the B200-native adaptive IHS hot path.
 *
 * This is the drop-in boundary for the reference's header-only C++ solver API
 * (/root/reference/proj/include/ihs/ headers). The reference has no FFI of its
 * own; every entry point below replaces one reference function and cites it.
 * The C++ shim `include/ihs_b200.hpp` (namespace ihs, reference signatures)
 * and the Python mirror `paper_2006_05874_b200/ihs.py` both sit on top of it.
 *
 * Conventions
 *   - plain pointers + sizes, no torch/Eigen types; matrices are column-major
 *     (Eigen's default, reference types.hpp:10) with an explicit leading dim.
 *   - host buffers are caller-owned; device state lives in opaque handles.
 *   - every function returns an ihs_status; the message of the last failure on
 *     the calling thread is available from ihs_gpu_last_error().
 *   - status codes map 1:1 onto the reference exception types
 *     (errors.hpp:15-40): InvalidInput, OutOfValidityRange, SketchTooLarge,
 *     NumericalBreakdown. CUDA/NCCL failures get their own codes.
 */
#ifndef IHS_GPU_H
#define IHS_GPU_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ihs_status {
    IHS_OK = 0,
    IHS_INVALID_INPUT = 1,          /* ihs::InvalidInput        errors.hpp:15 */
    IHS_OUT_OF_VALIDITY_RANGE = 2,  /* ihs::OutOfValidityRange  errors.hpp:23 */
    IHS_SKETCH_TOO_LARGE = 3,       /* ihs::SketchTooLarge      errors.hpp:30 */
    IHS_NUMERICAL_BREAKDOWN = 4,    /* ihs::NumericalBreakdown  errors.hpp:37 */
    IHS_CUDA_ERROR = 5,
    IHS_NCCL_ERROR = 6,
    IHS_INTERNAL_ERROR = 7
} ihs_status;

/* sketch.hpp:16 */
typedef enum ihs_sketch_kind { IHS_SKETCH_GAUSSIAN = 0, IHS_SKETCH_SRHT = 1 } ihs_sketch_kind;
/* solver.hpp:19-22 */
typedef enum ihs_solve_mode { IHS_MODE_POLYAK_THEN_GRADIENT = 0, IHS_MODE_GRADIENT_ONLY = 1 } ihs_solve_mode;
/* solver.hpp:24 */
typedef enum ihs_step_kind { IHS_STEP_POLYAK = 0, IHS_STEP_GRADIENT = 1, IHS_STEP_RESKETCH = 2 } ihs_step_kind;
/* sketched_system.hpp:12 */
typedef enum ihs_factor_kind { IHS_FACTOR_WOODBURY_INNER = 0, IHS_FACTOR_DIRECT_GRAM = 1 } ihs_factor_kind;
/* problem.hpp:13 */
typedef enum ihs_orientation { IHS_OVERDETERMINED = 0, IHS_UNDERDETERMINED = 1 } ihs_orientation;
/* solver.hpp:252 */
typedef enum ihs_fixed_mode { IHS_FIXED_GRADIENT = 0, IHS_FIXED_POLYAK = 1 } ihs_fixed_mode;

/* types.hpp:18-33 — analytic multiply-add counters, exact closed forms. */
typedef struct ihs_counters {
    uint64_t sketch;
    uint64_t factor;
    uint64_t solve;
    uint64_t matvec;
} ihs_counters;

/* tuning.hpp:13-21 */
typedef struct ihs_tuning {
    double lam, Lam, mu_gd, c_gd, mu_p, beta_p, c_p;
} ihs_tuning;

/* SolverConfig::sketch_override (solver.hpp:56): host callback that fills the
 * m x d column-major sketch of the problem's matrix (ld = m). The callback
 * receives the sub-seed derive_seed(cfg.seed, K) exactly like the reference
 * (solver.hpp:102,139,212). Return 0 on success; non-zero aborts the solve
 * with IHS_INVALID_INPUT. As in the reference, the override skips the sketch
 * counters. */
typedef int (*ihs_sketch_override_fn)(void* user, int64_t m, uint64_t sub_seed, double* SA_out);

/* SolverConfig (solver.hpp:28-57). Optional fields use explicit flags. */
typedef struct ihs_solver_config {
    double rho;                     /* 0.1  */
    double eta;                     /* 0.01 */
    int32_t sketch_kind;            /* ihs_sketch_kind, default Gaussian */
    int32_t mode;                   /* ihs_solve_mode */
    int64_t m_initial;              /* 1 */
    double eps;                     /* 1e-10 */
    int64_t max_iters;              /* 500 */
    int64_t max_sketch;             /* std::optional<Index>: <= 0 means unset */
    uint64_t seed;                  /* 0 */
    int32_t enforce_validity;       /* 1 */
    int32_t recompute_r_after_resketch; /* 1 */
    int32_t record_iterates;        /* 0 */
    int32_t has_tuning_override;    /* 0 */
    ihs_tuning tuning_override;
    const double* warm_start;       /* NULL = zero start; else d doubles (host) */
    ihs_sketch_override_fn sketch_override; /* NULL = none */
    void* sketch_override_user;
} ihs_solver_config;

/* IterationRecord (solver.hpp:62-68) */
typedef struct ihs_iteration_record {
    int64_t t;
    int64_t m;
    double r;
    double r_prev;
    int32_t branch;                 /* ihs_step_kind */
    int32_t _pad;
} ihs_iteration_record;

/* Per-phase device time of one solve (CUDA events on the solve stream). */
typedef struct ihs_phase_times {
    double sketch_ms;     /* D/P/S generation + sketch kernels */
    double factor_ms;     /* SYRK + Cholesky */
    double gradient_ms;   /* fused gradient kernels (+ collective) */
    double solve_ms;      /* triangular / Woodbury solves + decrement */
    int64_t n_sketch, n_factor, n_gradient, n_solve; /* n_gradient counts passes over A */
    int64_t kernel_launches; /* kernels this library launched during the solve */
    double total_ms;      /* CUDA-event time of the whole solve on the device timeline */
    double gradient_bytes; /* algorithmic HBM bytes of all gradient passes (8nd + 8n each) */
    double sketch_bytes;   /* algorithmic bytes of the SRHT sketches (8nd + 8md each) */
    double sketch_flops;   /* algorithmic flops of the Gaussian sketches (2mnd each) */
    double alloc_ms;       /* host time spent growing device buffers */
    double host_rng_ms;    /* host time drawing the SRHT row samples (Fisher-Yates) */
    double sketch_kernel_ms; /* device time of the sketch's main kernels alone (SRHT transform
                                kernels / the S*A DMMA GEMM), part of sketch_ms */
    int64_t n_sketch_kernel; /* number of such sketch-kernel intervals */
    double gradient_kernel_ms; /* device time of the gradient kernels alone (pass over A + fixed-order
                                  reduce), part of gradient_ms */
    int64_t n_gradient_kernel; /* number of gradient passes timed */
    int64_t n_srht_l2;         /* SRHT sketches run as the L2-resident single launch */
    int64_t n_srht_compact;    /* ... as the compact two-kernel path (n_pad = 2^20, small m) */
    int64_t n_srht_two_kernel; /* ... as the two-kernel (HBM round trip of T) or multi-pass path */
} ihs_phase_times;

/* SolveReport (solver.hpp:70-87). Arrays are caller-allocated; *_size is the
 * number of entries the solver produced (it may exceed *_capacity, in which
 * case only the first *_capacity entries were written). */
typedef struct ihs_solve_report {
    double* x;                      /* d doubles, caller-allocated (required) */
    int64_t iterations;
    int64_t rejections;
    int64_t final_m;
    double r1;
    double r_final;
    int32_t converged;
    int32_t sketch_exhausted;
    ihs_iteration_record* log;      /* may be NULL */
    int64_t log_capacity;
    int64_t log_size;
    double* iterates;               /* d * iterates_capacity doubles, may be NULL */
    int64_t iterates_capacity;
    int64_t iterates_size;
    ihs_counters counters;
    double wall_seconds;
    ihs_tuning tuning;
    int32_t recompute_r_after_resketch;
    int32_t _pad;
    ihs_phase_times times;          /* device-side breakdown (GPU only) */
    double* dual_final;             /* n doubles, caller-allocated, may be NULL: final dual iterate z_T of
                                       solve_underdetermined (solver.hpp:82); iterates then hold the dual trace */
} ihs_solve_report;

/* CgResult / PcgResult (baselines.hpp:16-36). residuals is caller-allocated
 * (residuals_capacity entries, may be NULL); residuals_size = iterations + 1
 * values were produced (only the first residuals_capacity written). */
typedef struct ihs_cg_report {
    double* x;                      /* d doubles, caller-allocated (required) */
    double* residuals;              /* ||H x_k - A^T b||, k = 0..iterations */
    int64_t residuals_capacity;
    int64_t residuals_size;
    int64_t iterations;
    int32_t converged;
    int32_t m_capped;               /* PCG: prescription exceeded n_pad and was capped */
    int64_t m;                      /* PCG: sketch rows used (0 for CG) */
    uint64_t setup_flops;           /* PCG: sketch + gram + Cholesky counter */
    ihs_counters counters;
    double wall_seconds;
    double device_ms;               /* GPU: CUDA-event time of the solve on the device timeline */
    int64_t kernel_launches;        /* GPU: kernels this library launched during the solve */
    ihs_phase_times times;          /* GPU: per-phase device time (sketch, factor, H p passes, recurrences) */
} ihs_cg_report;

/* Device / sharding options of a problem handle. */
typedef struct ihs_gpu_options {
    int32_t device;                 /* CUDA device ordinal */
    int32_t world_size;             /* 1 = single GPU */
    int32_t rank;
    int32_t _pad;
    void* nccl_comm;                /* ncclComm_t when world_size > 1, else NULL */
    int64_t n_global;               /* rows of the full problem (== n when world_size == 1) */
    int64_t row_offset;             /* first global row held by this rank */
} ihs_gpu_options;

typedef struct ihs_gpu_problem ihs_gpu_problem;
typedef struct ihs_gpu_system ihs_gpu_system;

/* ---------------------------------------------------------------- library */
const char* ihs_gpu_last_error(void);
const char* ihs_gpu_version(void);
/* number of kernels launched by this library in the calling process */
int64_t ihs_gpu_kernel_launch_count(void);
int ihs_gpu_device_count(void);

/* ------------------------------------------------------- host-side scalars
 * tuning.hpp:25-63 — pure host math, exported so every front end shares it. */
ihs_status ihs_rates_from_bounds(double lam, double Lam, ihs_tuning* out);
ihs_status ihs_gaussian_targets(double rho, double eta, int enforce_validity, double* lam, double* Lam);
ihs_status ihs_srht_targets(double rho, double* lam, double* Lam);
uint64_t ihs_derive_seed(uint64_t seed, uint64_t tag);   /* rng.hpp:23-28 */
int64_t ihs_next_pow2(int64_t n);                        /* sketch.hpp:26-28 */
void ihs_solver_config_default(ihs_solver_config* cfg);  /* solver.hpp:28-57 defaults */

/* ------------------------------------------------------- row sharding
 * H_{n_pad} = H_P (x) H_{n_pad/P}: rank r of P owns rows [r*n_loc, (r+1)*n_loc)
 * of the padded index space, n_loc = next_pow2(n_global)/P.
 * A sharded problem is created with ihs_gpu_problem_create on the local rows
 * and opts {world_size, rank, nccl_comm, n_global, row_offset}; the SRHT
 * partials are all-gathered and combined in the reference's butterfly order
 * (bit-exact), gradient and Gaussian-sketch partials are summed (NCCL). */
ihs_status ihs_gpu_shard_rows(int64_t n_global, int32_t world_size, int32_t rank, int64_t* row0, int64_t* rows);
ihs_status ihs_gpu_nccl_unique_id(uint8_t out[128]);
ihs_status ihs_gpu_nccl_comm_create(const uint8_t id[128], int32_t world_size, int32_t rank, int32_t device,
                                    void** comm);
void ihs_gpu_nccl_comm_destroy(void* comm);
/* Self-test of the sharded path's collectives (all-reduce sum, all-gather, all-to-all) on exact fp64 patterns:
 * *mismatches = wrong elements of this rank's results (0 on success). Any world size, NCCL or emulated. */
ihs_status ihs_gpu_comm_selftest(void* comm, int32_t device, int64_t count, int64_t* mismatches);
/* world_size EMULATED ranks of this process (comms[r] for rank r; free each with ihs_gpu_nccl_comm_destroy):
 * the row-sharded code runs unchanged with one host thread per rank, collectives become host barriers plus
 * device copies ordered by events (tests and single-GPU development of the sharded path). */
ihs_status ihs_gpu_emu_comm_create(int32_t world_size, int32_t device, void** comms);
/* MT19937-64 draws the calling thread's Gaussian sketches have generated so far (count and emission passes over
 * whole substreams): a row shard's share of the stream's generation work. */
int64_t ihs_gpu_thread_generated_draws(void);
/* Doublings (beyond the first sketch) that adaptive solves of the calling thread have sketched chunk by chunk behind
 * a chunked asynchronous upload of A (the speculative builds of ihs_gpu_problem_upload_async + adaptive_solve). */
int64_t ihs_gpu_thread_upload_doublings(void);
/* Rows of sketched Gram matrices SA^T SA that those solves enqueued block row by block row behind the upload
 * (the factorization then only reduces the split-K partials). */
int64_t ihs_gpu_thread_upload_gram_rows(void);
/* The sharded SRHT decomposition run back to back on one device (P virtual
 * shards of a single-GPU problem): proves the decomposition bit-exact. */
ihs_status ihs_gpu_sketch_sharded_emulated(ihs_gpu_problem* p, int32_t kind, int64_t m, uint64_t seed,
                                           int32_t shards, double* SA_out);

/* ------------------------------------------------------- problem (device) */
/* ProblemInstance (problem.hpp:20-55): validates like the reference, uploads A
 * (n x d, column-major, leading dim lda) and b to the device once. */
ihs_status ihs_gpu_problem_create(const double* A, int64_t n, int64_t d, int64_t lda,
                                  const double* b, double nu, int32_t orientation,
                                  const ihs_gpu_options* opts, ihs_gpu_problem** out);
void ihs_gpu_problem_destroy(ihs_gpu_problem* p);
int64_t ihs_gpu_problem_rows(const ihs_gpu_problem* p);
int64_t ihs_gpu_problem_cols(const ihs_gpu_problem* p);
/* re-upload A/b in place (same shape), e.g. for an end-to-end timed step */
ihs_status ihs_gpu_problem_upload(ihs_gpu_problem* p, const double* A, int64_t lda, const double* b);
/* Asynchronous re-upload: enqueues the copies of A / b (and the device row-major copy) on the problem's
 * side stream and returns; the next call on the problem orders its first A-reading kernel after them, so
 * A-independent work (Gaussian sketch RNG, SRHT signs and row sample) overlaps the transfer. The host
 * buffers (pinned for a true overlap) must stay valid until the next call on the problem returns. */
ihs_status ihs_gpu_problem_upload_async(ihs_gpu_problem* p, const double* A, int64_t lda, const double* b);
/* Per-phase CUDA-event timing of adaptive solves on this problem (ihs_phase_times; default on).
 * The events cost host time on the solve's critical path, so timed benchmark runs switch them off. */
ihs_status ihs_gpu_problem_set_phase_timing(ihs_gpu_problem* p, int32_t enabled);

/* Change nu of a resident problem (ProblemInstance checks, problem.hpp:24-32) without re-uploading A:
 * the regularization path solves one A at a decreasing sequence of nu (bench.hpp:131-171). */
ihs_status ihs_gpu_problem_set_nu(ihs_gpu_problem* p, double nu);
/* direct_solve (problem.hpp:73-82): the exact ridge minimizer (d doubles), computed on the device
 * from the Gram matrix of the resident A (DMMA), its Cholesky factor and iterative refinement with
 * the fused gradient pass; underdetermined instances through the kernel form x = A^T (A A^T + nu^2 I)^{-1} b. */
ihs_status ihs_gpu_direct_solve(ihs_gpu_problem* p, double* x_out);

/* gradient (problem.hpp:59-69): g = A^T(Ax - b) + nu^2 x, host in/out. */
ihs_status ihs_gpu_gradient(ihs_gpu_problem* p, const double* x, double* g, ihs_counters* counters);

/* apply_sketch / gaussian_sketch / srht_sketch (sketch.hpp:58-117) on the
 * problem's A. SA_out: m x d column-major host buffer (ld = m). */
ihs_status ihs_gpu_sketch(ihs_gpu_problem* p, int32_t kind, int64_t m, uint64_t seed,
                          double* SA_out, ihs_counters* counters);

/* ------------------------------------------------ stand-alone sketch ops */
/* fwht_inplace (sketch.hpp:33-49) on a host vector, computed on the device. */
ihs_status ihs_gpu_fwht(double* v, int64_t n);
/* srht_sketch / gaussian_sketch of an arbitrary host matrix (uploads it). */
ihs_status ihs_gpu_sketch_matrix(const double* A, int64_t n, int64_t d, int64_t lda, int32_t kind,
                                 int64_t m, uint64_t seed, double* SA_out, ihs_counters* counters);

/* ------------------------------------- the reference RNG, generated on GPU */
/* rademacher (rng.hpp:48-52) of mt19937_64(stream_seed): bit i of out (LSB
 * first in 32-bit words) is 1 iff entry i is +1. */
ihs_status ihs_gpu_rademacher_bits(uint64_t stream_seed, int64_t n, uint32_t* out_bits);
/* fill_gaussian (rng.hpp:35-40) of a rows x cols column-major matrix. */
ihs_status ihs_gpu_fill_gaussian(uint64_t stream_seed, int64_t rows, int64_t cols, double stddev,
                                 double* out);
/* normals [first, first + count) of the same stream (a row shard's window of S); streamed != 0 runs the
 * chunked generator of tall Gaussian sketches (blocks of `block` >= 2 normals) */
ihs_status ihs_gpu_fill_gaussian_window(uint64_t stream_seed, int64_t first, int64_t count, double stddev,
                                        int32_t streamed, int64_t block, double* out);
/* raw mt19937_64(stream_seed) draws 0..count-1 (device generator) */
ihs_status ihs_gpu_mt19937_64(uint64_t stream_seed, int64_t count, uint64_t* out);
/* sample_without_replacement (rng.hpp:56-66), host-side sparse Fisher-Yates */
ihs_status ihs_sample_without_replacement(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out);

/* -------------------------------------------------- sketched system */
/* SketchedSystem::factorize (sketched_system.hpp:25-31,69-84) from a host
 * m x d sketch (ld = lds). */
ihs_status ihs_gpu_system_factorize(const double* SA, int64_t m, int64_t d, int64_t lds, double nu,
                                    int32_t device, ihs_counters* counters, ihs_gpu_system** out);
void ihs_gpu_system_destroy(ihs_gpu_system* s);
int32_t ihs_gpu_system_kind(const ihs_gpu_system* s);
int64_t ihs_gpu_system_m(const ihs_gpu_system* s);
int64_t ihs_gpu_system_d(const ihs_gpu_system* s);
uint64_t ihs_gpu_system_factor_flops(const ihs_gpu_system* s);    /* :52-57 */
uint64_t ihs_gpu_system_flops_per_solve(const ihs_gpu_system* s); /* :61-66 */
/* SketchedSystem::solve (sketched_system.hpp:40-49): z = H_S^{-1} g */
ihs_status ihs_gpu_system_solve(const ihs_gpu_system* s, const double* g, double* z, ihs_counters* counters);
/* newton_decrement (sketched_system.hpp:95-101), host vectors */
ihs_status ihs_newton_decrement(const double* g, const double* gt, int64_t d, double* r);

/* ----------------------------------------------------------- solvers */
/* adaptive_solve (solver.hpp:242-250 -> adaptive_solve_core :106-232). The
 * whole loop runs against the device-resident problem; only the scalar
 * decrement r of each candidate crosses to the host for the accept/reject
 * decision, exactly as in the reference control flow. */
/* solve_underdetermined (dual.hpp:13-33): adaptive IHS on the dual ridge problem in A^T (gradient
 * A(A^T z) - b + nu^2 z, SRHT pads d); rep->x receives x = A^T z_T (d doubles), rep->dual_final z_T. */
/* prediction_error (problem.hpp:104-109): 1/2 ||A(x - x*)||^2 + nu^2/2 ||x - x*||^2; x, x_star: d doubles */
ihs_status ihs_gpu_prediction_error(ihs_gpu_problem* p, const double* x, const double* x_star, double* out);
ihs_status ihs_gpu_solve_underdetermined(ihs_gpu_problem* p, const ihs_solver_config* cfg, ihs_solve_report* rep);
ihs_status ihs_gpu_adaptive_solve(ihs_gpu_problem* p, const ihs_solver_config* cfg, ihs_solve_report* rep);

/* fixed_sketch_ihs (solver.hpp:258-276): T steps with a fixed system. Writes
 * (T+1) iterates, x_start first, to iterates_out (d*(T+1) doubles). */
ihs_status ihs_gpu_fixed_sketch_ihs(ihs_gpu_problem* p, const ihs_gpu_system* s, const ihs_tuning* tp,
                                    int64_t T, int32_t mode, const double* x_start, double* iterates_out);

/* ------------------------------------------------ CG / PCG baselines */
/* pcg_sketch_size (baselines.hpp:170-187): m = d/rho (Gaussian) or d ln(d)/rho (SRHT, capped at n_pad). */
ihs_status ihs_pcg_sketch_size(int64_t n, int64_t d, int32_t kind, double rho, int64_t* m, int32_t* capped);
/* cg_solve (baselines.hpp:40-92): CG on (A^T A + nu^2 I) x = A^T b, stops when
 * ||H x - A^T b|| <= tol ||A^T b||; x0 (d doubles) may be NULL (zero start). */
ihs_status ihs_gpu_cg_solve(ihs_gpu_problem* p, double tol, int64_t max_iters, const double* x0, ihs_cg_report* rep);
/* pcg_solve_with (baselines.hpp:98-165): CG preconditioned by the Cholesky factor of
 * SA^T SA + nu^2 I_d, SA a host m x d column-major sketch (leading dimension lds). */
ihs_status ihs_gpu_pcg_solve_with(ihs_gpu_problem* p, const double* SA, int64_t m, int64_t lds, double tol,
                                  int64_t max_iters, const double* x0, ihs_cg_report* rep);
/* pcg_solve (baselines.hpp:190-200): sketch of the prescribed size on the device, then pcg_solve_with. */
ihs_status ihs_gpu_pcg_solve(ihs_gpu_problem* p, int32_t kind, uint64_t seed, double rho, double tol,
                             int64_t max_iters, const double* x0, ihs_cg_report* rep);

/* ---------------------------------------------------- synthetic data
 * SURVEY.md §8(d) generator shared by bench and tests: A = G diag(sigma),
 * G block-streamed from make_stream(data_seed, 1000 + j*nb + q), x_true from
 * tag 12, noise from tag 13, optional outliers from tag 14. Host, threaded. */
typedef struct ihs_synth_spec {
    int64_t n, d;
    int32_t spectrum;       /* 0: sigma_j = decay^j, 1: sigma_j = 1/j (j = 1..d) */
    int32_t _pad;
    double decay;
    double noise_std;
    double outlier_frac;    /* 0 or e.g. 0.01 */
    double outlier_scale;   /* e.g. 100 */
    uint64_t data_seed;
    int32_t threads;        /* 0 = hardware concurrency */
    int32_t _pad2;
} ihs_synth_spec;
/* Fills rows [row0, row0+rows) of A (column-major, ld = lda) and b; x_true
 * (d doubles) optional. */
ihs_status ihs_synth_generate(const ihs_synth_spec* spec, int64_t row0, int64_t rows, double* A, int64_t lda,
                              double* b, double* x_true);

#ifdef __cplusplus
}
#endif
#endif /* IHS_GPU_H */
