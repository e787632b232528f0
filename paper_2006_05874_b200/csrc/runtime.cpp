// runtime.cpp — the C-ABI of include/ihs_gpu.h: problem handles, sketches,
// the sketched system and the adaptive Polyak-IHS loop on the device.
//
// Control flow mirrors the reference line by line (solver.hpp:106-232); every
// vector of the loop (x_t, x_{t-1}, g_t, g~_t and both candidates) stays in
// HBM and only the decrement scalars of each evaluation cross to the host
// for the accept/reject decision. Counters are the reference's closed forms
// and are charged only for the evaluations the reference performs.
#include "common.cuh"
#include "host_rng.h"
#include "mt_jump.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace ihs_b200 {

void synth_generate(const ihs_synth_spec& s, int64_t row0, int64_t rows, double* A, int64_t lda, double* b,
                    double* x_true);

namespace {
std::atomic<int64_t> g_launches{0};
thread_local std::string g_last_error;

template <class F>
ihs_status guarded(F&& f) {
    try {
        f();
        return IHS_OK;
    } catch (const Status& s) {
        g_last_error = s.what();
        return s.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return IHS_INTERNAL_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return IHS_INTERNAL_ERROR;
    }
}

// ------------------------------------------------------------ device buffers
// Device buffers come from the device's stream-ordered memory pool (kept
// resident: release threshold = max), so the per-doubling growth of the
// sketch/factor buffers neither synchronizes the device nor takes the
// driver's allocation path after warm-up.
std::atomic<int64_t> g_alloc_ns{0};
std::atomic<int64_t> g_host_rng_ns{0};
void configure_pool(int dev) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return;
    cudaMemPool_t pool;
    CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done.push_back(dev);
}

// Allocations are ordered on the stream of the API call in flight (set by a
// StreamScope at the top of every entry point that allocates).
thread_local cudaStream_t g_cur_stream = nullptr;
struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(g_cur_stream) { g_cur_stream = s; }
    ~StreamScope() { g_cur_stream = prev; }
};
// Owns a stream; declared as the first member of a handle so it is destroyed
// after every buffer that frees itself on that stream.
struct StreamOwner {
    cudaStream_t s = nullptr;
    ~StreamOwner() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;  // stream the buffer was allocated on (its free is ordered there)
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        const auto t0 = std::chrono::steady_clock::now();
        release();
        st = g_cur_stream;
        if (b == 0) return;
        cudaError_t e = cudaMallocAsync(&p, b, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            fail(IHS_CUDA_ERROR, "cudaMallocAsync(" + std::to_string(b) + " bytes): " + cudaGetErrorString(e));
        }
        bytes = b;
        g_alloc_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
    double* d() const { return static_cast<double*>(p); }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinnedBuf() { if (p) cudaFreeHost(p); }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        CUDA_CHECK(cudaMallocHost(&p, b));
        bytes = b;
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CUDA_CHECK(cudaGetDevice(&prev));
        if (prev != dev) CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

int sm_count(int dev) {
    int v = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
}

void check_finite_host(const double* v, int64_t count, const char* msg) {
    for (int64_t i = 0; i < count; ++i)
        if (!std::isfinite(v[i])) fail(IHS_INVALID_INPUT, msg);
}

// ------------------------------------------------------------ phase timer
struct PhaseTimer {
    cudaStream_t st;
    std::vector<std::pair<cudaEvent_t, int>> marks;  // (event, phase id) — phase id -1 = end
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    bool enabled = true;
    bool active = false;  // between reset() (solve start) and collect()
    explicit PhaseTimer(cudaStream_t s) : st(s) {}
    ~PhaseTimer() {
        for (auto e : pool) cudaEventDestroy(e);
    }
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            CUDA_CHECK(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    void mark(int phase) {
        if (!enabled || !active) return;
        cudaEvent_t e = get();
        CUDA_CHECK(cudaEventRecord(e, st));
        marks.push_back({e, phase});
    }
    void reset() {
        marks.clear();
        used = 0;
        active = true;
    }
    // sum of intervals [mark(phase), next mark) per phase id (0..4), and the
    // number of intervals per phase
    void collect(double out_ms[6], int64_t count[6]) {
        active = false;
        for (int i = 0; i < 6; ++i) out_ms[i] = 0.0, count[i] = 0;
        if (marks.size() < 2) return;
        CUDA_CHECK(cudaEventSynchronize(marks.back().first));
        for (size_t i = 0; i + 1 < marks.size(); ++i) {
            const int ph = marks[i].second;
            if (ph < 0 || ph > 5) continue;
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, marks[i].first, marks[i + 1].first));
            out_ms[ph] += ms;
            count[ph] += 1;
        }
    }
};
// cap on the SRHT phase-1 scratch (larger sketches run over column batches); IHS_SRHT_SCRATCH_CAP_MB
// overrides it (tests exercise the batched path on small problems)
const int64_t kSrhtScratchCap = [] {
    const char* e = std::getenv("IHS_SRHT_SCRATCH_CAP_MB");
    const long long mb = e ? std::atoll(e) : 0;
    return mb > 0 ? (int64_t)mb << 20 : (int64_t)16 << 30;
}();

// PH_SKETCH_KERNEL: the sketch's main kernels inside a PH_SKETCH interval
// PH_GRAD_KERNEL: the gradient kernels (grad pass + fixed-order reduce) inside a PH_GRAD interval
enum { PH_SKETCH = 0, PH_FACTOR = 1, PH_GRAD = 2, PH_SOLVE = 3, PH_SKETCH_KERNEL = 4, PH_GRAD_KERNEL = 5, PH_END = -1 };

}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace ihs_b200

using namespace ihs_b200;

// ============================================================ opaque handles
struct ihs_gpu_system {
    StreamOwner owner;  // first member: destroyed after the buffers below
    int device = 0;
    int64_t m = 0, d = 0;
    double nu = 0.0;
    int kind = IHS_FACTOR_DIRECT_GRAM;
    bool force_gram = false;  // PCG preconditioner: the d x d Gram form whatever m (baselines.hpp:111-114)
    const double* SA_view = nullptr;  // factor a matrix owned elsewhere (direct_solve: the problem's A, ld lds_view)
    int64_t lds_view = 0;
    void* gram_comm = nullptr;        // row-sharded A: all-reduce the Gram partials before the factorization
    // adaptive loop: the factorization's status is read back with the next host synchronization the
    // loop makes anyway (system_check) instead of a dedicated round trip per factorization
    bool defer_info = false;
    bool info_pending = false;
    PinnedBuf h_info;
    cudaStream_t st = nullptr;
    int num_sms = 148;
    DevBuf SA;    // m x d
    DevBuf L;     // k x k Cholesky factor (k = m or d), lower
    DevBuf W;     // L^{-1} (lower) with L^{-T} mirrored into the strict upper triangle
    DevBuf Xd;    // inverses of L's 64x64 diagonal blocks (from the factorization)
    DevBuf Hinv;  // direct-Gram path: H_S^{-1} = L^{-T} L^{-1} (k x k), one mat-vec per solve
    DevBuf gv;    // gemv_tiled partials + arrival counters
    DevBuf inv_tmp;
    DevBuf work;  // split-K workspace
    DevBuf tmp;   // solve scratch
    DevBuf info;
    int64_t k() const { return kind == IHS_FACTOR_WOODBURY_INNER ? m : d; }
    uint64_t factor_flops() const {  // sketched_system.hpp:52-57
        const uint64_t mm = (uint64_t)m, dd = (uint64_t)d;
        if (kind == IHS_FACTOR_WOODBURY_INNER) return mm * mm * dd + mm * mm * mm / 3;
        return dd * dd * mm + dd * dd * dd / 3;
    }
    uint64_t flops_per_solve() const {  // sketched_system.hpp:61-66
        const uint64_t mm = (uint64_t)m, dd = (uint64_t)d;
        if (kind == IHS_FACTOR_WOODBURY_INNER) return 2 * mm * dd + mm * mm + 2 * dd;
        return dd * dd + dd;
    }
};

struct ihs_gpu_problem {
    StreamOwner owner;  // first member: destroyed after the buffers below
    int device = 0;
    int64_t n = 0, d = 0;
    double nu = 0.0;
    int orientation = IHS_OVERDETERMINED;
    ihs_gpu_options opts{};
    cudaStream_t st = nullptr;
    int num_sms = 148;
    int64_t lda = 0;             // device leading dimension: n rounded up to 32 (256 B columns)
    DevBuf A, b;                 // A (lda x d, column-major), b (lda); padding rows are zero
    DevBuf Arm;                  // row-major copy of A for the gradient (lda x d), when it fits
    GradPlan gplan{};
    DevBuf grad_work;
    // sketch workspaces
    DevBuf T, signbits, rng_scratch, entries, tiles, gauss_scratch, S, gemm_work;
    DevBuf shard_U, shard_hi;    // sharded SRHT partials [P][m][d] and r_hi(k)
    DevBuf fused_ctl;            // work-queue counters of the fused SRHT kernel
    DevBuf srht_mask;            // phase-1 store mask (active low-index groups)
    uint32_t h_mask[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool mask_valid = false;
    PinnedBuf h_stage;
    std::vector<int64_t> h_rows;
    std::vector<int2> h_entries;
    std::vector<int4> h_tiles;
    // solver vectors
    DevBuf vecs;                 // 28 * d doubles (start state + four candidate-evaluation sets)
    DevBuf dots;                 // 24 doubles (4 per evaluation set + first/resketch decrements)
    PinnedBuf h_dots;
    cudaEvent_t set_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // evaluation-set completion events
    cudaEvent_t set_ready[4] = {nullptr, nullptr, nullptr, nullptr};  // evaluation results ready on st
    // side stream for the decision read-backs: the main stream then runs the evaluation kernels back
    // to back, so each may launch programmatically while its predecessor drains
    cudaStream_t st2 = nullptr;
    StreamOwner owner2;
    // asynchronous re-upload (ihs_gpu_problem_upload_async): A, b and the row-major copy are written on st2;
    // the first kernel that reads them waits for a_ready (ensure_A), so A-independent work — the Gaussian
    // sketch's RNG, the SRHT's signs and row sample — overlaps the host-to-device copy
    cudaEvent_t a_ready = nullptr;
    bool a_pending = false;
    // underdetermined instances (dual.hpp): the dual problem in A^T, built on first use, and on the dual
    // problem itself the observation vector subtracted from every gradient (non-owning, n doubles)
    std::unique_ptr<ihs_gpu_problem> dual;
    const double* gsub = nullptr;
    // CG / PCG baselines: zero observation vector (H v = gradient pass with b = 0), the recurrence
    // vectors + device state, and its pinned read-back
    DevBuf zb, cgv;
    PinnedBuf h_cg;
    bool zb_ready = false;
    ~ihs_gpu_problem() {
        for (auto e : set_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : set_ready)
            if (e) cudaEventDestroy(e);
        if (a_ready) cudaEventDestroy(a_ready);
    }
    std::unique_ptr<PhaseTimer> timer;
};

namespace ihs_b200 {
namespace {

// -------------------------------------------------------- sketches (device)
// T scratch and the fused kernel's control block; nullptr control = the
// two-kernel path (default: measured faster; IHS_SRHT_FUSED=1 selects the
// persistent single-launch kernel for A/B measurements).
unsigned long long* srht_prepare_scratch(ihs_gpu_problem* P, const SrhtPlan& plan) {
    if (plan.l2) {  // L2-resident single launch: a ring of column slots + the work/completion counters
        P->T.ensure(srht_l2_scratch_bytes(plan));
        P->fused_ctl.ensure(srht_l2_ctl_bytes(plan));
        return P->fused_ctl.as<unsigned long long>();
    }
    if (!plan.stream) {  // two-kernel path (srht_plan_stream declined)
        P->T.ensure(srht_scratch_bytes(plan));
        return nullptr;
    }
    size_t ctl_bytes = 0;
    P->T.ensure(srht_fused_scratch_bytes(plan, &ctl_bytes, P->num_sms));
    P->fused_ctl.ensure(ctl_bytes);
    return P->fused_ctl.as<unsigned long long>();
}

// Upload host-built SRHT entries/tiles through the pinned staging buffer.
void upload_entries(ihs_gpu_problem* P) {
    cudaStream_t st = P->st;
    const size_t eb = P->h_entries.size() * sizeof(int2), tb = P->h_tiles.size() * sizeof(int4);
    P->h_stage.ensure(eb + tb + 64);
    // the previous sketch's copy out of the staging buffer must be done
    CUDA_CHECK(cudaStreamSynchronize(st));
    std::memcpy(P->h_stage.p, P->h_entries.data(), eb);
    std::memcpy(static_cast<char*>(P->h_stage.p) + eb, P->h_tiles.data(), tb);
    std::memcpy(static_cast<char*>(P->h_stage.p) + eb + tb, P->h_mask, sizeof(P->h_mask));
    P->entries.ensure(eb + 16);
    P->tiles.ensure(tb + 16);
    P->srht_mask.ensure(sizeof(P->h_mask));
    CUDA_CHECK(cudaMemcpyAsync(P->entries.p, P->h_stage.p, eb, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(P->tiles.p, static_cast<char*>(P->h_stage.p) + eb, tb, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(P->srht_mask.p, static_cast<char*>(P->h_stage.p) + eb + tb, sizeof(P->h_mask),
                               cudaMemcpyHostToDevice, st));
}

// SA (m x d, ld m, device) = apply_sketch(A, {kind, m, seed}) (sketch.hpp:110-117).
// Row-sharded problems (world_size > 1) compute their shard's part and
// exchange it over NCCL; `emulate_shards` > 1 runs the same sharded SRHT
// decomposition on one device (shards back to back), which the tests use to
// prove the decomposition bit-exact.
void ensure_A(ihs_gpu_problem* P);
void device_sketch(ihs_gpu_problem* P, int kind, int64_t m, uint64_t seed, double* d_SA, ihs_counters* c,
                   int emulate_shards = 1) {
    const int64_t n = P->n, d = P->d;
    const int world = P->opts.world_size;
    const int64_t n_glob = world > 1 ? P->opts.n_global : n;
    cudaStream_t st = P->st;
    if (kind == IHS_SKETCH_SRHT) {
        if (m < 1) fail(IHS_INVALID_INPUT, "srht_sketch: m must be >= 1");
        SrhtPlan plan = srht_plan(n_glob, d, P->lda, m);
        if (m > plan.n_pad) fail(IHS_SKETCH_TOO_LARGE, "srht_sketch: m exceeds padded row count");
        // D: rademacher(n_pad, make_stream(seed, 1)) as bits (sketch.hpp:85,87)
        P->signbits.ensure((size_t)((plan.n_pad + 31) / 32) * 4);
        P->rng_scratch.ensure(rademacher_scratch_bytes(plan.n_pad));
        mt_rademacher_bits(derive_seed(seed, 1), plan.n_pad, P->signbits.as<uint32_t>(), P->rng_scratch.p, st);
        // P: sample_without_replacement(n_pad, m, make_stream(seed, 2)) (sketch.hpp:86,88)
        P->h_rows.resize((size_t)m);
        const auto t_rng = std::chrono::steady_clock::now();
        sample_without_replacement(derive_seed(seed, 2), plan.n_pad, m, P->h_rows.data());
        const int shards = world > 1 ? world : std::max(1, emulate_shards);
        if (shards == 1) {
            srht_plan_stream(plan, P->num_sms);  // decides the emitting-tile shape before the entries are built
            if (!srht_plan_compact(plan, P->h_rows.data())) srht_plan_l2(plan);
            srht_build_entries(plan, P->h_rows.data(), P->h_entries, P->h_tiles);
            P->mask_valid = srht_build_mask(plan, P->h_tiles, P->h_mask);
            g_host_rng_ns +=
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_rng).count();
            upload_entries(P);
            // columns are independent: when the phase-1 scratch of all d columns would exceed the cap,
            // the transform runs over column batches that share one smaller scratch (and the row sample)
            const int64_t cols_per_batch =
                plan.l2 ? d  // the L2-resident launch needs only its slot ring, whatever d
                        : std::max<int64_t>(1, std::min<int64_t>(d, kSrhtScratchCap / (plan.n_pad * (int64_t)sizeof(double))));
            ensure_A(P);  // the signs and the row sample above did not need A
            SrhtPlan bp = plan;
            bp.d = std::min<int64_t>(d, cols_per_batch);
            // compact plans carry the low-index map (128 int4) after their tiles
            const int n_tiles = (int)P->h_tiles.size() - (plan.compact ? (int)(1024 * sizeof(short) / sizeof(int4)) : 0) -
                                (plan.l2 ? 4 : 0);
            unsigned long long* ctl = srht_prepare_scratch(P, bp);
            if (P->timer) P->timer->mark(PH_SKETCH_KERNEL);
            for (int64_t j0 = 0; j0 < d; j0 += cols_per_batch) {
                bp.d = std::min<int64_t>(cols_per_batch, d - j0);
                srht_run_device(bp, P->A.d() + j0 * P->lda, P->signbits.as<uint32_t>(), P->entries.as<int2>(),
                                P->tiles.as<int4>(), n_tiles, P->T.d(), d_SA + j0 * m, st, ctl,
                                P->num_sms, P->mask_valid ? P->srht_mask.as<uint32_t>() : nullptr);
            }
            if (P->timer) P->timer->mark(PH_SKETCH);
        } else {
            // shard p holds rows [p*n_loc, (p+1)*n_loc) of the padded index space
            const int64_t n_loc = plan.n_pad / shards;
            std::vector<int64_t> lo((size_t)m);
            std::vector<uint8_t> hi((size_t)m);
            for (int64_t k = 0; k < m; ++k) {
                lo[(size_t)k] = P->h_rows[(size_t)k] % n_loc;
                hi[(size_t)k] = (uint8_t)(P->h_rows[(size_t)k] / n_loc);
            }
            SrhtPlan sp = srht_plan_shard(std::min(n_loc, n), n_loc, d, P->lda, m);
            srht_plan_stream(sp, P->num_sms);
            srht_build_entries(sp, lo.data(), P->h_entries, P->h_tiles);
            P->mask_valid = srht_build_mask(sp, P->h_tiles, P->h_mask);
            g_host_rng_ns +=
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_rng).count();
            if (world <= 1) upload_entries(P);  // (the sharded exchange remaps the entries first)
            // r_hi(k), zero-padded to whole owner blocks
            const int64_t mq_pad = ceil_div(m, shards) * shards;
            hi.resize((size_t)mq_pad, 0);
            P->shard_hi.ensure((size_t)mq_pad + 16);
            CUDA_CHECK(cudaMemcpyAsync(P->shard_hi.p, hi.data(), (size_t)mq_pad, cudaMemcpyHostToDevice, st));
            ensure_A(P);
            // emulated shards: [P][m][d] partials; a rank of a sharded problem: send/recv owner blocks, its own
            // combined block and the gathered blocks ((2 P + 1 + P) mq d doubles)
            const int64_t mq = ceil_div(m, shards);
            P->shard_U.ensure(world > 1 ? (size_t)(3 * shards + 1) * mq * d * sizeof(double)
                                        : (size_t)shards * m * d * sizeof(double));
            unsigned long long* ctl = srht_prepare_scratch(P, sp);
            double* U = P->shard_U.d();
            auto run_shard = [&](int p, const double* A_p, int64_t n_real) {
                SrhtPlan s = sp;
                s.n = n_real;
                srht_run_device(s, A_p, P->signbits.as<uint32_t>() + (p * n_loc) / 32, P->entries.as<int2>(),
                                P->tiles.as<int4>(), (int)P->h_tiles.size(), P->T.d(), U + (int64_t)p * m * d, st,
                                ctl, P->num_sms, P->mask_valid ? P->srht_mask.as<uint32_t>() : nullptr);
            };
            if (world > 1) {
                // owner-reduce exchange (per rank ~2 m d doubles received instead of the P m d of an all-gather of
                // the partials): rank q owns sampled rows [q mq, (q+1) mq). The shard's emitting pass writes its
                // partials straight into owner blocks (entries remapped to q mq d + kk, column stride mq); an
                // all-to-all hands every owner the P partials of its rows, the owner combines them in the
                // reference's butterfly order (bit-exact), and an all-gather + unpack assemble SA on every rank.
                const int r = P->opts.rank;
                const int64_t mq = ceil_div(m, world);
                for (int2& e : P->h_entries) {
                    const int64_t k = e.y, q = k / mq;
                    e.y = (int)(q * mq * d + (k - q * mq));
                }
                upload_entries(P);
                double* send = U;                                  // [q][mq x d] partial blocks
                double* recv = U + (int64_t)world * mq * d;        // [p][mq x d] partials of my rows
                double* own = recv + (int64_t)world * mq * d;      // my combined rows (mq x d)
                double* gathered = own + mq * d;                   // [q][mq x d] combined blocks
                SrhtPlan s = sp;
                s.n = n;
                s.sa_ld = mq;
                srht_run_device(s, P->A.d(), P->signbits.as<uint32_t>() + (r * n_loc) / 32, P->entries.as<int2>(),
                                P->tiles.as<int4>(), (int)P->h_tiles.size(), P->T.d(), send, st, ctl, P->num_sms,
                                P->mask_valid ? P->srht_mask.as<uint32_t>() : nullptr);
                nccl_alltoall(send, recv, (size_t)(mq * d), P->opts.nccl_comm, st);
                srht_combine(recv, world, mq, d, P->shard_hi.as<uint8_t>() + (int64_t)r * mq, plan.scale1, plan.scale2,
                             own, st);
                nccl_allgather(own, gathered, (size_t)(mq * d), P->opts.nccl_comm, st);
                srht_unpack_blocks(gathered, world, mq, m, d, d_SA, st);
            } else {
                for (int p = 0; p < shards; ++p) {
                    const int64_t n_real = std::max<int64_t>(0, std::min<int64_t>(n_loc, n - p * n_loc));
                    run_shard(p, P->A.d() + p * n_loc, n_real);
                }
                srht_combine(U, shards, m, d, P->shard_hi.as<uint8_t>(), plan.scale1, plan.scale2, d_SA, st);
            }
        }
        if (c) {  // sketch.hpp:99-106
            const uint64_t np = (uint64_t)plan.n_pad, dd = (uint64_t)d;
            c->sketch += dd * np * (uint64_t)plan.logn + (uint64_t)n_glob * dd + (uint64_t)m * dd;
        }
    } else if (kind == IHS_SKETCH_GAUSSIAN) {
        if (m < 1) fail(IHS_INVALID_INPUT, "gaussian_sketch: m must be >= 1");
        // S (m x n) ~ N(0, 1/m) from make_stream(seed, 0), column-major (sketch.hpp:62-64);
        // a shard holds the columns of its rows, i.e. normals [row0*m, (row0+n)*m)
        const int64_t count = m * n;
        const int64_t first = world > 1 ? P->opts.row_offset * m : 0;
        const double stddev = 1.0 / std::sqrt(static_cast<double>(m));
        // materialise S when it and the generator's scratch fit comfortably; otherwise stream it in column
        // blocks into an accumulating GEMM (IHS_GAUSS_STREAM=1 forces, IHS_GAUSS_STREAM_COLS sets the block)
        static const int force_stream = [] {
            const char* e = std::getenv("IHS_GAUSS_STREAM");
            return e ? std::atoi(e) : -1;
        }();
        const size_t s_bytes = (size_t)count * sizeof(double), g_bytes = gaussian_scratch_bytes(first + count);
        bool stream = force_stream == 1;
        if (force_stream != 1 && force_stream != 0 && (P->S.bytes < s_bytes || P->gauss_scratch.bytes < g_bytes)) {
            // the buffers would grow: materialise only while that leaves room (the query is skipped when they fit)
            size_t free_b = 0, total_b = 0;
            CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
            stream = s_bytes + g_bytes + (8ull << 30) > free_b + P->S.bytes + P->gauss_scratch.bytes;
        }
        if (!stream) {
            P->S.ensure((size_t)count * sizeof(double));
            P->gauss_scratch.ensure(gaussian_scratch_bytes(first + count));
            mt_fill_gaussian(derive_seed(seed, 0), first, count, stddev, P->S.d(), P->gauss_scratch.p, st);
            // SA = S * A on the DMMA path (sketch.hpp:68)
            const int splitk = dgemm_pick_splitk(m, d, n, P->num_sms);
            if (splitk > 1) P->gemm_work.ensure((size_t)splitk * m * d * sizeof(double));
            ensure_A(P);  // S was generated without A
            if (P->timer) P->timer->mark(PH_SKETCH_KERNEL);
            dgemm(false, false, m, d, n, 1.0, P->S.d(), m, P->A.d(), P->lda, 0.0, d_SA, m, false, splitk,
                  splitk > 1 ? P->gemm_work.d() : nullptr, st);
            if (P->timer) P->timer->mark(PH_SKETCH);
        } else {
            static const int64_t env_cols = [] {
                const char* e = std::getenv("IHS_GAUSS_STREAM_COLS");
                return e ? (int64_t)std::atoll(e) : (int64_t)0;
            }();
            // column blocks of ~1 GiB of S (>= 2 columns), the buffer also holds one chunk's normals
            const int64_t cols = std::max<int64_t>(2, env_cols > 0 ? env_cols : (int64_t)(128ll << 20) / m);
            const int64_t block = cols * m;
            const int64_t cap = block + 2 * gaussian_stream_chunk_attempts() + 2 * m + 16;
            P->S.ensure((size_t)cap * sizeof(double));
            P->gauss_scratch.ensure(gaussian_stream_scratch_bytes());
            ensure_A(P);
            int64_t col_done = 0;
            auto consume = [&](int64_t base, int64_t ready) -> int64_t {
                int64_t ncols = std::min<int64_t>(ready / m, n - col_done);
                // an even column count keeps the next block's A operand (A + col_done) 16-byte aligned
                if (col_done + ncols < n) ncols &= ~int64_t{1};
                if (ncols <= 0) return 0;
                const int splitk = dgemm_pick_splitk(m, d, ncols, P->num_sms);
                if (splitk > 1) P->gemm_work.ensure((size_t)splitk * m * d * sizeof(double));
                if (P->timer) P->timer->mark(PH_SKETCH_KERNEL);
                dgemm(false, false, m, d, ncols, 1.0, P->S.d(), m, P->A.d() + col_done, P->lda, col_done ? 1.0 : 0.0,
                      d_SA, m, false, splitk, splitk > 1 ? P->gemm_work.d() : nullptr, st);
                if (P->timer) P->timer->mark(PH_SKETCH);
                col_done += ncols;
                return ncols * m;
            };
            mt_gaussian_stream(derive_seed(seed, 0), first, count, stddev, P->S.d(), cap, block, P->gauss_scratch.p,
                               st, consume);
            if (col_done != n) fail(IHS_INTERNAL_ERROR, "gaussian stream: incomplete sketch");
        }
        if (world > 1) nccl_allreduce_sum(d_SA, (size_t)(m * d), P->opts.nccl_comm, st);
        if (c) c->sketch += (uint64_t)m * (uint64_t)n_glob * (uint64_t)d;  // sketch.hpp:65-67
    } else {
        fail(IHS_INVALID_INPUT, "apply_sketch: unknown sketch kind");
    }
}

// ---------------------------------------------------- sketched system (device)
// SketchedSystem::factorize (sketched_system.hpp:25-31, 69-84) of a device SA
// already stored in sys->SA.
// Raise the status of the last factorization (sketched_system.hpp:82-83); the stream must have
// passed the factorization's status copy (a synchronization after it).
void system_check(ihs_gpu_system* S) {
    if (!S->info_pending) return;
    S->info_pending = false;
    const int* h = static_cast<const int*>(S->h_info.p);
    if (h[1]) fail(IHS_INVALID_INPUT, "SketchedSystem: non-finite sketched matrix");
    if (h[0]) fail(IHS_NUMERICAL_BREAKDOWN, "SketchedSystem: Cholesky factorization failed");
}

void system_factorize(ihs_gpu_system* S, ihs_counters* c) {
    const int64_t m = S->m, d = S->d;
    cudaStream_t st = S->st;
    if (!(S->nu > 0.0)) fail(IHS_INVALID_INPUT, "SketchedSystem: nu must be positive");
    const double* SA = S->SA_view ? S->SA_view : S->SA.d();
    const int64_t lds = S->SA_view ? S->lds_view : m;
    S->info.ensure(2 * sizeof(int));
    int* d_flag = S->info.as<int>() + 1;
    CUDA_CHECK(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
    if (m * d > 0 && !S->SA_view) check_finite(SA, m * d, d_flag, st);
    S->kind = m < d && !S->force_gram ? IHS_FACTOR_WOODBURY_INNER : IHS_FACTOR_DIRECT_GRAM;
    const int64_t k = S->k();
    S->L.ensure((size_t)k * k * sizeof(double));
    const double nu2 = S->nu * S->nu;
    if (S->kind == IHS_FACTOR_WOODBURY_INNER) {
        // inner = SA SA^T + nu^2 I_m (lower)
        const int splitk = dgemm_pick_splitk(m, m, d, S->num_sms, false, true, true);
        if (splitk > 1) S->work.ensure((size_t)splitk * m * m * sizeof(double));
        dgemm(false, true, m, m, d, 1.0, SA, lds, SA, lds, 0.0, S->L.d(), m, true, splitk,
              splitk > 1 ? S->work.d() : nullptr, st);
    } else {
        // gram = SA^T SA + nu^2 I_d (lower)
        const int splitk = dgemm_pick_splitk(d, d, m, S->num_sms, true, false, true);
        if (splitk > 1) S->work.ensure((size_t)splitk * d * d * sizeof(double));
        dgemm(true, false, d, d, m, 1.0, SA, lds, SA, lds, 0.0, S->L.d(), d, true, splitk,
              splitk > 1 ? S->work.d() : nullptr, st);
        if (S->gram_comm) nccl_allreduce_sum(S->L.d(), (size_t)d * d, S->gram_comm, st);
    }
    add_diag(S->L.d(), k, nu2, st);
    // IHS_CHOL_MODE: 2 (default) one cooperative launch; 1 per-panel kernels with fused diagonal
    // factor+inverse; 0 per-panel column-serial kernels
    static const int chol_mode = [] {
        const char* e = std::getenv("IHS_CHOL_MODE");
        return e ? std::atoi(e) : 0;
    }();
    double* Xd = nullptr;
    int xd_block = 64;
    if (chol_mode >= 1) {
        S->Xd.ensure(cholesky_diag_inv_doubles(k) * sizeof(double));
        Xd = S->Xd.d();
    }
    if (chol_mode == 2 && cholesky_factor_coop(S->L.d(), k, Xd, S->info.as<int>(), S->num_sms, st)) {
        xd_block = 32;
    } else {
        cholesky_factor(S->L.d(), k, chol_mode == 1 ? Xd : nullptr, S->info.as<int>(), S->num_sms, st);
        if (chol_mode != 1) Xd = nullptr;
    }
    // W = L^{-1} once per factorization; every later solve is two mat-vecs
    const int64_t hk = (k + 1) / 2 + 64;
    S->W.ensure((size_t)k * k * sizeof(double));
    S->inv_tmp.ensure((size_t)hk * hk * sizeof(double));
    cholesky_invert(S->L.d(), k, S->W.d(), S->inv_tmp.d(), Xd, st, xd_block);
    if (S->kind == IHS_FACTOR_DIRECT_GRAM) {
        // H_S^{-1} = (L^{-1})^T L^{-1} explicitly (DMMA, k^3 flop once per factorization): every solve
        // is then a single symmetric mat-vec instead of two dependent triangular ones
        S->Hinv.ensure((size_t)k * k * sizeof(double));
        tril_copy(S->W.d(), k, S->L.d(), st);  // the factor itself is not needed after the inverse
        const int splitk = dgemm_pick_splitk(k, k, k, S->num_sms, true, false, false);
        if (splitk > 1) S->work.ensure((size_t)splitk * k * k * sizeof(double));
        dgemm(true, false, k, k, k, 1.0, S->L.d(), k, S->L.d(), k, 0.0, S->Hinv.d(), k, false, splitk,
              splitk > 1 ? S->work.d() : nullptr, st);
    }
    const int64_t gm = S->kind == IHS_FACTOR_DIRECT_GRAM ? d : m;
    S->gv.ensure((gemv_tiled_work_doubles(gm, d) + 8) * sizeof(double));
    gemv_tiled_reset(S->gv.d(), gm, d, st);
    S->h_info.ensure(2 * sizeof(int));
    CUDA_CHECK(cudaMemcpyAsync(S->h_info.p, S->info.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    S->info_pending = true;
    if (!S->defer_info) {
        CUDA_CHECK(cudaStreamSynchronize(st));
        system_check(S);
    }
    S->tmp.ensure((size_t)(4 * std::max(m, d) + cholesky_solve_work_doubles(k)) * sizeof(double));
    if (c) c->factor += S->factor_flops();
}

// z = H_S^{-1} g and the decrement dots (g.z, g.g per RHS) into dots; fused into the
// mat-vec's last block on the direct-Gram path
void system_solve_dev(const ihs_gpu_system* S, const double* g, double* z, int nrhs);
void system_solve_dots(const ihs_gpu_system* S, const double* g, double* z, int nrhs, double* dots) {
    if (S->kind == IHS_FACTOR_DIRECT_GRAM) {
        symv_col(S->Hinv.d(), S->d, g, nrhs, S->d, z, S->d, S->gv.d(), S->st, dots);
    } else {
        system_solve_dev(S, g, z, nrhs);
        decrement_dots(g, z, S->d, nrhs, dots, S->st);
    }
}

// z[:, q] = H_S^{-1} g[:, q] (sketched_system.hpp:40-49), device vectors, ld = d
void system_solve_dev(const ihs_gpu_system* S, const double* g, double* z, int nrhs) {
    const int64_t m = S->m, d = S->d;
    cudaStream_t st = S->st;
    double* work = S->tmp.d() + 4 * std::max(m, d);
    if (S->kind == IHS_FACTOR_WOODBURY_INNER) {
        double* u = S->tmp.d();      // nrhs x m : u = SA g
        double* w = u + 2 * m;       // nrhs x m : w = (SA SA^T + nu^2 I)^{-1} u
        gemv_tiled(S->SA.d(), m, d, m, g, nrhs, d, u, m, S->gv.d(), st);
        cholesky_solve_inv(S->W.d(), m, u, w, nrhs, work, st);
        woodbury_finish(S->SA.d(), m, d, g, w, S->nu * S->nu, nrhs, z, st);
    } else {
        symv_col(S->Hinv.d(), d, g, nrhs, d, z, d, S->gv.d(), st);
    }
}

// Device copy of A with 32-row-aligned columns (zero padding rows) and b.
void upload_Ab(ihs_gpu_problem* P, const double* A, int64_t lda_host, const double* b, cudaStream_t st = nullptr) {
    if (!st) st = P->st;
    if (A)
        CUDA_CHECK(cudaMemcpy2DAsync(P->A.p, (size_t)P->lda * sizeof(double), A, (size_t)lda_host * sizeof(double),
                                     (size_t)P->n * sizeof(double), (size_t)P->d, cudaMemcpyHostToDevice, st));
    if (b) CUDA_CHECK(cudaMemcpyAsync(P->b.p, b, (size_t)P->n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (A && P->Arm.p) transpose_to_rowmajor(P->A.d(), P->lda, P->lda, P->d, P->Arm.d(), st);
}
// order the problem's stream after a pending asynchronous upload of A / b
void ensure_A(ihs_gpu_problem* P) {
    if (!P->a_pending) return;
    CUDA_CHECK(cudaStreamWaitEvent(P->st, P->a_ready, 0));
    P->a_pending = false;
}

void alloc_and_upload(ihs_gpu_problem* P, const double* A, int64_t lda_host, const double* b) {
    P->lda = ceil_div(P->n, 32) * 32;
    P->A.ensure((size_t)P->lda * P->d * sizeof(double));
    P->b.ensure((size_t)P->lda * sizeof(double));
    if (P->lda != P->n) CUDA_CHECK(cudaMemsetAsync(P->A.p, 0, (size_t)P->lda * P->d * sizeof(double), P->st));
    CUDA_CHECK(cudaMemsetAsync(P->b.p, 0, (size_t)P->lda * sizeof(double), P->st));
    upload_Ab(P, A, lda_host, b);
}

// g = A^T(Ax - b) + nu^2 x; on a row-sharded problem the A_p^T(A_p x - b_p)
// partials are summed over NCCL (identical bytes on every rank) before the
// nu^2 x term is added once.
void problem_grad(ihs_gpu_problem* P, const double* X, int nrhs, double* G, const CandSpec* cs = nullptr,
                  const double* bvec = nullptr) {
    ensure_A(P);
    const double nu2 = P->nu * P->nu;
    const double* b = bvec ? bvec : P->b.d();
    if (cs) X = cs->out;
    // inside a solve: the gradient kernels' own interval (bench roofline), then back to PH_GRAD
    if (P->timer) P->timer->mark(PH_GRAD_KERNEL);
    if (P->opts.world_size > 1) {
        grad_run(P->gplan, P->A.d(), b, 0.0, X, nrhs, G, P->grad_work.d(), P->st, P->Arm.d(), cs);
        if (P->timer) P->timer->mark(PH_GRAD);
        nccl_allreduce_sum(G, (size_t)nrhs * P->d, P->opts.nccl_comm, P->st);
        add_scaled(G, X, nu2, (int64_t)nrhs * P->d, P->st);
    } else {
        grad_run(P->gplan, P->A.d(), b, nu2, X, nrhs, G, P->grad_work.d(), P->st, P->Arm.d(), cs);
        if (P->timer) P->timer->mark(PH_GRAD);
    }
    // dual problem (dual.hpp:20-22): g = M^T(M z) + nu^2 z - b
    if (P->gsub)
        for (int q = 0; q < nrhs; ++q) add_scaled(G + (int64_t)q * P->d, P->gsub, -1.0, P->d, P->st);
}

// CG / sketch-preconditioned CG (baselines.hpp:40-92, 98-165) on the device-resident problem.
// S: the preconditioner (direct-Gram system with explicit H_S^{-1}: M^{-1} r is one mat-vec whose
// last CTA also forms r.z) or nullptr for plain CG. Iterations are enqueued in batches of B between
// read-backs of the device state (B ~ 256 MB of A traffic per batch, 1..16); a batch that passes the
// stopping point only runs no-op recurrence kernels after it (their H p passes are wasted work, not
// a change of result). Counters follow the reference's analytic formulas (baselines.hpp:51,117,120).
// Rows of the largest shard: the same on every rank of a sharded problem (n for a single GPU).
// Host-side plans that change the number of collectives a rank issues must be derived from this.
int64_t shard_rows_max(const ihs_gpu_problem* P) {
    if (P->opts.world_size <= 1) return P->n;
    return ihs_next_pow2(P->opts.n_global) / P->opts.world_size;
}

void cg_run(ihs_gpu_problem* P, const ihs_gpu_system* S, double tol, int64_t max_iters, const double* x0,
            ihs_cg_report* rep, ihs_counters& C) {
    const int64_t d = P->d, n = P->n;
    cudaStream_t st = P->st;
    const bool pcg = S != nullptr;
    const uint64_t nn = (uint64_t)(P->opts.world_size > 1 ? P->opts.n_global : n), dd = (uint64_t)d;
    const uint64_t hv_count = 2 * nn * dd + 2 * dd, minv_count = 2 * dd * dd;
    // B must agree on every rank (each H p pass all-reduces): size it from the largest shard's rows,
    // a rank-invariant value, not from this rank's own row count
    const double pass_bytes = 8.0 * (double)shard_rows_max(P) * (double)d;
    const int64_t B = std::max<int64_t>(1, std::min<int64_t>(16, (int64_t)(256e6 / std::max(pass_bytes, 1.0))));
    if (!P->zb_ready) {
        P->zb.ensure((size_t)P->lda * sizeof(double));
        CUDA_CHECK(cudaMemsetAsync(P->zb.p, 0, (size_t)P->lda * sizeof(double), st));
        P->zb_ready = true;
    }
    const size_t nvec = (size_t)7 * d + 8 + (size_t)(B + 1) + 8;
    P->cgv.ensure(nvec * sizeof(double) + cg_state_bytes());
    double* x = P->cgv.d();
    double *r = x + d, *p = r + d, *hp = p + d, *z = hp + d, *g0 = z + d, *hx = g0 + d, *dots = hx + d;
    double* resid = dots + 8;
    void* state = resid + B + 1 + 8;
    const size_t sb = cg_state_bytes();
    P->h_cg.ensure(sb + (size_t)(B + 1) * sizeof(double));
    void* h_state = P->h_cg.p;
    double* h_resid = reinterpret_cast<double*>(static_cast<char*>(P->h_cg.p) + sb);
    auto read_back = [&](int64_t from, int64_t count) {
        CUDA_CHECK(cudaMemcpyAsync(h_state, state, sb, cudaMemcpyDeviceToHost, st));
        if (count > 0)
            CUDA_CHECK(cudaMemcpyAsync(h_resid + from, resid + from, (size_t)count * sizeof(double),
                                       cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
    };
    PhaseTimer* tm = P->timer.get();
    auto mark = [&](int ph) {
        if (tm) tm->mark(ph);
    };
    int64_t passes = 1 + (x0 ? 1 : 0);
    // atb = -(A^T(A 0 - b) + nu^2 0); not counted (baselines.hpp:55 is outside apply_h)
    CUDA_CHECK(cudaMemsetAsync(z, 0, (size_t)d * sizeof(double), st));
    mark(PH_GRAD);
    problem_grad(P, z, 1, g0);
    if (x0) {
        CUDA_CHECK(cudaMemcpyAsync(x, x0, (size_t)d * sizeof(double), cudaMemcpyHostToDevice, st));
        problem_grad(P, x, 1, hx, nullptr, P->zb.d());  // H x0
    } else {
        CUDA_CHECK(cudaMemsetAsync(x, 0, (size_t)d * sizeof(double), st));
    }
    C.matvec += hv_count;  // the starting residual's H x (baselines.hpp:57 / :128)
    mark(PH_SOLVE);
    cg_begin(g0, x0 ? hx : nullptr, r, p, tol, d, state, resid, pcg, st);
    if (pcg) {
        symv_col(S->Hinv.d(), d, r, 1, d, z, d, S->gv.d(), st, dots);
        cg_dir(state, z, dots, p, d, true, st);
    }
    mark(PH_END);
    read_back(0, 1);
    std::vector<double> residuals{h_resid[0]};
    bool done = cg_state_done(h_state);
    if (!done && pcg) C.solve += minv_count;
    int64_t launched = 0;
    while (!done && launched < max_iters) {
        const int64_t nb = std::min(B, max_iters - launched);
        for (int64_t k = 0; k < nb; ++k) {
            mark(PH_GRAD);
            problem_grad(P, p, 1, hp, nullptr, P->zb.d());  // hp = A^T(A p) + nu^2 p
            mark(PH_SOLVE);
            cg_step(state, p, hp, x, r, resid, launched, d, pcg, st);
            if (pcg) {
                symv_col(S->Hinv.d(), d, r, 1, d, z, d, S->gv.d(), st, dots);
                cg_dir(state, z, dots, p, d, false, st);
            }
        }
        mark(PH_END);
        passes += nb;
        read_back(1, nb);
        const int64_t it = cg_state_iter(h_state);
        for (int64_t j = 1; j <= it - launched; ++j) residuals.push_back(h_resid[j]);
        done = cg_state_done(h_state);
        launched += nb;
    }
    const int64_t iters = (int64_t)residuals.size() - 1;
    rep->times.n_gradient += passes;
    rep->times.gradient_bytes += (double)passes * (8.0 * (double)n * (double)d + 8.0 * (double)n);
    C.matvec += (uint64_t)iters * hv_count;
    if (pcg && iters > 0) C.solve += (uint64_t)(done ? iters - 1 : iters) * minv_count;
    CUDA_CHECK(cudaMemcpyAsync(rep->x, x, (size_t)d * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    rep->iterations = iters;
    rep->converged = done;
    rep->residuals_size = (int64_t)residuals.size();
    if (rep->residuals)
        for (int64_t i = 0; i < rep->residuals_size && i < rep->residuals_capacity; ++i)
            rep->residuals[i] = residuals[(size_t)i];
}

// Ridge minimizer of Q (problem.hpp:73-82's direct_solve, reached on the device by the normal
// equations instead of the stacked QR): H = A^T A + nu^2 I from one DMMA Gram over the resident A
// (all-reduced over NCCL on a row-sharded problem), its Cholesky factor and explicit inverse, then
// x = H^{-1} (-grad(0)) and fixed-count iterative refinement x -= H^{-1} grad(x) with the fused
// gradient pass: each step shrinks the normal-equations error by ~cond(H) eps, so the result matches
// the QR solve to working accuracy on the conditioning the suite uses. x: device, d doubles.
void direct_solve_dev(ihs_gpu_problem* Q, double* x, int refinements = 3) {
    ensure_A(Q);
    const int64_t d = Q->d;
    cudaStream_t st = Q->st;
    ihs_gpu_system S;
    S.device = Q->device;
    S.d = d;
    S.m = Q->lda;
    S.nu = Q->nu;
    S.st = st;
    S.num_sms = Q->num_sms;
    S.force_gram = true;
    S.SA_view = Q->A.d();
    S.lds_view = Q->lda;
    S.gram_comm = Q->opts.world_size > 1 ? Q->opts.nccl_comm : nullptr;
    try {
        system_factorize(&S, nullptr);
    } catch (const Status& e) {
        if (e.code == IHS_NUMERICAL_BREAKDOWN) fail(IHS_NUMERICAL_BREAKDOWN, "direct_solve: factorization failed");
        throw;
    }
    DevBuf v;
    v.ensure((size_t)3 * d * sizeof(double));
    double *g = v.d(), *dx = g + d, *zero = dx + d;
    CUDA_CHECK(cudaMemsetAsync(zero, 0, (size_t)d * sizeof(double), st));
    problem_grad(Q, zero, 1, g);  // -rhs
    symv_col(S.Hinv.d(), d, g, 1, d, dx, d, S.gv.d(), st);
    CUDA_CHECK(cudaMemsetAsync(x, 0, (size_t)d * sizeof(double), st));
    add_scaled(x, dx, -1.0, d, st);
    for (int it = 0; it < refinements; ++it) {
        problem_grad(Q, x, 1, g);
        symv_col(S.Hinv.d(), d, g, 1, d, dx, d, S.gv.d(), st);
        add_scaled(x, dx, -1.0, d, st);
    }
    CUDA_CHECK(cudaStreamSynchronize(st));
    S.st = nullptr;
}

// pcg_sketch_size (baselines.hpp:170-187)
std::pair<int64_t, bool> pcg_sketch_size_impl(int64_t n, int64_t d, int32_t kind, double rho) {
    if (!(rho > 0.0 && rho < 1.0)) fail(IHS_INVALID_INPUT, "pcg_sketch_size: rho must be in (0,1)");
    const double m_raw = kind == IHS_SKETCH_GAUSSIAN ? (double)d / rho : (double)d * std::log((double)d) / rho;
    int64_t m = std::max<int64_t>((int64_t)std::ceil(m_raw), 1);
    bool capped = false;
    if (kind == IHS_SKETCH_SRHT) {
        int64_t n_pad = 1;
        while (n_pad < n) n_pad <<= 1;
        if (m > n_pad) {
            m = n_pad;
            capped = true;
        }
    }
    return {m, capped};
}

}  // namespace
}  // namespace ihs_b200

// ============================================================== C-ABI
// Gradient plan (+ row-major copy of A when it fits), solver vectors, events and the phase
// timer of a problem whose A and b are on the device.
void finish_setup(ihs_gpu_problem* Q) {
    Q->gplan = grad_plan(Q->n, Q->d, Q->lda, Q->num_sms);
    {
        // row-major copy of A for the gradient when it fits comfortably in HBM
        size_t free_b = 0, total_b = 0;
        CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
        const size_t need = (size_t)Q->lda * Q->d * sizeof(double);
        // keep room for the SRHT scratch (capped, see kSrhtScratchCap) and 8 GiB of other buffers
        int64_t np = 1;
        while (np < Q->n) np <<= 1;
        const size_t srht_scratch = (size_t)std::min<int64_t>(np * Q->d * (int64_t)sizeof(double), kSrhtScratchCap);
        GradPlan rm = Q->gplan;
        if (need + srht_scratch + (8ull << 30) < free_b && grad_plan_use_rowmajor(rm)) {
            Q->gplan = rm;
            Q->Arm.ensure(need);
            transpose_to_rowmajor(Q->A.d(), Q->lda, Q->lda, Q->d, Q->Arm.d(), Q->st);
        } else {
            grad_plan_attach_tma(Q->gplan, Q->A.d());
        }
    }
    Q->grad_work.ensure(grad_work_doubles(Q->gplan) * sizeof(double));
    Q->vecs.ensure((size_t)28 * Q->d * sizeof(double));
    Q->dots.ensure(24 * sizeof(double));
    Q->h_dots.ensure(24 * sizeof(double));
    for (auto& e : Q->set_ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : Q->set_ready) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_CHECK(cudaStreamCreateWithFlags(&Q->st2, cudaStreamNonBlocking));
    Q->owner2.s = Q->st2;
    CUDA_CHECK(cudaEventCreateWithFlags(&Q->a_ready, cudaEventDisableTiming));
    Q->timer = std::make_unique<PhaseTimer>(Q->st);
    {
        // IHS_PHASE_TIMER=0: no per-phase events (A/B of the timers' own cost)
        const char* e = std::getenv("IHS_PHASE_TIMER");
        Q->timer->enabled = !(e && e[0] == '0');
    }
}

// The dual of an underdetermined instance (dual.hpp:13-33): an overdetermined ridge problem in
// M = A^T (d x n), observation vector 0 and gradient M^T(M z) + nu^2 z - b, built on the device.
ihs_gpu_problem* dual_problem(ihs_gpu_problem* P) {
    ensure_A(P);
    if (P->dual) return P->dual.get();
    auto D = std::make_unique<ihs_gpu_problem>();
    D->device = P->device;
    D->opts = P->opts;
    D->opts.world_size = 1;
    D->opts.n_global = P->d;
    D->opts.row_offset = 0;
    D->n = P->d;
    D->d = P->n;
    D->nu = P->nu;
    D->orientation = IHS_OVERDETERMINED;
    D->num_sms = P->num_sms;
    D->st = P->st;  // shares the instance's stream (no owner: P owns it)
    D->lda = ceil_div(D->n, 32) * 32;
    D->A.ensure((size_t)D->lda * D->d * sizeof(double));
    D->b.ensure((size_t)D->lda * sizeof(double));
    CUDA_CHECK(cudaMemsetAsync(D->A.p, 0, (size_t)D->lda * D->d * sizeof(double), D->st));
    CUDA_CHECK(cudaMemsetAsync(D->b.p, 0, (size_t)D->lda * sizeof(double), D->st));
    // D->A[i + j * lda_D] = A[j + i * lda]: A's rows become M's columns
    transpose_to_rowmajor(P->A.d(), P->lda, P->n, P->d, D->A.d(), D->st, D->lda);
    D->gsub = P->b.d();
    finish_setup(D.get());
    CUDA_CHECK(cudaStreamSynchronize(D->st));
    P->dual = std::move(D);
    return P->dual.get();
}


void adaptive_solve_impl(ihs_gpu_problem* P, const ihs_solver_config* cfg, ihs_solve_report* rep);

extern "C" {

const char* ihs_gpu_last_error(void) { return ihs_b200::g_last_error.c_str(); }
const char* ihs_gpu_version(void) { return "ihs-b200 0.1.0 (sm_100a)"; }
int64_t ihs_gpu_kernel_launch_count(void) { return ihs_b200::g_launches.load(); }
int ihs_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t ihs_derive_seed(uint64_t seed, uint64_t tag) { return ihs_b200::derive_seed(seed, tag); }
int64_t ihs_next_pow2(int64_t n) {
    int64_t p = 1;
    while (p < n) p <<= 1;
    return n <= 0 ? 1 : p;
}

ihs_status ihs_rates_from_bounds(double lam, double Lam, ihs_tuning* tp) {  // tuning.hpp:25-38
    return guarded([&] {
        if (!(lam > 0.0) || !(lam <= Lam)) fail(IHS_INVALID_INPUT, "rates_from_bounds: need 0 < lam <= Lam");
        tp->lam = lam;
        tp->Lam = Lam;
        tp->mu_gd = 2.0 / (1.0 / lam + 1.0 / Lam);
        const double r = (Lam - lam) / (Lam + lam);
        tp->c_gd = r * r;
        const double sl = std::sqrt(lam), sL = std::sqrt(Lam);
        tp->mu_p = 4.0 / ((1.0 / sl + 1.0 / sL) * (1.0 / sl + 1.0 / sL));
        const double q = (sL - sl) / (sL + sl);
        tp->beta_p = tp->c_p = q * q;
    });
}

ihs_status ihs_gaussian_targets(double rho, double eta, int enforce, double* lam, double* Lam) {  // :47-56
    return guarded([&] {
        if (!(rho > 0.0) || !(eta > 0.0)) fail(IHS_INVALID_INPUT, "gaussian_targets: rho, eta must be positive");
        if (enforce && (rho > 0.18 || eta > 0.01))
            fail(IHS_OUT_OF_VALIDITY_RANGE, "gaussian_targets: proven region is rho <= 0.18, eta <= 0.01");
        const double ce = (1.0 + 3.0 * std::sqrt(eta)) * (1.0 + 3.0 * std::sqrt(eta));
        const double s = std::sqrt(ce * rho);
        if (s >= 1.0) fail(IHS_OUT_OF_VALIDITY_RANGE, "gaussian_targets: c_eta * rho must be < 1");
        *lam = (1.0 - s) * (1.0 - s);
        *Lam = (1.0 + s) * (1.0 + s);
    });
}

ihs_status ihs_srht_targets(double rho, double* lam, double* Lam) {  // :59-63
    return guarded([&] {
        if (!(rho > 0.0 && rho < 1.0)) fail(IHS_INVALID_INPUT, "srht_targets: rho must be in (0,1)");
        const double s = std::sqrt(rho);
        *lam = 1.0 - s;
        *Lam = 1.0 + s;
    });
}

void ihs_solver_config_default(ihs_solver_config* c) {  // solver.hpp:28-57
    std::memset(c, 0, sizeof(*c));
    c->rho = 0.1;
    c->eta = 0.01;
    c->sketch_kind = IHS_SKETCH_GAUSSIAN;
    c->mode = IHS_MODE_POLYAK_THEN_GRADIENT;
    c->m_initial = 1;
    c->eps = 1e-10;
    c->max_iters = 500;
    c->max_sketch = 0;
    c->seed = 0;
    c->enforce_validity = 1;
    c->recompute_r_after_resketch = 1;
    c->record_iterates = 0;
}

ihs_status ihs_sample_without_replacement(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out) {
    return guarded([&] {
        if (m < 0 || m > n) fail(IHS_INVALID_INPUT, "sample_without_replacement: need 0 <= m <= n");
        ihs_b200::sample_without_replacement(stream_seed, n, m, out);
    });
}

ihs_status ihs_newton_decrement(const double* g, const double* gt, int64_t d, double* r) {  // :95-101
    return guarded([&] {
        double dot = 0.0, sq = 0.0;
        for (int64_t i = 0; i < d; ++i) {
            dot += g[i] * gt[i];
            sq += g[i] * g[i];
        }
        const double v = 0.5 * dot;
        if (v < -1e-12 * (1.0 + sq)) fail(IHS_NUMERICAL_BREAKDOWN, "newton_decrement: negative decrement");
        *r = v < 0.0 ? 0.0 : v;
    });
}

// ------------------------------------------------------------------ sharding
ihs_status ihs_gpu_shard_rows(int64_t n_global, int32_t world_size, int32_t rank, int64_t* row0, int64_t* rows) {
    return guarded([&] {
        if (n_global < 1 || world_size < 1 || rank < 0 || rank >= world_size)
            fail(IHS_INVALID_INPUT, "shard_rows: bad arguments");
        const int64_t n_loc = ihs_next_pow2(n_global) / world_size;
        if (n_loc < 32) fail(IHS_INVALID_INPUT, "shard_rows: fewer than 32 padded rows per shard");
        *row0 = (int64_t)rank * n_loc;
        *rows = std::max<int64_t>(0, std::min<int64_t>(n_loc, n_global - *row0));
        if (*rows < 1) fail(IHS_INVALID_INPUT, "shard_rows: a shard would hold no real rows");
    });
}

ihs_status ihs_gpu_nccl_unique_id(uint8_t out[128]) {
    return guarded([&] { nccl_unique_id(out); });
}

ihs_status ihs_gpu_nccl_comm_create(const uint8_t id[128], int32_t world_size, int32_t rank, int32_t device,
                                    void** comm) {
    return guarded([&] {
        DeviceGuard g(device);
        *comm = nccl_comm_create(id, world_size, rank);
    });
}

ihs_status ihs_gpu_emu_comm_create(int32_t world_size, int32_t device, void** comms) {
    return guarded([&] {
        if (!comms || world_size < 1 || world_size > 64) fail(IHS_INVALID_INPUT, "emu_comm_create: bad arguments");
        DeviceGuard g(device);
        emu_comm_create(world_size, comms);
    });
}

void ihs_gpu_nccl_comm_destroy(void* comm) {
    try {
        nccl_comm_destroy(comm);
    } catch (...) {
    }
}

ihs_status ihs_gpu_sketch_sharded_emulated(ihs_gpu_problem* P, int32_t kind, int64_t m, uint64_t seed,
                                           int32_t shards, double* SA_out) {
    return guarded([&] {
        if (!P || !SA_out) fail(IHS_INVALID_INPUT, "null argument");
        if (P->opts.world_size > 1) fail(IHS_INVALID_INPUT, "emulation runs on a single-GPU problem");
        if (kind != IHS_SKETCH_SRHT) fail(IHS_INVALID_INPUT, "sharded emulation covers the SRHT");
        DeviceGuard dg(P->device);
        StreamScope scope(P->st);
        DevBuf SA;
        SA.ensure((size_t)m * P->d * sizeof(double));
        device_sketch(P, kind, m, seed, SA.d(), nullptr, shards);
        CUDA_CHECK(cudaMemcpyAsync(SA_out, SA.p, (size_t)m * P->d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

// ------------------------------------------------------------------ problem
ihs_status ihs_gpu_problem_create(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                                  int32_t orientation, const ihs_gpu_options* opts, ihs_gpu_problem** out) {
    return guarded([&] {
        *out = nullptr;
        // ProblemInstance validation order (problem.hpp:24-32)
        if (!(nu > 0.0)) fail(IHS_INVALID_INPUT, "ProblemInstance: nu must be strictly positive");
        if (n < 1 || d < 1) fail(IHS_INVALID_INPUT, "ProblemInstance: empty matrix");
        if (!A || !b) fail(IHS_INVALID_INPUT, "ProblemInstance: size of b must match rows of A");
        if (lda < n) fail(IHS_INVALID_INPUT, "ProblemInstance: lda < n");
        for (int64_t j = 0; j < d; ++j) check_finite_host(A + j * lda, n, "ProblemInstance: non-finite input");
        check_finite_host(b, n, "ProblemInstance: non-finite input");
        if (!std::isfinite(nu)) fail(IHS_INVALID_INPUT, "ProblemInstance: non-finite input");
        const int64_t n_global = (opts && opts->world_size > 1) ? opts->n_global : n;
        if (orientation == IHS_OVERDETERMINED && n_global < d)
            fail(IHS_INVALID_INPUT, "ProblemInstance: overdetermined orientation requires n >= d");
        if (orientation == IHS_UNDERDETERMINED && d < n_global)
            fail(IHS_INVALID_INPUT, "ProblemInstance: underdetermined orientation requires d >= n");
        if (orientation == IHS_UNDERDETERMINED && opts && opts->world_size > 1)
            fail(IHS_INVALID_INPUT, "ihs_gpu: underdetermined (dual) instances run on a single GPU");
        auto P = std::make_unique<ihs_gpu_problem>();
        P->device = opts ? opts->device : 0;
        if (opts) P->opts = *opts;
        if (P->opts.world_size < 1) P->opts.world_size = 1;
        if (P->opts.world_size > 1) {
            // row shard of the padded index space: rank r owns [r*n_loc, (r+1)*n_loc)
            const int w = P->opts.world_size, r = P->opts.rank;
            if ((w & (w - 1)) != 0 || w > 16) fail(IHS_INVALID_INPUT, "sharded problem: world_size must be 2, 4, 8 or 16");
            if (r < 0 || r >= w) fail(IHS_INVALID_INPUT, "sharded problem: rank out of range");
            if (!P->opts.nccl_comm) fail(IHS_INVALID_INPUT, "sharded problem: nccl_comm is required");
            int64_t row0 = 0, rows = 0;
            if (ihs_gpu_shard_rows(P->opts.n_global, w, r, &row0, &rows) != IHS_OK) fail(IHS_INVALID_INPUT, g_last_error);
            if (P->opts.row_offset != row0 || n != rows)
                fail(IHS_INVALID_INPUT, "sharded problem: local rows must be ihs_gpu_shard_rows(n_global, world, rank)");
        } else {
            P->opts.n_global = n;
            P->opts.row_offset = 0;
        }
        DeviceGuard g(P->device);
        P->n = n;
        P->d = d;
        P->nu = nu;
        P->orientation = orientation;
        P->num_sms = sm_count(P->device);
        configure_pool(P->device);
        CUDA_CHECK(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
        P->owner.s = P->st;
        StreamScope scope(P->st);
        alloc_and_upload(P.get(), A, lda, b);
        finish_setup(P.get());
        CUDA_CHECK(cudaStreamSynchronize(P->st));
        *out = P.release();
    });
}

void ihs_gpu_problem_destroy(ihs_gpu_problem* p) {
    if (!p) return;
    try {
        DeviceGuard g(p->device);
        cudaStreamSynchronize(p->st);
        delete p;
    } catch (...) {
    }
}

int64_t ihs_gpu_problem_rows(const ihs_gpu_problem* p) { return p ? p->n : 0; }
int64_t ihs_gpu_problem_cols(const ihs_gpu_problem* p) { return p ? p->d : 0; }

ihs_status ihs_gpu_problem_set_phase_timing(ihs_gpu_problem* P, int32_t enabled) {
    return guarded([&] {
        if (!P || !P->timer) fail(IHS_INVALID_INPUT, "set_phase_timing: null problem");
        P->timer->enabled = enabled != 0;
    });
}

ihs_status ihs_gpu_problem_upload(ihs_gpu_problem* P, const double* A, int64_t lda, const double* b) {
    return guarded([&] {
        if (!P) fail(IHS_INVALID_INPUT, "null problem");
        DeviceGuard g(P->device);
        if (A && lda < P->n) fail(IHS_INVALID_INPUT, "lda < n");
        ensure_A(P);
        upload_Ab(P, A, lda, b);
        if (A && P->dual) {  // the dual problem holds a transposed copy of A: rebuild it on next use
            CUDA_CHECK(cudaStreamSynchronize(P->st));
            P->dual.reset();
        }
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

ihs_status ihs_gpu_problem_upload_async(ihs_gpu_problem* P, const double* A, int64_t lda, const double* b) {
    return guarded([&] {
        if (!P) fail(IHS_INVALID_INPUT, "null problem");
        DeviceGuard g(P->device);
        if (A && lda < P->n) fail(IHS_INVALID_INPUT, "lda < n");
        // the copy must not overtake work still reading the previous A (or a previous pending copy)
        CUDA_CHECK(cudaEventRecord(P->a_ready, P->st));
        CUDA_CHECK(cudaStreamWaitEvent(P->st2, P->a_ready, 0));
        upload_Ab(P, A, lda, b, P->st2);
        CUDA_CHECK(cudaEventRecord(P->a_ready, P->st2));
        P->a_pending = true;
        if (A && P->dual) {  // rebuilt from the new A on next use (after ensure_A)
            CUDA_CHECK(cudaStreamSynchronize(P->st));
            P->dual.reset();
        }
    });
}

ihs_status ihs_gpu_gradient(ihs_gpu_problem* P, const double* x, double* g, ihs_counters* c) {
    return guarded([&] {
        if (!P || !x || !g) fail(IHS_INVALID_INPUT, "gradient: dimension mismatch");
        DeviceGuard dg(P->device);
        const int64_t d = P->d;
        double* X = P->vecs.d();
        double* G = X + d;
        CUDA_CHECK(cudaMemcpyAsync(X, x, (size_t)d * sizeof(double), cudaMemcpyHostToDevice, P->st));
        problem_grad(P, X, 1, G);
        CUDA_CHECK(cudaMemcpyAsync(g, G, (size_t)d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
        if (c) c->matvec += 2 * (uint64_t)P->n * (uint64_t)d + (uint64_t)P->n + 2 * (uint64_t)d;  // problem.hpp:66
    });
}

// ------------------------------------------------ CG / PCG baselines (baselines.hpp)
ihs_status ihs_pcg_sketch_size(int64_t n, int64_t d, int32_t kind, double rho, int64_t* m, int32_t* capped) {
    return guarded([&] {
        if (!m || !capped) fail(IHS_INVALID_INPUT, "pcg_sketch_size: null output");
        auto [mm, c] = pcg_sketch_size_impl(n, d, kind, rho);
        *m = mm;
        *capped = c;
    });
}

extern "C++" {
namespace {
// shared frame of the three entry points: validation, device/stream scope, wall clock, device
// events and launch count; `body` runs the solve and fills the counters
template <class F>
ihs_status cg_entry(ihs_gpu_problem* P, const char* who, ihs_cg_report* rep, F&& body) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!P || !rep || !rep->x) fail(IHS_INVALID_INPUT, std::string(who) + ": null argument");
        DeviceGuard dg(P->device);
        StreamScope scope(P->st);
        const int64_t l0 = g_launches.load();
        cudaEvent_t ev[2];
        for (auto& e : ev) CUDA_CHECK(cudaEventCreate(&e));
        CUDA_CHECK(cudaEventRecord(ev[0], P->st));
        ihs_counters C{};
        rep->m = 0;
        rep->m_capped = 0;
        rep->setup_flops = 0;
        rep->times = ihs_phase_times{};
        if (P->timer) P->timer->reset();
        try {
            body(C);
        } catch (...) {
            if (P->timer) P->timer->active = false;
            for (auto e : ev) cudaEventDestroy(e);
            throw;
        }
        CUDA_CHECK(cudaEventRecord(ev[1], P->st));
        CUDA_CHECK(cudaEventSynchronize(ev[1]));
        if (P->timer) {
            double ph[6];
            int64_t phn[6];
            P->timer->collect(ph, phn);
            ihs_phase_times& T = rep->times;
            T.sketch_ms = ph[PH_SKETCH] + ph[PH_SKETCH_KERNEL];
            T.sketch_kernel_ms = ph[PH_SKETCH_KERNEL];
            T.n_sketch_kernel = phn[PH_SKETCH_KERNEL];
            T.factor_ms = ph[PH_FACTOR];
            T.gradient_ms = ph[PH_GRAD] + ph[PH_GRAD_KERNEL];
            T.gradient_kernel_ms = ph[PH_GRAD_KERNEL];
            T.n_gradient_kernel = phn[PH_GRAD_KERNEL];
            T.solve_ms = ph[PH_SOLVE];
            T.n_solve = phn[PH_SOLVE];
        }
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        for (auto e : ev) CUDA_CHECK(cudaEventDestroy(e));
        rep->counters = C;
        rep->device_ms = ms;
        rep->kernel_launches = g_launches.load() - l0;
        rep->times.kernel_launches = rep->kernel_launches;
        rep->times.total_ms = ms;
        rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// the preconditioner from a device sketch SA (m x d, already in sys.SA): Gram form + Cholesky + H_S^{-1}
void pcg_factor(ihs_gpu_problem* P, ihs_gpu_system& sys, ihs_counters& C, ihs_cg_report* rep) {
    if (P->timer) P->timer->mark(PH_FACTOR);
    rep->times.n_factor = 1;
    try {
        system_factorize(&sys, nullptr);
    } catch (const Status& e) {
        if (e.code == IHS_NUMERICAL_BREAKDOWN)
            fail(IHS_NUMERICAL_BREAKDOWN, "pcg_solve: preconditioner factorization failed");
        throw;
    }
    const uint64_t dd = (uint64_t)sys.d, mm = (uint64_t)sys.m;
    C.factor += dd * dd * mm + dd * dd * dd / 3;  // baselines.hpp:119-120
    rep->setup_flops += dd * dd * mm + dd * dd * dd / 3;
    rep->m = sys.m;
}

void pcg_system_init(ihs_gpu_problem* P, ihs_gpu_system& sys, int64_t m) {
    sys.device = P->device;
    sys.d = P->d;
    sys.m = m;
    sys.nu = P->nu;
    sys.st = P->st;
    sys.num_sms = P->num_sms;
    sys.force_gram = true;
    sys.SA.ensure((size_t)m * P->d * sizeof(double));
}
}  // namespace
}  // extern "C++"

ihs_status ihs_gpu_cg_solve(ihs_gpu_problem* P, double tol, int64_t max_iters, const double* x0,
                            ihs_cg_report* rep) {
    return cg_entry(P, "cg_solve", rep, [&](ihs_counters& C) {
        if (P->orientation != IHS_OVERDETERMINED) fail(IHS_INVALID_INPUT, "cg_solve: expects an overdetermined instance");
        cg_run(P, nullptr, tol, max_iters, x0, rep, C);
    });
}

ihs_status ihs_gpu_pcg_solve_with(ihs_gpu_problem* P, const double* SA, int64_t m, int64_t lds, double tol,
                                  int64_t max_iters, const double* x0, ihs_cg_report* rep) {
    return cg_entry(P, "pcg_solve", rep, [&](ihs_counters& C) {
        if (P->orientation != IHS_OVERDETERMINED)
            fail(IHS_INVALID_INPUT, "pcg_solve: expects an overdetermined instance");
        if (!SA || m < 1 || lds < m) fail(IHS_INVALID_INPUT, "pcg_solve: bad sketch shape");
        ihs_gpu_system sys;
        pcg_system_init(P, sys, m);
        CUDA_CHECK(cudaMemcpy2DAsync(sys.SA.p, (size_t)m * sizeof(double), SA, (size_t)lds * sizeof(double),
                                     (size_t)m * sizeof(double), (size_t)P->d, cudaMemcpyHostToDevice, P->st));
        pcg_factor(P, sys, C, rep);
        cg_run(P, &sys, tol, max_iters, x0, rep, C);
    });
}

ihs_status ihs_gpu_pcg_solve(ihs_gpu_problem* P, int32_t kind, uint64_t seed, double rho, double tol,
                             int64_t max_iters, const double* x0, ihs_cg_report* rep) {
    return cg_entry(P, "pcg_solve", rep, [&](ihs_counters& C) {
        const int64_t n_rows = P->opts.world_size > 1 ? P->opts.n_global : P->n;
        auto [m, capped] = pcg_sketch_size_impl(n_rows, P->d, kind, rho);
        if (P->orientation != IHS_OVERDETERMINED)
            fail(IHS_INVALID_INPUT, "pcg_solve: expects an overdetermined instance");
        rep->m_capped = capped;
        ihs_gpu_system sys;
        pcg_system_init(P, sys, m);
        if (P->timer) P->timer->mark(PH_SKETCH);
        device_sketch(P, kind, m, seed, sys.SA.d(), &C);  // apply_sketch(A, {kind, m, seed}) (baselines.hpp:195)
        rep->times.n_sketch = 1;
        if (kind == IHS_SKETCH_SRHT)
            rep->times.sketch_bytes = 8.0 * (double)P->n * (double)P->d + 8.0 * (double)m * (double)P->d;
        else
            rep->times.sketch_flops = 2.0 * (double)m * (double)P->n * (double)P->d;
        rep->setup_flops += C.sketch;
        pcg_factor(P, sys, C, rep);
        rep->m_capped = capped;
        cg_run(P, &sys, tol, max_iters, x0, rep, C);
    });
}

// direct_solve (problem.hpp:73-82): the exact ridge minimizer. Underdetermined instances go
// through the dual problem in A^T (x = A^T z*, z* = (A A^T + nu^2 I)^{-1} b).
ihs_status ihs_gpu_direct_solve(ihs_gpu_problem* P, double* x_out) {
    return guarded([&] {
        if (!P || !x_out) fail(IHS_INVALID_INPUT, "direct_solve: null argument");
        DeviceGuard dg(P->device);
        StreamScope scope(P->st);
        DevBuf xb;
        if (P->orientation == IHS_OVERDETERMINED) {
            xb.ensure((size_t)P->d * sizeof(double));
            direct_solve_dev(P, xb.d());
        } else {
            if (P->opts.world_size > 1) fail(IHS_INVALID_INPUT, "direct_solve: underdetermined sharded instance");
            ihs_gpu_problem* D = dual_problem(P);
            xb.ensure((size_t)(P->n + P->d) * sizeof(double));
            double* z = xb.d() + P->d;
            direct_solve_dev(D, z);
            DevBuf work;
            work.ensure((gemv_tiled_work_doubles(D->n, D->d) + 8) * sizeof(double));
            gemv_tiled_reset(work.d(), D->n, D->d, P->st);
            gemv_tiled(D->A.d(), D->n, D->d, D->lda, z, 1, D->d, xb.d(), D->n, work.d(), P->st);  // x = A^T z
        }
        CUDA_CHECK(cudaMemcpyAsync(x_out, xb.p, (size_t)P->d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

// nu of a resident problem (ProblemInstance ctor checks, problem.hpp:24-32): the regularization path
// keeps A on the device across its nu values (bench.hpp:131-171 rebuilds the instance each time)
ihs_status ihs_gpu_problem_set_nu(ihs_gpu_problem* P, double nu) {
    return guarded([&] {
        if (!P) fail(IHS_INVALID_INPUT, "null problem");
        if (!(nu > 0.0)) fail(IHS_INVALID_INPUT, "ProblemInstance: nu must be strictly positive");
        if (!std::isfinite(nu)) fail(IHS_INVALID_INPUT, "ProblemInstance: non-finite input");
        P->nu = nu;
        if (P->dual) P->dual->nu = nu;
    });
}

// problem.hpp:104-109: 1/2 ||A (x - x*)||^2 + nu^2/2 ||x - x*||^2 (one tiled mat-vec over A)
ihs_status ihs_gpu_prediction_error(ihs_gpu_problem* P, const double* x, const double* x_star, double* out) {
    return guarded([&] {
        if (!P || !x || !x_star || !out) fail(IHS_INVALID_INPUT, "prediction_error: dimension mismatch");
        DeviceGuard dg(P->device);
        StreamScope scope(P->st);
        ensure_A(P);
        const int64_t n = P->n, d = P->d;
        DevBuf v, r, work, dots;
        v.ensure((size_t)2 * d * sizeof(double));
        r.ensure((size_t)n * sizeof(double));
        work.ensure((gemv_tiled_work_doubles(n, d) + 8) * sizeof(double));
        dots.ensure(8 * sizeof(double));
        gemv_tiled_reset(work.d(), n, d, P->st);
        CUDA_CHECK(cudaMemcpyAsync(v.p, x, (size_t)d * sizeof(double), cudaMemcpyHostToDevice, P->st));
        CUDA_CHECK(cudaMemcpyAsync(v.d() + d, x_star, (size_t)d * sizeof(double), cudaMemcpyHostToDevice, P->st));
        add_scaled(v.d(), v.d() + d, -1.0, d, P->st);  // diff = x - x*
        gemv_tiled(P->A.d(), n, d, P->lda, v.d(), 1, d, r.d(), n, work.d(), P->st);
        decrement_dots(r.d(), r.d(), n, 1, dots.d(), P->st);          // ||A diff||^2 (local rows)
        decrement_dots(v.d(), v.d(), d, 1, dots.d() + 2, P->st);      // ||diff||^2
        if (P->opts.world_size > 1) nccl_allreduce_sum(dots.d(), 1, P->opts.nccl_comm, P->st);
        double h[4];
        CUDA_CHECK(cudaMemcpyAsync(h, dots.p, sizeof(h), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
        *out = 0.5 * h[0] + 0.5 * P->nu * P->nu * h[2];
    });
}

ihs_status ihs_gpu_sketch(ihs_gpu_problem* P, int32_t kind, int64_t m, uint64_t seed, double* SA_out,
                          ihs_counters* c) {
    return guarded([&] {
        if (!P) fail(IHS_INVALID_INPUT, "null problem");
        DeviceGuard dg(P->device);
        StreamScope scope(P->st);
        if (m < 1) fail(IHS_INVALID_INPUT, kind == IHS_SKETCH_SRHT ? "srht_sketch: m must be >= 1"
                                                                    : "gaussian_sketch: m must be >= 1");
        DevBuf SA;
        SA.ensure((size_t)m * P->d * sizeof(double));
        device_sketch(P, kind, m, seed, SA.d(), c);
        if (SA_out)
            CUDA_CHECK(cudaMemcpyAsync(SA_out, SA.p, (size_t)m * P->d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

ihs_status ihs_gpu_sketch_matrix(const double* A, int64_t n, int64_t d, int64_t lda, int32_t kind, int64_t m,
                                 uint64_t seed, double* SA_out, ihs_counters* c) {
    return guarded([&] {
        if (n < 1 || d < 1 || lda < n) fail(IHS_INVALID_INPUT, "sketch: empty or malformed matrix");
        if (m < 1) fail(IHS_INVALID_INPUT, kind == IHS_SKETCH_SRHT ? "srht_sketch: m must be >= 1"
                                                                    : "gaussian_sketch: m must be >= 1");
        // a throw-away problem (b = 0, nu = 1); the sketch does not look at b or nu
        ihs_gpu_problem* P = nullptr;
        auto P_holder = std::unique_ptr<ihs_gpu_problem, void (*)(ihs_gpu_problem*)>(nullptr, ihs_gpu_problem_destroy);
        {
            auto Pp = std::make_unique<ihs_gpu_problem>();
            Pp->device = 0;
            Pp->opts.world_size = 1;
            Pp->opts.n_global = n;
            CUDA_CHECK(cudaGetDevice(&Pp->device));
            Pp->n = n;
            Pp->d = d;
            Pp->nu = 1.0;
            Pp->num_sms = sm_count(Pp->device);
            configure_pool(Pp->device);
            CUDA_CHECK(cudaStreamCreateWithFlags(&Pp->st, cudaStreamNonBlocking));
            Pp->owner.s = Pp->st;
            StreamScope scope(Pp->st);
            alloc_and_upload(Pp.get(), A, lda, nullptr);
            P = Pp.release();
            P_holder.reset(P);
        }
        StreamScope scope(P->st);
        DevBuf SA;
        SA.ensure((size_t)m * d * sizeof(double));
        device_sketch(P, kind, m, seed, SA.d(), c);
        CUDA_CHECK(cudaMemcpyAsync(SA_out, SA.p, (size_t)m * d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

ihs_status ihs_gpu_fwht(double* v, int64_t n) {  // fwht_inplace (sketch.hpp:33-49)
    return guarded([&] {
        if (n <= 0 || (n & (n - 1)) != 0) fail(IHS_INVALID_INPUT, "fwht_inplace: length must be a power of two");
        int dev = 0;
        CUDA_CHECK(cudaGetDevice(&dev));
        configure_pool(dev);
        cudaStream_t st;
        CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        StreamOwner owner;
        owner.s = st;
        StreamScope scope(st);
        DevBuf dv, dT, dbits, dent, dtiles, dout;
        SrhtPlan p = srht_plan(n, 1, n, n);
        p.scale2 = 1.0;  // a single normalization pass, v *= 1/sqrt(n)
        dv.ensure((size_t)n * 8);
        dout.ensure((size_t)n * 8);
        CUDA_CHECK(cudaMemcpyAsync(dv.p, v, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        const int64_t words = (n + 31) / 32;
        dbits.ensure((size_t)words * 4);
        CUDA_CHECK(cudaMemsetAsync(dbits.p, 0xFF, (size_t)words * 4, st));  // all signs +1
        std::vector<int64_t> rows((size_t)n);
        for (int64_t i = 0; i < n; ++i) rows[(size_t)i] = i;
        std::vector<int2> ent;
        std::vector<int4> til;
        srht_build_entries(p, rows.data(), ent, til);
        dent.ensure(ent.size() * sizeof(int2));
        dtiles.ensure(til.size() * sizeof(int4) + 16);
        CUDA_CHECK(cudaMemcpyAsync(dent.p, ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
        CUDA_CHECK(cudaMemcpyAsync(dtiles.p, til.data(), til.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
        dT.ensure(srht_scratch_bytes(p) + 8);
        srht_run_device(p, dv.d(), dbits.as<uint32_t>(), dent.as<int2>(), dtiles.as<int4>(), (int)til.size(), dT.d(),
                        dout.d(), st);
        CUDA_CHECK(cudaMemcpyAsync(v, dout.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

// ------------------------------------------------------------- RNG parity
ihs_status ihs_gpu_rademacher_bits(uint64_t stream_seed, int64_t n, uint32_t* out_bits) {
    return guarded([&] {
        if (n < 0) fail(IHS_INVALID_INPUT, "rademacher: n < 0");
        const int64_t words = (n + 31) / 32;
        DevBuf buf;
        buf.ensure((size_t)words * 4 + 4);
        DevBuf scratch;
        scratch.ensure(rademacher_scratch_bytes(n));
        mt_rademacher_bits(stream_seed, n, buf.as<uint32_t>(), scratch.p, 0);
        CUDA_CHECK(cudaMemcpy(out_bits, buf.p, (size_t)words * 4, cudaMemcpyDeviceToHost));
    });
}

ihs_status ihs_gpu_fill_gaussian(uint64_t stream_seed, int64_t rows, int64_t cols, double stddev, double* out) {
    return guarded([&] {
        const int64_t count = rows * cols;
        if (rows < 0 || cols < 0) fail(IHS_INVALID_INPUT, "fill_gaussian: negative shape");
        if (count == 0) return;
        DevBuf o, scratch;
        o.ensure((size_t)count * 8);
        scratch.ensure(gaussian_scratch_bytes(count));
        mt_fill_gaussian(stream_seed, 0, count, stddev, o.d(), scratch.p, 0);
        CUDA_CHECK(cudaMemcpy(out, o.p, (size_t)count * 8, cudaMemcpyDeviceToHost));
    });
}

// normals [first, first + count) of fill_gaussian(make_stream) — a row shard's columns of S; streamed != 0
// uses the chunked generator of tall Gaussian sketches (in blocks of `block` normals)
ihs_status ihs_gpu_fill_gaussian_window(uint64_t stream_seed, int64_t first, int64_t count, double stddev,
                                        int32_t streamed, int64_t block, double* out) {
    return guarded([&] {
        if (first < 0 || count < 0) fail(IHS_INVALID_INPUT, "fill_gaussian: negative window");
        if (count == 0) return;
        DevBuf o, scratch;
        if (!streamed) {
            o.ensure((size_t)count * 8);
            scratch.ensure(gaussian_scratch_bytes(first + count));
            mt_fill_gaussian(stream_seed, first, count, stddev, o.d(), scratch.p, 0);
            CUDA_CHECK(cudaMemcpy(out, o.p, (size_t)count * 8, cudaMemcpyDeviceToHost));
            return;
        }
        if (block < 2) fail(IHS_INVALID_INPUT, "fill_gaussian: block must be >= 2");
        const int64_t cap = block + 2 * gaussian_stream_chunk_attempts() + 16;
        o.ensure((size_t)cap * 8);
        scratch.ensure(gaussian_stream_scratch_bytes());
        int64_t done = 0;
        auto consume = [&](int64_t base, int64_t ready) -> int64_t {
            // any even prefix (the window is not column-structured here); the window's end is taken whole
            const int64_t use = base + ready >= first + count ? ready : (ready & ~int64_t{1});
            if (use <= 0) return 0;
            CUDA_CHECK(cudaMemcpy(out + (base - first), o.p, (size_t)use * 8, cudaMemcpyDeviceToHost));
            done += use;
            return use;
        };
        mt_gaussian_stream(stream_seed, first, count, stddev, o.d(), cap, block, scratch.p, 0, consume);
        if (done != count) fail(IHS_INTERNAL_ERROR, "fill_gaussian: incomplete window");
    });
}

ihs_status ihs_gpu_mt19937_64(uint64_t stream_seed, int64_t count, uint64_t* out) {
    return guarded([&] {
        if (count <= 0) return;
        DevBuf o;
        o.ensure((size_t)count * 8);
        mt_generate_raw(stream_seed, count, o.as<uint64_t>(), 0);
        CUDA_CHECK(cudaMemcpy(out, o.p, (size_t)count * 8, cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------------------------ system
ihs_status ihs_gpu_system_factorize(const double* SA, int64_t m, int64_t d, int64_t lds, double nu, int32_t device,
                                    ihs_counters* c, ihs_gpu_system** out) {
    return guarded([&] {
        *out = nullptr;
        if (!(nu > 0.0)) fail(IHS_INVALID_INPUT, "SketchedSystem: nu must be positive");
        if (m < 1 || d < 1 || lds < m) fail(IHS_INVALID_INPUT, "SketchedSystem: bad shape");
        for (int64_t j = 0; j < d; ++j) check_finite_host(SA + j * lds, m, "SketchedSystem: non-finite sketched matrix");
        DeviceGuard g(device);
        auto S = std::make_unique<ihs_gpu_system>();
        S->device = device;
        S->m = m;
        S->d = d;
        S->nu = nu;
        S->num_sms = sm_count(device);
        configure_pool(device);
        CUDA_CHECK(cudaStreamCreateWithFlags(&S->st, cudaStreamNonBlocking));
        S->owner.s = S->st;
        StreamScope scope(S->st);
        S->SA.ensure((size_t)m * d * sizeof(double));
        CUDA_CHECK(cudaMemcpy2DAsync(S->SA.p, (size_t)m * sizeof(double), SA, (size_t)lds * sizeof(double),
                                     (size_t)m * sizeof(double), (size_t)d, cudaMemcpyHostToDevice, S->st));
        system_factorize(S.get(), c);
        *out = S.release();
    });
}

void ihs_gpu_system_destroy(ihs_gpu_system* s) {
    if (!s) return;
    try {
        DeviceGuard g(s->device);
        cudaStreamSynchronize(s->st);
        delete s;
    } catch (...) {
    }
}
int32_t ihs_gpu_system_kind(const ihs_gpu_system* s) { return s ? s->kind : -1; }
int64_t ihs_gpu_system_m(const ihs_gpu_system* s) { return s ? s->m : 0; }
int64_t ihs_gpu_system_d(const ihs_gpu_system* s) { return s ? s->d : 0; }
uint64_t ihs_gpu_system_factor_flops(const ihs_gpu_system* s) { return s ? s->factor_flops() : 0; }
uint64_t ihs_gpu_system_flops_per_solve(const ihs_gpu_system* s) { return s ? s->flops_per_solve() : 0; }

ihs_status ihs_gpu_system_solve(const ihs_gpu_system* S, const double* g, double* z, ihs_counters* c) {
    return guarded([&] {
        if (!S || !g || !z) fail(IHS_INVALID_INPUT, "SketchedSystem::solve: dimension mismatch");
        DeviceGuard dg(S->device);
        StreamScope scope(S->st);
        DevBuf buf;
        buf.ensure((size_t)2 * S->d * sizeof(double));
        double* dg_ = buf.d();
        double* dz = dg_ + S->d;
        CUDA_CHECK(cudaMemcpyAsync(dg_, g, (size_t)S->d * 8, cudaMemcpyHostToDevice, S->st));
        system_solve_dev(S, dg_, dz, 1);
        CUDA_CHECK(cudaMemcpyAsync(z, dz, (size_t)S->d * 8, cudaMemcpyDeviceToHost, S->st));
        CUDA_CHECK(cudaStreamSynchronize(S->st));
        if (c) c->solve += S->flops_per_solve();
    });
}

// ------------------------------------------------------------ adaptive solve
ihs_status ihs_gpu_adaptive_solve(ihs_gpu_problem* P, const ihs_solver_config* cfg, ihs_solve_report* rep) {
    return guarded([&] {
        if (!P || !cfg || !rep || !rep->x) fail(IHS_INVALID_INPUT, "adaptive_solve: null argument");
        // solver.hpp:243-245
        if (P->orientation != IHS_OVERDETERMINED)
            fail(IHS_INVALID_INPUT, "adaptive_solve: expects an overdetermined instance (use solve_underdetermined for d > n)");
        adaptive_solve_impl(P, cfg, rep);
    });
}

// dual.hpp:13-33: adaptive IHS on the dual problem in A^T, primal x = A^T z
ihs_status ihs_gpu_solve_underdetermined(ihs_gpu_problem* P, const ihs_solver_config* cfg, ihs_solve_report* rep) {
    return guarded([&] {
        if (!P || !cfg || !rep || !rep->x) fail(IHS_INVALID_INPUT, "solve_underdetermined: null argument");
        if (P->orientation != IHS_UNDERDETERMINED)
            fail(IHS_INVALID_INPUT, "solve_underdetermined: expects an underdetermined instance");
        DeviceGuard dgd(P->device);
        StreamScope scope(P->st);
        ihs_gpu_problem* D = dual_problem(P);
        const int64_t n = P->n, d = P->d;
        std::vector<double> z((size_t)n);
        ihs_solve_report rd = *rep;
        rd.x = z.data();
        adaptive_solve_impl(D, cfg, &rd);
        double* x_out = rep->x;
        double* dual_out = rep->dual_final;
        *rep = rd;
        rep->x = x_out;
        rep->dual_final = dual_out;
        if (dual_out) std::memcpy(dual_out, z.data(), (size_t)n * sizeof(double));
        // x = A^T z = M z (M = A^T, d x n on the dual problem)
        DevBuf dz, dx, work;
        dz.ensure((size_t)n * sizeof(double));
        dx.ensure((size_t)d * sizeof(double));
        work.ensure((gemv_tiled_work_doubles(d, n) + 8) * sizeof(double));
        gemv_tiled_reset(work.d(), d, n, P->st);
        CUDA_CHECK(cudaMemcpyAsync(dz.p, z.data(), (size_t)n * sizeof(double), cudaMemcpyHostToDevice, P->st));
        gemv_tiled(D->A.d(), d, n, D->lda, dz.d(), 1, n, dx.d(), d, work.d(), P->st);
        CUDA_CHECK(cudaMemcpyAsync(x_out, dx.p, (size_t)d * sizeof(double), cudaMemcpyDeviceToHost, P->st));
        CUDA_CHECK(cudaStreamSynchronize(P->st));
    });
}

}  // extern "C"

// The adaptive loop (solver.hpp:106-232) on a device problem; throws Status.
void adaptive_solve_impl(ihs_gpu_problem* P, const ihs_solver_config* cfg, ihs_solve_report* rep) {
    {
        DeviceGuard dgd(P->device);
        StreamScope scope(P->st);
        // solver.hpp:107-109
        if (!(cfg->eps > 0.0 && cfg->eps < 1.0)) fail(IHS_INVALID_INPUT, "adaptive_solve: eps must be in (0,1)");
        if (cfg->m_initial < 1) fail(IHS_INVALID_INPUT, "adaptive_solve: m_initial must be >= 1");
        if (cfg->max_iters < 1) fail(IHS_INVALID_INPUT, "adaptive_solve: max_iters must be >= 1");

        const auto t_start = std::chrono::steady_clock::now();
        // IHS_TRACE=1: host-side timeline of the solve on stderr (where the host blocks and for how long)
        static const bool trace_on = [] {
            const char* e = std::getenv("IHS_TRACE");
            return e && e[0] == '1';
        }();
        auto trace = [&](const char* what, double a = 0.0) {
            if (!trace_on) return;
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
            std::fprintf(stderr, "[ihs-trace] %9.3f ms  %s %g\n", ms, what, a);
        };
        const int64_t dim = P->d;
        const int64_t n_rows = P->opts.world_size > 1 ? P->opts.n_global : P->n;
        cudaStream_t st = P->st;
        PhaseTimer& tm = *P->timer;
        tm.reset();
        const int64_t launches0 = g_launches.load();
        const int64_t alloc0 = g_alloc_ns.load(), rng0 = g_host_rng_ns.load();
        ihs_phase_times PT{};
        cudaEvent_t ev_begin = tm.get(), ev_end = tm.get();
        CUDA_CHECK(cudaEventRecord(ev_begin, st));

        // tuning (solver.hpp:115-124)
        ihs_tuning tp{};
        if (cfg->has_tuning_override) {
            tp = cfg->tuning_override;
        } else {
            double lam = 0, Lam = 0;
            ihs_status s = cfg->sketch_kind == IHS_SKETCH_GAUSSIAN
                               ? ihs_gaussian_targets(cfg->rho, cfg->eta, cfg->enforce_validity, &lam, &Lam)
                               : ihs_srht_targets(cfg->rho, &lam, &Lam);
            if (s != IHS_OK) fail(s, g_last_error);
            s = ihs_rates_from_bounds(lam, Lam, &tp);
            if (s != IHS_OK) fail(s, g_last_error);
        }
        // growth cap (solver.hpp:128-130)
        int64_t cap = cfg->sketch_kind == IHS_SKETCH_SRHT ? ihs_next_pow2(n_rows) : n_rows;
        if (cfg->max_sketch > 0) cap = std::min(cap, cfg->max_sketch);
        cap = std::max(cap, cfg->m_initial);

        ihs_counters C{};
        std::vector<ihs_iteration_record> log;
        int64_t iterates_written = 0;
        auto push_iterate = [&](const double* d_x) {
            if (!cfg->record_iterates) return;
            if (rep->iterates && iterates_written < rep->iterates_capacity)
                CUDA_CHECK(cudaMemcpyAsync(rep->iterates + iterates_written * dim, d_x, (size_t)dim * 8,
                                           cudaMemcpyDeviceToHost, st));
            ++iterates_written;
        };

        int64_t m = cfg->m_initial, K = 0;
        // system for the current sketch
        ihs_gpu_system sys;
        sys.device = P->device;
        sys.d = dim;
        sys.nu = P->nu;
        sys.st = st;
        sys.num_sms = P->num_sms;
        sys.defer_info = true;
        auto sketch_and_factor = [&](int64_t mm, uint64_t sub_seed) {
            trace("sketch+factor enqueue begin m=", (double)mm);
            sys.m = mm;
            sys.SA.ensure((size_t)mm * dim * sizeof(double));
            tm.mark(PH_SKETCH);
            PT.n_sketch++;
            PT.n_factor++;
            if (cfg->sketch_kind == IHS_SKETCH_SRHT)
                PT.sketch_bytes += 8.0 * (double)P->n * (double)dim + 8.0 * (double)mm * (double)dim;
            else
                PT.sketch_flops += 2.0 * (double)mm * (double)P->n * (double)dim;
            if (cfg->sketch_override) {  // solver.hpp:102: host hook, no sketch counters
                std::vector<double> h((size_t)mm * dim);
                if (cfg->sketch_override(cfg->sketch_override_user, mm, sub_seed, h.data()) != 0)
                    fail(IHS_INVALID_INPUT, "sketch_override failed");
                CUDA_CHECK(cudaMemcpyAsync(sys.SA.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
                CUDA_CHECK(cudaStreamSynchronize(st));
            } else {
                device_sketch(P, cfg->sketch_kind, mm, sub_seed, sys.SA.d(), &C);
            }
            trace("sketch enqueued");
            tm.mark(PH_FACTOR);
            system_factorize(&sys, &C);
            tm.mark(PH_END);
            trace("factor enqueued");
        };

        // Device vectors. x0/xprev0/g0/gt0 hold the starting state; candidate evaluations rotate over
        // four sets {X2 = [x_polyak; x_gd], G2, GT2, dots}, and the accepted state is a set of pointers
        // into them (no copies on accept). While the evaluation in set c is decided, the live sets are
        // c-2 (x_{t-1}), c-1 (x_t), c and the speculative evaluation's c+1, so a ring of four never
        // overwrites live data whatever the decision (accept, or re-sketch with the state unchanged).
        constexpr int NSETS = 4;
        P->vecs.ensure((size_t)(4 + 6 * NSETS) * dim * sizeof(double));
        double* base = P->vecs.d();
        double* xcur = base + 0 * dim;
        double* xprev = base + 1 * dim;
        double* g = base + 2 * dim;
        double* gt = base + 3 * dim;
        struct EvalSet {
            double *X2, *G2, *GT2, *dots, *hd;
            cudaEvent_t ev, ready;
            bool polyak;  // both candidates evaluated
        } sets[NSETS];
        P->dots.ensure(24 * sizeof(double));
        P->h_dots.ensure(24 * sizeof(double));
        double* dots = P->dots.d() + 4 * NSETS;  // first evaluation / resketch decrements
        double* hd = static_cast<double*>(P->h_dots.p) + 4 * NSETS;
        for (int k = 0; k < NSETS; ++k) {
            double* sb = base + (4 + 6 * k) * dim;
            sets[k] = EvalSet{sb, sb + 2 * dim, sb + 4 * dim, P->dots.d() + 4 * k,
                              static_cast<double*>(P->h_dots.p) + 4 * k, P->set_ev[k], P->set_ready[k], false};
        }

        auto decrement = [&](double dotv, double sq) -> double {  // sketched_system.hpp:95-101
            const double r = 0.5 * dotv;
            if (r < -1e-12 * (1.0 + sq)) fail(IHS_NUMERICAL_BREAKDOWN, "newton_decrement: negative decrement");
            return r < 0.0 ? 0.0 : r;
        };

        sketch_and_factor(m, derive_seed(cfg->seed, 0));  // solver.hpp:139-140

        if (cfg->warm_start) {
            CUDA_CHECK(cudaMemcpyAsync(xcur, cfg->warm_start, (size_t)dim * 8, cudaMemcpyHostToDevice, st));
        } else {
            CUDA_CHECK(cudaMemsetAsync(xcur, 0, (size_t)dim * 8, st));
        }
        CUDA_CHECK(cudaMemcpyAsync(xprev, xcur, (size_t)dim * 8, cudaMemcpyDeviceToDevice, st));

        // g = grad(x); gt = solve(g); r = decrement  (solver.hpp:146-150)
        tm.mark(PH_GRAD);
        problem_grad(P, xcur, 1, g);
        const double grad_pass_bytes = 8.0 * (double)P->n * (double)dim + 8.0 * (double)P->n;
        PT.n_gradient++;
        PT.gradient_bytes += grad_pass_bytes;
        PT.n_solve++;
        C.matvec += 2 * (uint64_t)n_rows * (uint64_t)dim + (uint64_t)n_rows + 2 * (uint64_t)dim;
        tm.mark(PH_SOLVE);
        system_solve_dev(&sys, g, gt, 1);
        C.solve += sys.flops_per_solve();
        decrement_dots(g, gt, dim, 1, dots, st);
        tm.mark(PH_END);
        CUDA_CHECK(cudaMemcpyAsync(hd, dots, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        system_check(&sys);
        double r = decrement(hd[0], hd[1]);
        const double r1 = r;
        push_iterate(xcur);

        int64_t t = 1;
        bool converged = !(r > cfg->eps * r1) || r1 == 0.0;  // :154
        bool checks_enabled = true;
        bool exhausted = false;

        // Enqueue the evaluation of both heavy-ball candidates of state (x, x_prev, g~) into set k:
        // built from the same state and evaluated in one pass over A (2 RHS), since the gradient
        // candidate does not depend on the Polyak outcome (:182, :190). The decrement dot products
        // are copied to the set's pinned slot and its event recorded; counters are charged only
        // when the host consumes an evaluation the reference performs.
        auto enqueue_eval = [&](int k, const double* x, const double* xp, const double* gtv, bool polyak) {
            EvalSet& S = sets[k];
            tm.mark(PH_GRAD);
            const int nr = polyak ? 2 : 1;
            double* Xe = polyak ? S.X2 : S.X2 + dim;
            double* Ge = polyak ? S.G2 : S.G2 + dim;
            double* GTe = polyak ? S.GT2 : S.GT2 + dim;
            CandSpec cs;  // the candidates are formed inside the gradient pass where the kernel supports it
            cs.x = x;
            cs.xprev = xp;
            cs.gt = gtv;
            cs.mu_p = tp.mu_p;
            cs.beta_p = tp.beta_p;
            cs.mu_gd = tp.mu_gd;
            cs.out = Xe;
            problem_grad(P, Xe, nr, Ge, &cs);
            PT.n_gradient++;
            PT.gradient_bytes += grad_pass_bytes;
            PT.n_solve += nr;
            tm.mark(PH_SOLVE);
            system_solve_dots(&sys, Ge, GTe, nr, S.dots);
            tm.mark(PH_END);
            CUDA_CHECK(cudaEventRecord(S.ready, st));
            CUDA_CHECK(cudaStreamWaitEvent(P->st2, S.ready, 0));
            CUDA_CHECK(cudaMemcpyAsync(S.hd, S.dots, (size_t)2 * nr * sizeof(double), cudaMemcpyDeviceToHost, P->st2));
            CUDA_CHECK(cudaEventRecord(S.ev, P->st2));
            S.polyak = polyak;
        };
        // Speculation: while the host waits for evaluation t, the evaluation of t+1 under the predicted
        // outcome (the previous accepted candidate kind) is already queued, hiding the host round trip.
        // Only for cheap passes over A (a wasted evaluation costs one pass) and only after an accept.
        // rank-invariant (every speculative evaluation all-reduces its gradient partials, so all ranks must
        // speculate alike): decided from the largest shard's rows, not this rank's own row count
        const bool cheap_pass = 8.0 * (double)shard_rows_max(P) * (double)(dim + 1) < (double)(1ll << 30);
        int cur = 0;        // set holding the evaluation for the current state
        int spec = -1;      // set holding a speculative evaluation (or -1)
        int spec_slot = -1; // candidate slot the speculation assumed accepted
        int last_kind = -1; // kind of the last accepted step
        const bool polyak_mode = cfg->mode == IHS_MODE_POLYAK_THEN_GRADIENT;
        if (!converged && t < cfg->max_iters) enqueue_eval(cur, xcur, xprev, gt, checks_enabled && polyak_mode);

        auto accept = [&](int slot, double rc, int kind) {  // :167-178
            const double r_prev = r;
            EvalSet& S = sets[cur];
            xprev = xcur;
            xcur = S.X2 + slot * dim;
            g = S.G2 + slot * dim;
            gt = S.GT2 + slot * dim;
            r = rc;
            ++t;
            log.push_back({t, m, r, r_prev, kind, 0});
            push_iterate(xcur);
            converged = r <= cfg->eps * r1;
            last_kind = kind;
        };
        // after the current state changed: use the speculation if it matches, else evaluate anew
        auto next_eval = [&](int accepted_slot) {
            const int nxt = (cur + 1) % NSETS;
            const bool polyak = checks_enabled && polyak_mode;
            if (spec >= 0 && accepted_slot == spec_slot && sets[spec].polyak == polyak) {
                cur = spec;
            } else {
                cur = nxt;
                if (!converged && t < cfg->max_iters) enqueue_eval(cur, xcur, xprev, gt, polyak);
            }
            spec = -1;
        };

        while (!converged && t < cfg->max_iters) {  // :180
            const bool want_polyak = checks_enabled && polyak_mode;
            EvalSet& S = sets[cur];
            // speculate the next evaluation before blocking on this one
            if (cheap_pass && last_kind >= 0 && t + 1 < cfg->max_iters) {
                spec_slot = (last_kind == IHS_STEP_POLYAK && S.polyak) ? 0 : 1;
                spec = (cur + 1) % NSETS;
                enqueue_eval(spec, S.X2 + spec_slot * dim, xcur, S.GT2 + spec_slot * dim, want_polyak);
            }
            trace("wait eval t=", (double)t);
            CUDA_CHECK(cudaEventSynchronize(S.ev));
            trace("eval ready");
            system_check(&sys);
            const double* hv = S.hd;
            const uint64_t grad_cost = 2 * (uint64_t)n_rows * (uint64_t)dim + (uint64_t)n_rows + 2 * (uint64_t)dim;
            if (want_polyak) {
                C.matvec += grad_cost;
                C.solve += sys.flops_per_solve();
                const double rp = decrement(hv[0], hv[1]);
                const double ratio = std::pow(rp / r1, 1.0 / static_cast<double>(t));  // :183
                if (ratio <= tp.c_p || rp <= cfg->eps * r1) {
                    accept(0, rp, IHS_STEP_POLYAK);
                    next_eval(0);
                    continue;
                }
            }
            C.matvec += grad_cost;
            C.solve += sys.flops_per_solve();
            const double rg = want_polyak ? decrement(hv[2], hv[3]) : decrement(hv[0], hv[1]);
            const bool pass = checks_enabled ? (rg <= tp.c_gd * r || rg <= cfg->eps * r1) : rg <= r;  // :191-193
            if (pass) {
                accept(1, rg, IHS_STEP_GRADIENT);
                next_eval(1);
                continue;
            }
            spec = -1;  // the state did not advance: any speculation is void
            last_kind = -1;
            if (!checks_enabled) break;  // :198
            if (2 * m > cap) {           // :201-209
                exhausted = true;
                checks_enabled = false;
                if (rg <= r) {
                    accept(1, rg, IHS_STEP_GRADIENT);
                    last_kind = -1;
                    next_eval(1);
                    continue;
                }
                break;
            }
            m *= 2;  // :210-220
            ++K;
            sketch_and_factor(m, derive_seed(cfg->seed, (uint64_t)K));
            tm.mark(PH_SOLVE);
            system_solve_dev(&sys, g, gt, 1);
            C.solve += sys.flops_per_solve();
            const double r_old = r;
            if (cfg->recompute_r_after_resketch) {
                decrement_dots(g, gt, dim, 1, dots, st);
                tm.mark(PH_END);
                CUDA_CHECK(cudaMemcpyAsync(hd, dots, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
                trace("wait resketch decrement");
                CUDA_CHECK(cudaStreamSynchronize(st));
                trace("resketch decrement ready");
                system_check(&sys);
                r = decrement(hd[0], hd[1]);
                converged = r <= cfg->eps * r1;
            } else {
                tm.mark(PH_END);
            }
            log.push_back({t, m, r, r_old, IHS_STEP_RESKETCH, 0});
            // re-evaluate the current state under the new system, into the same set (its rejected
            // candidates are dead; the speculation, if any, sits in the next set and is void)
            if (!converged && t < cfg->max_iters) enqueue_eval(cur, xcur, xprev, gt, checks_enabled && polyak_mode);
        }

        CUDA_CHECK(cudaMemcpyAsync(rep->x, xcur, (size_t)dim * 8, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaEventRecord(ev_end, st));
        trace("wait end");
        CUDA_CHECK(cudaStreamSynchronize(st));
        trace("end");
        system_check(&sys);
        {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev_begin, ev_end));
            PT.total_ms = ms;
        }
        rep->iterations = t;
        rep->rejections = K;
        rep->final_m = m;
        rep->r1 = r1;
        rep->r_final = r;
        rep->converged = converged ? 1 : 0;
        rep->sketch_exhausted = exhausted ? 1 : 0;
        rep->log_size = (int64_t)log.size();
        if (rep->log)
            for (int64_t i = 0; i < rep->log_size && i < rep->log_capacity; ++i) rep->log[i] = log[(size_t)i];
        rep->iterates_size = iterates_written;
        rep->counters = C;
        rep->tuning = tp;
        rep->recompute_r_after_resketch = cfg->recompute_r_after_resketch;
        rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        double ph[6];
        int64_t phn[6];
        tm.collect(ph, phn);
        PT.alloc_ms = (double)(g_alloc_ns.load() - alloc0) * 1e-6;
        PT.host_rng_ms = (double)(g_host_rng_ns.load() - rng0) * 1e-6;
        rep->times = PT;
        rep->times.sketch_ms = ph[PH_SKETCH] + ph[PH_SKETCH_KERNEL];
        rep->times.sketch_kernel_ms = ph[PH_SKETCH_KERNEL];
        rep->times.n_sketch_kernel = phn[PH_SKETCH_KERNEL];
        rep->times.factor_ms = ph[PH_FACTOR];
        rep->times.gradient_ms = ph[PH_GRAD] + ph[PH_GRAD_KERNEL];
        rep->times.gradient_kernel_ms = ph[PH_GRAD_KERNEL];
        rep->times.n_gradient_kernel = phn[PH_GRAD_KERNEL];
        rep->times.solve_ms = ph[PH_SOLVE];
        rep->times.kernel_launches = g_launches.load() - launches0;
        sys.st = nullptr;  // owned by the problem
    }
}

extern "C" {

ihs_status ihs_gpu_fixed_sketch_ihs(ihs_gpu_problem* P, const ihs_gpu_system* S, const ihs_tuning* tp, int64_t T,
                                    int32_t mode, const double* x_start, double* iterates_out) {
    return guarded([&] {
        if (!P || !S || !tp || !iterates_out || T < 0) fail(IHS_INVALID_INPUT, "fixed_sketch_ihs: bad argument");
        if (S->d != P->d) fail(IHS_INVALID_INPUT, "fixed_sketch_ihs: dimension mismatch");
        DeviceGuard dgd(P->device);
        const int64_t d = P->d;
        cudaStream_t st = P->st;
        // the system lives on its own stream: order it before ours
        cudaEvent_t ev;
        CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventRecord(ev, S->st));
        CUDA_CHECK(cudaStreamWaitEvent(st, ev, 0));
        const double mu = mode == IHS_FIXED_GRADIENT ? tp->mu_gd : tp->mu_p;  // solver.hpp:261-262
        const double beta = mode == IHS_FIXED_GRADIENT ? 0.0 : tp->beta_p;
        double* base = P->vecs.d();
        double* x = base;
        double* xp = base + d;
        double* gg = base + 2 * d;
        double* step = base + 3 * d;
        double* xn = base + 4 * d;
        if (x_start) CUDA_CHECK(cudaMemcpyAsync(x, x_start, (size_t)d * 8, cudaMemcpyHostToDevice, st));
        else CUDA_CHECK(cudaMemsetAsync(x, 0, (size_t)d * 8, st));
        CUDA_CHECK(cudaMemcpyAsync(xp, x, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
        CUDA_CHECK(cudaMemcpyAsync(iterates_out, x, (size_t)d * 8, cudaMemcpyDeviceToHost, st));
        // the system's solve kernels run on S->st; rebind temporarily to ours
        ihs_gpu_system* Sm = const_cast<ihs_gpu_system*>(S);
        cudaStream_t sst = Sm->st;
        Sm->st = st;
        try {
            for (int64_t it = 0; it < T; ++it) {
                problem_grad(P, x, 1, gg);
                system_solve_dev(Sm, gg, step, 1);
                fixed_step(x, xp, step, mu, beta, d, xn, st);
                std::swap(xp, x);   // x_prev <- x
                std::swap(x, xn);   // x <- x_next (xn becomes scratch)
                CUDA_CHECK(cudaMemcpyAsync(iterates_out + (it + 1) * d, x, (size_t)d * 8, cudaMemcpyDeviceToHost, st));
            }
            CUDA_CHECK(cudaStreamSynchronize(st));
        } catch (...) {
            Sm->st = sst;
            cudaEventDestroy(ev);
            throw;
        }
        Sm->st = sst;
        cudaEventDestroy(ev);
    });
}

ihs_status ihs_synth_generate(const ihs_synth_spec* spec, int64_t row0, int64_t rows, double* A, int64_t lda,
                              double* b, double* x_true) {
    return guarded([&] {
        if (!spec) fail(IHS_INVALID_INPUT, "synth: null spec");
        synth_generate(*spec, row0, rows, A, lda, b, x_true);
    });
}

}  // extern "C"
