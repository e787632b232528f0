// ihs_oracle_capi.cpp — ctypes surface of the CPU ORACLE (test infrastructure
// only). Shares the boundary structs of include/ihs_gpu.h so the parity tests
// drive the oracle and the CUDA path with identical configs and reports.
#include "ihs_oracle.hpp"
#include "../include/ihs_gpu.h"

#include <chrono>
#include <cstring>
#include <string>

using namespace ihs_oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return IHS_OK;
    } catch (const InvalidInput& e) { g_err = e.what(); return IHS_INVALID_INPUT; }
    catch (const OutOfValidityRange& e) { g_err = e.what(); return IHS_OUT_OF_VALIDITY_RANGE; }
    catch (const SketchTooLarge& e) { g_err = e.what(); return IHS_SKETCH_TOO_LARGE; }
    catch (const NumericalBreakdown& e) { g_err = e.what(); return IHS_NUMERICAL_BREAKDOWN; }
    catch (const std::exception& e) { g_err = e.what(); return IHS_INTERNAL_ERROR; }
}

Mat to_mat(const double* A, Index n, Index d, Index lda) {
    Mat M(n, d);
    for (Index j = 0; j < d; ++j) std::memcpy(M.col(j), A + j * lda, sizeof(double) * static_cast<size_t>(n));
    return M;
}
void add_counters(ihs_counters* out, const CostCounters& c) {
    if (!out) return;
    out->sketch += c.sketch; out->factor += c.factor; out->solve += c.solve; out->matvec += c.matvec;
}
}  // namespace

static int oracle_solve(bool dual, const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                        const ihs_solver_config* c, ihs_solve_report* rep) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu, dual);
        SolverConfig cfg;
        cfg.rho = c->rho;
        cfg.eta = c->eta;
        cfg.sketch_kind = c->sketch_kind == IHS_SKETCH_SRHT ? SketchKind::SRHT : SketchKind::Gaussian;
        cfg.m_initial = c->m_initial;
        cfg.eps = c->eps;
        cfg.max_iters = c->max_iters;
        if (c->max_sketch > 0) cfg.max_sketch = c->max_sketch;
        cfg.mode = c->mode == IHS_MODE_GRADIENT_ONLY ? SolveMode::GradientOnly : SolveMode::PolyakThenGradient;
        cfg.seed = c->seed;
        cfg.enforce_validity = c->enforce_validity != 0;
        cfg.recompute_r_after_resketch = c->recompute_r_after_resketch != 0;
        cfg.record_iterates = c->record_iterates != 0;
        if (c->warm_start) cfg.warm_start = Vec(c->warm_start, c->warm_start + (dual ? n : d));
        if (c->has_tuning_override) {
            const auto& t = c->tuning_override;
            cfg.tuning_override = TuningParams{t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
        }
        if (c->sketch_override) {
            auto fn = c->sketch_override;
            void* user = c->sketch_override_user;
            cfg.sketch_override = [fn, user](const Mat& Am, Index mm, std::uint64_t sub) {
                Mat SA(mm, Am.cols);
                if (fn(user, mm, sub, SA.a.data()) != 0) throw InvalidInput("sketch_override failed");
                return SA;
            };
        }
        SolveReport r = dual ? solve_underdetermined(p, cfg) : adaptive_solve(p, cfg);
        std::memcpy(rep->x, r.x.data(), sizeof(double) * static_cast<size_t>(d));
        if (dual && rep->dual_final)
            std::memcpy(rep->dual_final, r.dual_final.data(), sizeof(double) * static_cast<size_t>(n));
        const int64_t dim = dual ? n : d;  // iterates: the dual trace for underdetermined solves
        rep->iterations = r.iterations;
        rep->rejections = r.rejections;
        rep->final_m = r.final_m;
        rep->r1 = r.r1;
        rep->r_final = r.r_final;
        rep->converged = r.converged;
        rep->sketch_exhausted = r.sketch_exhausted;
        rep->log_size = static_cast<int64_t>(r.log.size());
        if (rep->log)
            for (int64_t i = 0; i < rep->log_size && i < rep->log_capacity; ++i) {
                const auto& e = r.log[static_cast<size_t>(i)];
                rep->log[i] = {e.t, e.m, e.r, e.r_prev, static_cast<int32_t>(e.branch), 0};
            }
        rep->iterates_size = static_cast<int64_t>(r.iterates.size());
        if (rep->iterates)
            for (int64_t i = 0; i < rep->iterates_size && i < rep->iterates_capacity; ++i)
                std::memcpy(rep->iterates + i * dim, r.iterates[static_cast<size_t>(i)].data(), sizeof(double) * static_cast<size_t>(dim));
        rep->counters = {r.counters.sketch, r.counters.factor, r.counters.solve, r.counters.matvec};
        rep->wall_seconds = r.wall_seconds;
        const auto& t = r.tuning;
        rep->tuning = {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
        rep->recompute_r_after_resketch = r.recompute_r_after_resketch;
    });
}


extern "C" {

const char* ihs_oracle_last_error(void) { return g_err.c_str(); }

uint64_t ihs_oracle_derive_seed(uint64_t seed, uint64_t tag) { return derive_seed(seed, tag); }

void ihs_oracle_mt_raw(uint64_t stream_seed, int64_t count, uint64_t* out) {
    std::mt19937_64 gen(stream_seed);
    for (int64_t i = 0; i < count; ++i) out[i] = gen();
}

void ihs_oracle_rademacher(uint64_t stream_seed, int64_t n, double* out) {
    std::mt19937_64 gen(stream_seed);
    auto e = rademacher(n, gen);
    std::memcpy(out, e.data(), sizeof(double) * static_cast<size_t>(n));
}

void ihs_oracle_sample_wor(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out) {
    std::mt19937_64 gen(stream_seed);
    auto s = sample_without_replacement(n, m, gen);
    for (int64_t k = 0; k < m; ++k) out[k] = s[static_cast<size_t>(k)];
}

void ihs_oracle_fill_gaussian(uint64_t stream_seed, int64_t rows, int64_t cols, double stddev, double* out) {
    std::mt19937_64 gen(stream_seed);
    fill_gaussian(out, rows, cols, gen, stddev);
}

int ihs_oracle_fwht(double* v, int64_t n) {
    return guarded([&] { fwht_inplace(v, static_cast<size_t>(n < 0 ? 0 : n)); });
}

int64_t ihs_oracle_next_pow2(int64_t n) { return next_pow2(n); }

int ihs_oracle_sketch(const double* A, int64_t n, int64_t d, int64_t lda, int32_t kind, int64_t m, uint64_t seed,
                      double* SA, ihs_counters* counters) {
    return guarded([&] {
        Mat Am = to_mat(A, n, d, lda);
        CostCounters c;
        Mat R = apply_sketch(Am, kind == IHS_SKETCH_SRHT ? SketchKind::SRHT : SketchKind::Gaussian, m, seed, &c);
        std::memcpy(SA, R.a.data(), sizeof(double) * R.a.size());
        add_counters(counters, c);
    });
}

int ihs_oracle_gradient(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                        const double* x, double* g, ihs_counters* counters) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        CostCounters c;
        Vec gv = gradient(p, Vec(x, x + d), &c);
        std::memcpy(g, gv.data(), sizeof(double) * static_cast<size_t>(d));
        add_counters(counters, c);
    });
}

int ihs_oracle_system_solve(const double* SA, int64_t m, int64_t d, int64_t lds, double nu, const double* g,
                            double* z, int32_t* kind, uint64_t* factor_flops, uint64_t* flops_per_solve,
                            ihs_counters* counters) {
    return guarded([&] {
        CostCounters c;
        auto sys = SketchedSystem::factorize(to_mat(SA, m, d, lds), nu, &c);
        if (kind) *kind = static_cast<int32_t>(sys.kind());
        if (factor_flops) *factor_flops = sys.factor_flops();
        if (flops_per_solve) *flops_per_solve = sys.flops_per_solve();
        if (g && z) {
            Vec zv = sys.solve(Vec(g, g + d), &c);
            std::memcpy(z, zv.data(), sizeof(double) * static_cast<size_t>(d));
        }
        add_counters(counters, c);
    });
}

int ihs_oracle_newton_decrement(const double* g, const double* gt, int64_t d, double* r) {
    return guarded([&] { *r = newton_decrement(Vec(g, g + d), Vec(gt, gt + d)); });
}

int ihs_oracle_rates_from_bounds(double lam, double Lam, ihs_tuning* out) {
    return guarded([&] {
        auto t = rates_from_bounds(lam, Lam);
        *out = {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
    });
}
int ihs_oracle_gaussian_targets(double rho, double eta, int enforce, double* lam, double* Lam) {
    return guarded([&] { auto [a, b] = gaussian_targets(rho, eta, enforce != 0); *lam = a; *Lam = b; });
}
int ihs_oracle_srht_targets(double rho, double* lam, double* Lam) {
    return guarded([&] { auto [a, b] = srht_targets(rho); *lam = a; *Lam = b; });
}

int ihs_oracle_adaptive_solve(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                              const ihs_solver_config* c, ihs_solve_report* rep) {
    return oracle_solve(false, A, n, d, lda, b, nu, c, rep);
}

// The reference tests' data helpers (proj/tests/support.hpp:32-47): gen = mt19937_64(seed);
// M = random_matrix(rows, cols, gen) (column-major, one normal_distribution), then optionally
// v = random_vector(vlen, gen) with a fresh distribution object on the same generator.
int ihs_oracle_test_support_data(uint64_t seed, int64_t rows, int64_t cols, double* M, int64_t vlen, double* v) {
    return guarded([&] {
        std::mt19937_64 gen(seed);
        {
            std::normal_distribution<double> dist;
            for (int64_t j = 0; j < cols; ++j)
                for (int64_t i = 0; i < rows; ++i) M[i + j * rows] = dist(gen);
        }
        if (vlen > 0 && v) {
            std::normal_distribution<double> dist;
            for (int64_t i = 0; i < vlen; ++i) v[i] = dist(gen);
        }
    });
}
int ihs_oracle_solve_underdetermined(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                                     const ihs_solver_config* c, ihs_solve_report* rep) {
    return oracle_solve(true, A, n, d, lda, b, nu, c, rep);
}

int ihs_oracle_fixed_sketch_ihs(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                                const double* SA, int64_t m, const ihs_tuning* tp, int64_t T, int32_t mode,
                                const double* x_start, double* out) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        auto sys = SketchedSystem::factorize(to_mat(SA, m, d, m), nu);
        TuningParams t{tp->lam, tp->Lam, tp->mu_gd, tp->c_gd, tp->mu_p, tp->beta_p, tp->c_p};
        Vec xs;
        if (x_start) xs.assign(x_start, x_start + d);
        auto its = fixed_sketch_ihs(p, sys, t, T, mode == IHS_FIXED_POLYAK ? FixedMode::Polyak : FixedMode::Gradient,
                                    x_start ? &xs : nullptr);
        for (size_t i = 0; i < its.size(); ++i) std::memcpy(out + i * d, its[i].data(), sizeof(double) * static_cast<size_t>(d));
    });
}

int ihs_oracle_direct_solve(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu, double* x) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        Vec xv = direct_solve(p);
        std::memcpy(x, xv.data(), sizeof(double) * static_cast<size_t>(d));
    });
}

int ihs_oracle_prediction_error(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                                const double* x, const double* xs, double* out) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        *out = prediction_error(p, Vec(x, x + d), Vec(xs, xs + d));
    });
}

int ihs_oracle_synth(const ihs_synth_spec* s, double* A, double* b, double* x_true) {
    return guarded([&] {
        SynthSpec sp;
        sp.n = s->n; sp.d = s->d; sp.spectrum = s->spectrum; sp.decay = s->decay; sp.noise_std = s->noise_std;
        sp.outlier_frac = s->outlier_frac; sp.outlier_scale = s->outlier_scale; sp.data_seed = s->data_seed;
        Mat Am; Vec bv, xt;
        synth_generate(sp, Am, bv, xt);
        std::memcpy(A, Am.a.data(), sizeof(double) * Am.a.size());
        std::memcpy(b, bv.data(), sizeof(double) * bv.size());
        if (x_true) std::memcpy(x_true, xt.data(), sizeof(double) * xt.size());
    });
}

// baselines.hpp: method 0 = cg_solve, 1 = pcg_solve_with(SA), 2 = pcg_solve(kind, seed, rho)
int ihs_oracle_cg(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu, int32_t method,
                  const double* SA, int64_t m, int64_t lds, int32_t kind, uint64_t seed, double rho, double tol,
                  int64_t max_iters, const double* x0, ihs_cg_report* rep) {
    return guarded([&] {
        Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        Vec xs;
        if (x0) xs.assign(x0, x0 + d);
        const Vec* xp = x0 ? &xs : nullptr;
        const SketchKind k = kind == IHS_SKETCH_SRHT ? SketchKind::SRHT : SketchKind::Gaussian;
        CgResult r = method == 0   ? cg_solve(p, tol, max_iters, xp)
                     : method == 1 ? pcg_solve_with(p, to_mat(SA, m, d, lds), tol, max_iters, CgResult{}, xp)
                                   : pcg_solve(p, k, seed, rho, tol, max_iters, xp);
        std::memcpy(rep->x, r.x.data(), sizeof(double) * static_cast<size_t>(d));
        rep->residuals_size = static_cast<int64_t>(r.residuals.size());
        if (rep->residuals)
            for (int64_t i = 0; i < rep->residuals_size && i < rep->residuals_capacity; ++i)
                rep->residuals[i] = r.residuals[static_cast<size_t>(i)];
        rep->iterations = r.iterations;
        rep->converged = r.converged;
        rep->m = r.m;
        rep->m_capped = r.m_capped;
        rep->setup_flops = r.setup_flops;
        rep->counters = ihs_counters{};
        add_counters(&rep->counters, r.counters);
    });
}

int ihs_oracle_pcg_sketch_size(int64_t n, int64_t d, int32_t kind, double rho, int64_t* m, int32_t* capped) {
    return guarded([&] {
        auto [mm, c] = pcg_sketch_size(n, d, kind == IHS_SKETCH_SRHT ? SketchKind::SRHT : SketchKind::Gaussian, rho);
        *m = mm;
        *capped = c;
    });
}

// ---- bench.py cpu_baseline: host timings of the restated reference operations on bounded samples. Inputs are
// built outside the timed region (the reference builds ProblemInstance / SketchedSystem once per solve); the
// steady_clock scope is the operation itself, as in SolveReport::wall_seconds (solver.hpp:111, 229-230).
static double secs_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ihs_oracle_time_sketch(const double* A, int64_t n, int64_t d, int64_t lda, int32_t kind, int64_t m, uint64_t seed,
                           double* seconds, ihs_counters* counters) {
    return guarded([&] {
        const Mat Am = to_mat(A, n, d, lda);
        CostCounters c;
        const auto t0 = std::chrono::steady_clock::now();
        const Mat R = apply_sketch(Am, kind == IHS_SKETCH_SRHT ? SketchKind::SRHT : SketchKind::Gaussian, m, seed, &c);
        *seconds = secs_since(t0);
        add_counters(counters, c);
        if (R.rows != m) throw InvalidInput("time_sketch: bad result");
    });
}

int ihs_oracle_time_fill_gaussian(uint64_t stream_seed, int64_t rows, int64_t cols, double* seconds) {
    return guarded([&] {
        Mat S(rows, cols);
        std::mt19937_64 gen(stream_seed);
        const auto t0 = std::chrono::steady_clock::now();
        fill_gaussian(S.a.data(), rows, cols, gen, 1.0);
        *seconds = secs_since(t0);
    });
}

int ihs_oracle_time_gradient(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                             const double* x, int32_t reps, double* seconds, ihs_counters* counters) {
    return guarded([&] {
        const Problem p(to_mat(A, n, d, lda), Vec(b, b + n), nu);
        const Vec xv(x, x + d);
        CostCounters c;
        double sink = 0.0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int32_t r = 0; r < reps; ++r) sink += gradient(p, xv, &c)[0];
        *seconds = secs_since(t0);
        add_counters(counters, c);
        if (!std::isfinite(sink)) throw InvalidInput("time_gradient: non-finite");
    });
}

int ihs_oracle_time_system(const double* SA, int64_t m, int64_t d, int64_t lds, double nu, const double* g,
                           int32_t solves, double* t_factor, double* t_solve, ihs_counters* counters) {
    return guarded([&] {
        Mat S = to_mat(SA, m, d, lds);
        const Vec gv(g, g + d);
        CostCounters c;
        auto t0 = std::chrono::steady_clock::now();
        auto sys = SketchedSystem::factorize(std::move(S), nu, &c);
        *t_factor = secs_since(t0);
        double sink = 0.0;
        t0 = std::chrono::steady_clock::now();
        for (int32_t r = 0; r < solves; ++r) sink += sys.solve(gv, &c)[0];
        *t_solve = secs_since(t0);
        add_counters(counters, c);
        if (!std::isfinite(sink)) throw InvalidInput("time_system: non-finite");
    });
}

}  // extern "C"
