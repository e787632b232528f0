// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// ctypes surface of the REFERENCE ITSELF: this file includes the reference's own headers unchanged from
// /root/reference/proj/include/ihs (rng, sketch, problem, sketched_system, tuning, solver, dual, baselines)
// and compiles them against the Eigen-API subset in oracle/eigen_stub (Eigen is absent from the image).
// oracle/Makefile builds it into oracle/_ref/libihs_ref.so (git-ignored; never part of the product).
//
// The entry points mirror oracle/ihs_oracle_capi.cpp one for one (prefix ihs_ref_ instead of ihs_oracle_),
// so tests/test_ref_pin.py drives the restated oracle and the reference code with identical inputs and
// compares them: bit-for-bit on D, P, S, the SRHT sketch, the seeds, the tuning scalars and the counters;
// m-schedule, branch log and iteration counts identical; dense-algebra results to fp64 tolerance (the
// stub's products sum in a fixed ascending order, Eigen's blocked kernels in another).
#include "ihs/baselines.hpp"
#include "ihs/dual.hpp"
#include "ihs/solver.hpp"

#include "../include/ihs_gpu.h"

#include <cstring>
#include <string>

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return IHS_OK;
    } catch (const ihs::InvalidInput& e) { g_err = e.what(); return IHS_INVALID_INPUT; }
    catch (const ihs::OutOfValidityRange& e) { g_err = e.what(); return IHS_OUT_OF_VALIDITY_RANGE; }
    catch (const ihs::SketchTooLarge& e) { g_err = e.what(); return IHS_SKETCH_TOO_LARGE; }
    catch (const ihs::NumericalBreakdown& e) { g_err = e.what(); return IHS_NUMERICAL_BREAKDOWN; }
    catch (const std::exception& e) { g_err = e.what(); return IHS_INTERNAL_ERROR; }
}

ihs::Matrix to_mat(const double* A, int64_t n, int64_t d, int64_t lda) {
    ihs::Matrix M(n, d);
    for (int64_t j = 0; j < d; ++j) std::memcpy(M.col(j).data(), A + j * lda, sizeof(double) * static_cast<size_t>(n));
    return M;
}
ihs::Vector to_vec(const double* v, int64_t n) {
    ihs::Vector out(n);
    std::memcpy(out.data(), v, sizeof(double) * static_cast<size_t>(n));
    return out;
}
void put(double* dst, const ihs::Vector& v) { std::memcpy(dst, v.data(), sizeof(double) * static_cast<size_t>(v.size())); }
void add_counters(ihs_counters* out, const ihs::CostCounters& c) {
    if (!out) return;
    out->sketch += c.sketch; out->factor += c.factor; out->solve += c.solve; out->matvec += c.matvec;
}
ihs::SketchKind kind_of(int32_t k) { return k == IHS_SKETCH_SRHT ? ihs::SketchKind::SRHT : ihs::SketchKind::Gaussian; }

int ref_solve(bool dual, const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
              const ihs_solver_config* c, ihs_solve_report* rep) {
    return guarded([&] {
        ihs::ProblemInstance p(to_mat(A, n, d, lda), to_vec(b, n), nu,
                               dual ? ihs::Orientation::Underdetermined : ihs::Orientation::Overdetermined);
        ihs::SolverConfig cfg;
        cfg.rho = c->rho;
        cfg.eta = c->eta;
        cfg.sketch_kind = kind_of(c->sketch_kind);
        cfg.m_initial = c->m_initial;
        cfg.eps = c->eps;
        cfg.max_iters = c->max_iters;
        if (c->max_sketch > 0) cfg.max_sketch = c->max_sketch;
        cfg.mode = c->mode == IHS_MODE_GRADIENT_ONLY ? ihs::SolveMode::GradientOnly : ihs::SolveMode::PolyakThenGradient;
        cfg.seed = c->seed;
        cfg.enforce_validity = c->enforce_validity != 0;
        cfg.recompute_r_after_resketch = c->recompute_r_after_resketch != 0;
        cfg.record_iterates = c->record_iterates != 0;
        if (c->warm_start) cfg.warm_start = to_vec(c->warm_start, dual ? n : d);
        if (c->has_tuning_override) {
            const auto& t = c->tuning_override;
            cfg.tuning_override = ihs::TuningParams{t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
        }
        if (c->sketch_override) {
            auto fn = c->sketch_override;
            void* user = c->sketch_override_user;
            cfg.sketch_override = [fn, user](const ihs::Matrix& Am, ihs::Index mm, std::uint64_t sub) {
                ihs::Matrix SA(mm, Am.cols());
                if (fn(user, mm, sub, SA.data()) != 0) throw ihs::InvalidInput("sketch_override failed");
                return SA;
            };
        }
        ihs::SolveReport r = dual ? ihs::solve_underdetermined(p, cfg) : ihs::adaptive_solve(p, cfg);
        put(rep->x, r.x);
        if (dual && rep->dual_final) put(rep->dual_final, r.dual_final);
        const int64_t dim = dual ? n : d;
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
                std::memcpy(rep->iterates + i * dim, r.iterates[static_cast<size_t>(i)].data(),
                            sizeof(double) * static_cast<size_t>(dim));
        rep->counters = {r.counters.sketch, r.counters.factor, r.counters.solve, r.counters.matvec};
        rep->wall_seconds = r.wall_seconds;
        const auto& t = r.tuning;
        rep->tuning = {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
        rep->recompute_r_after_resketch = r.recompute_r_after_resketch;
    });
}
}  // namespace

extern "C" {

const char* ihs_ref_last_error(void) { return g_err.c_str(); }

uint64_t ihs_ref_derive_seed(uint64_t seed, uint64_t tag) { return ihs::derive_seed(seed, tag); }

// raw draws of std::mt19937_64(stream_seed), the engine make_stream returns (rng.hpp:30-32)
void ihs_ref_mt_raw(uint64_t stream_seed, int64_t count, uint64_t* out) {
    std::mt19937_64 gen(stream_seed);
    for (int64_t i = 0; i < count; ++i) out[i] = gen();
}

void ihs_ref_rademacher(uint64_t stream_seed, int64_t n, double* out) {
    std::mt19937_64 gen(stream_seed);
    const auto e = ihs::rademacher(n, gen);
    std::memcpy(out, e.data(), sizeof(double) * static_cast<size_t>(n));
}

void ihs_ref_sample_wor(uint64_t stream_seed, int64_t n, int64_t m, int64_t* out) {
    std::mt19937_64 gen(stream_seed);
    const auto s = ihs::sample_without_replacement(n, m, gen);
    for (int64_t k = 0; k < m; ++k) out[k] = s[static_cast<size_t>(k)];
}

void ihs_ref_fill_gaussian(uint64_t stream_seed, int64_t rows, int64_t cols, double stddev, double* out) {
    std::mt19937_64 gen(stream_seed);
    ihs::Matrix M(rows, cols);
    ihs::fill_gaussian(M, gen, stddev);
    std::memcpy(out, M.data(), sizeof(double) * static_cast<size_t>(rows * cols));
}

int ihs_ref_fwht(double* v, int64_t n) {
    return guarded([&] { ihs::fwht_inplace(std::span<double>(v, static_cast<size_t>(n < 0 ? 0 : n))); });
}

int64_t ihs_ref_next_pow2(int64_t n) { return ihs::next_pow2(n); }

int ihs_ref_sketch(const double* A, int64_t n, int64_t d, int64_t lda, int32_t kind, int64_t m, uint64_t seed,
                   double* SA, ihs_counters* counters) {
    return guarded([&] {
        ihs::CostCounters c;
        const ihs::Matrix R = ihs::apply_sketch(to_mat(A, n, d, lda), ihs::SketchConfig{kind_of(kind), m, seed}, &c);
        std::memcpy(SA, R.data(), sizeof(double) * static_cast<size_t>(R.size()));
        add_counters(counters, c);
    });
}

int ihs_ref_gradient(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu, const double* x,
                     double* g, ihs_counters* counters) {
    return guarded([&] {
        const ihs::ProblemInstance p = ihs::ProblemInstance::make(to_mat(A, n, d, lda), to_vec(b, n), nu);
        ihs::CostCounters c;
        put(g, ihs::gradient(p, to_vec(x, d), &c));
        add_counters(counters, c);
    });
}

int ihs_ref_system_solve(const double* SA, int64_t m, int64_t d, int64_t lds, double nu, const double* g, double* z,
                         int32_t* kind, uint64_t* factor_flops, uint64_t* flops_per_solve, ihs_counters* counters) {
    return guarded([&] {
        ihs::CostCounters c;
        const auto sys = ihs::SketchedSystem::factorize(to_mat(SA, m, d, lds), nu, &c);
        if (kind) *kind = static_cast<int32_t>(sys.kind());
        if (factor_flops) *factor_flops = sys.factor_flops();
        if (flops_per_solve) *flops_per_solve = sys.flops_per_solve();
        if (g && z) put(z, sys.solve(to_vec(g, d), &c));
        add_counters(counters, c);
    });
}

int ihs_ref_newton_decrement(const double* g, const double* gt, int64_t d, double* r) {
    return guarded([&] { *r = ihs::newton_decrement(to_vec(g, d), to_vec(gt, d)); });
}

int ihs_ref_rates_from_bounds(double lam, double Lam, ihs_tuning* out) {
    return guarded([&] {
        const auto t = ihs::rates_from_bounds(lam, Lam);
        *out = {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
    });
}
int ihs_ref_gaussian_targets(double rho, double eta, int enforce, double* lam, double* Lam) {
    return guarded([&] { auto [a, b] = ihs::gaussian_targets(rho, eta, enforce != 0); *lam = a; *Lam = b; });
}
int ihs_ref_srht_targets(double rho, double* lam, double* Lam) {
    return guarded([&] { auto [a, b] = ihs::srht_targets(rho); *lam = a; *Lam = b; });
}

int ihs_ref_adaptive_solve(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                           const ihs_solver_config* c, ihs_solve_report* rep) {
    return ref_solve(false, A, n, d, lda, b, nu, c, rep);
}
// proj/tests/support.hpp:32-47 (random_matrix, then random_vector on the same engine); support.hpp itself
// pulls in the spectral labs through ihs.hpp, so its two loops are restated here
int ihs_ref_test_support_data(uint64_t seed, int64_t rows, int64_t cols, double* M, int64_t vlen, double* v) {
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

int ihs_ref_solve_underdetermined(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                                  const ihs_solver_config* c, ihs_solve_report* rep) {
    return ref_solve(true, A, n, d, lda, b, nu, c, rep);
}

int ihs_ref_fixed_sketch_ihs(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                             const double* SA, int64_t m, const ihs_tuning* tp, int64_t T, int32_t mode,
                             const double* x_start, double* out) {
    return guarded([&] {
        const ihs::ProblemInstance p = ihs::ProblemInstance::make(to_mat(A, n, d, lda), to_vec(b, n), nu);
        const auto sys = ihs::SketchedSystem::factorize(to_mat(SA, m, d, m), nu);
        const ihs::TuningParams t{tp->lam, tp->Lam, tp->mu_gd, tp->c_gd, tp->mu_p, tp->beta_p, tp->c_p};
        ihs::Vector xs;
        if (x_start) xs = to_vec(x_start, d);
        const auto its = ihs::fixed_sketch_ihs(p, sys, t, T,
                                               mode == IHS_FIXED_POLYAK ? ihs::FixedMode::Polyak : ihs::FixedMode::Gradient,
                                               x_start ? &xs : nullptr);
        for (size_t i = 0; i < its.size(); ++i) put(out + i * d, its[i]);
    });
}

int ihs_ref_direct_solve(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu, double* x) {
    return guarded([&] {
        const ihs::ProblemInstance p = ihs::ProblemInstance::make(to_mat(A, n, d, lda), to_vec(b, n), nu);
        put(x, ihs::direct_solve(p));
    });
}

int ihs_ref_prediction_error(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu,
                             const double* x, const double* xs, double* out) {
    return guarded([&] {
        const ihs::ProblemInstance p = ihs::ProblemInstance::make(to_mat(A, n, d, lda), to_vec(b, n), nu);
        *out = ihs::prediction_error(p, to_vec(x, d), to_vec(xs, d));
    });
}

// SURVEY §8(d) synthetic generator expressed with the reference's own primitives (make_stream,
// fill_gaussian, sample_without_replacement): G column j, row block q from make_stream(seed, 1000 + j nb + q)
// (a fresh distribution per block), x_true tag 12, noise tag 13, outliers tag 14, b = A x_true + noise
// summed over j in order.
int ihs_ref_synth(const ihs_synth_spec* s, double* A, double* b, double* x_true) {
    return guarded([&] {
        const ihs::Index n = s->n, d = s->d;
        const ihs::Index n_pad = ihs::next_pow2(n);
        const ihs::Index B = std::min<ihs::Index>(ihs::Index{1} << 16, n_pad);
        const ihs::Index nb = (n + B - 1) / B;
        for (ihs::Index j = 0; j < d; ++j) {
            const double sigma = s->spectrum == 0 ? std::pow(s->decay, static_cast<double>(j + 1))
                                                  : 1.0 / static_cast<double>(j + 1);
            for (ihs::Index q = 0; q < nb; ++q) {
                auto gen = ihs::make_stream(s->data_seed, static_cast<std::uint64_t>(1000 + j * nb + q));
                const ihs::Index r0 = q * B, r1 = std::min(n, r0 + B);
                ihs::Vector v(r1 - r0);
                ihs::fill_gaussian(v, gen, 1.0);
                for (ihs::Index i = r0; i < r1; ++i) A[i + j * n] = v(i - r0) * sigma;
            }
        }
        if (s->outlier_frac > 0.0) {
            const ihs::Index k = static_cast<ihs::Index>(static_cast<double>(n) * s->outlier_frac);
            auto gen = ihs::make_stream(s->data_seed, 14);
            for (ihs::Index r : ihs::sample_without_replacement(n, k, gen))
                for (ihs::Index j = 0; j < d; ++j) A[r + j * n] *= s->outlier_scale;
        }
        ihs::Vector xt(d);
        {
            auto gen = ihs::make_stream(s->data_seed, 12);
            ihs::fill_gaussian(xt, gen, 1.0);
        }
        ihs::Vector noise(n);
        {
            auto gen = ihs::make_stream(s->data_seed, 13);
            ihs::fill_gaussian(noise, gen, s->noise_std);
        }
        for (ihs::Index i = 0; i < n; ++i) {
            double acc = 0.0;
            for (ihs::Index j = 0; j < d; ++j) acc += A[i + j * n] * xt(j);
            b[i] = acc + noise(i);
        }
        if (x_true) put(x_true, xt);
    });
}

// baselines.hpp: method 0 = cg_solve, 1 = pcg_solve_with(SA), 2 = pcg_solve(kind, seed, rho)
int ihs_ref_cg(const double* A, int64_t n, int64_t d, int64_t lda, const double* b, double nu, int32_t method,
               const double* SA, int64_t m, int64_t lds, int32_t kind, uint64_t seed, double rho, double tol,
               int64_t max_iters, const double* x0, ihs_cg_report* rep) {
    return guarded([&] {
        const ihs::ProblemInstance p = ihs::ProblemInstance::make(to_mat(A, n, d, lda), to_vec(b, n), nu);
        ihs::Vector xs;
        if (x0) xs = to_vec(x0, d);
        const ihs::Vector* xp = x0 ? &xs : nullptr;
        auto fill = [&](const ihs::Vector& x, const std::vector<double>& res, ihs::Index its, bool conv,
                        const ihs::CostCounters& cc) {
            put(rep->x, x);
            rep->residuals_size = static_cast<int64_t>(res.size());
            if (rep->residuals)
                for (int64_t i = 0; i < rep->residuals_size && i < rep->residuals_capacity; ++i)
                    rep->residuals[i] = res[static_cast<size_t>(i)];
            rep->iterations = its;
            rep->converged = conv;
            rep->counters = ihs_counters{};
            add_counters(&rep->counters, cc);
        };
        if (method == 0) {
            const ihs::CgResult r = ihs::cg_solve(p, tol, max_iters, xp);
            fill(r.x, r.residuals, r.iterations, r.converged, r.counters);
            rep->m = 0;
            rep->m_capped = 0;
            rep->setup_flops = 0;
        } else {
            const ihs::PcgResult r = method == 1 ? ihs::pcg_solve_with(p, to_mat(SA, m, d, lds), tol, max_iters, {}, xp)
                                                 : ihs::pcg_solve(p, kind_of(kind), seed, rho, tol, max_iters, xp);
            fill(r.x, r.residuals, r.iterations, r.converged, r.counters);
            rep->m = r.m;
            rep->m_capped = r.m_capped;
            rep->setup_flops = r.setup_flops;
        }
    });
}

int ihs_ref_pcg_sketch_size(int64_t n, int64_t d, int32_t kind, double rho, int64_t* m, int32_t* capped) {
    return guarded([&] {
        auto [mm, c] = ihs::pcg_sketch_size(n, d, kind_of(kind), rho);
        *m = mm;
        *capped = c;
    });
}

}  // extern "C"
