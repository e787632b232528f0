// ihs_oracle.cpp — CPU ORACLE (test infrastructure only; see ihs_oracle.hpp).
//
// Restates /root/reference/proj/include/ihs/{rng,sketch,problem,
// sketched_system,tuning,solver}.hpp without Eigen. Built with -O3 -DNDEBUG
// -ffp-contract=off and no -march, like the reference's Release build
// (proj/CMakeLists.txt:8-10), so every double operation of the RNG path
// rounds exactly as in the reference.
#include "ihs_oracle.hpp"

#include <algorithm>
#include <bit>
#include <chrono>
#include <numeric>
#include <span>

namespace ihs_oracle {

// =============================================================== rng.hpp
std::uint64_t splitmix64(std::uint64_t& state) {  // rng.hpp:13-18
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {  // rng.hpp:23-28
    std::uint64_t s = seed + 0x632be59bd9b4e019ULL * (tag + 1);
    std::uint64_t a = splitmix64(s);
    std::uint64_t b = splitmix64(s);
    return a ^ (b << 1);
}

std::mt19937_64 make_stream(std::uint64_t seed, std::uint64_t tag) {  // rng.hpp:30-32
    return std::mt19937_64(derive_seed(seed, tag));
}

void fill_gaussian(double* M, Index rows, Index cols, std::mt19937_64& gen, double stddev) {
    // rng.hpp:35-40: one distribution object per fill, column-major order.
    std::normal_distribution<double> dist(0.0, stddev);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) M[i + j * rows] = dist(gen);
}

std::vector<double> rademacher(Index n, std::mt19937_64& gen) {  // rng.hpp:48-52
    std::vector<double> eps(static_cast<std::size_t>(n));
    for (auto& e : eps) e = (gen() & 1ULL) ? 1.0 : -1.0;
    return eps;
}

std::vector<Index> sample_without_replacement(Index n, Index m, std::mt19937_64& gen) {  // rng.hpp:56-66
    std::vector<Index> pool(static_cast<std::size_t>(n));
    std::iota(pool.begin(), pool.end(), Index{0});
    std::vector<Index> out(static_cast<std::size_t>(m));
    for (Index k = 0; k < m; ++k) {
        std::uniform_int_distribution<Index> pick(k, n - 1);
        std::swap(pool[static_cast<std::size_t>(k)], pool[static_cast<std::size_t>(pick(gen))]);
        out[static_cast<std::size_t>(k)] = pool[static_cast<std::size_t>(k)];
    }
    return out;
}

// =============================================================== sketch.hpp
Index next_pow2(Index n) {  // sketch.hpp:26-28
    return static_cast<Index>(std::bit_ceil(static_cast<std::uint64_t>(n)));
}

void fwht_inplace(double* v, std::size_t n) {  // sketch.hpp:33-49
    if (n == 0 || !std::has_single_bit(n)) throw InvalidInput("fwht_inplace: length must be a power of two");
    for (std::size_t h = 1; h < n; h <<= 1)
        for (std::size_t i = 0; i < n; i += 2 * h)
            for (std::size_t j = i; j < i + h; ++j) {
                const double s = v[j];
                const double t = v[j + h];
                v[j] = s + t;
                v[j + h] = s - t;
            }
    const double scale = 1.0 / std::sqrt(static_cast<double>(n));
    for (std::size_t j = 0; j < n; ++j) v[j] *= scale;
}

// C (m x d) = S (m x n) * A (n x d), all column-major. Stand-in for Eigen's
// GEMM (sketch.hpp:68); blocked for cache, k-order accumulation per entry.
static void gemm_nn(const double* S, Index m, Index n, const double* A, Index lda, Index d, double* C) {
    std::fill(C, C + m * d, 0.0);
    const Index KB = 256, IB = 256;
    for (Index j0 = 0; j0 < d; j0 += 4) {
        const Index jn = std::min<Index>(4, d - j0);
        for (Index k0 = 0; k0 < n; k0 += KB) {
            const Index k1 = std::min(n, k0 + KB);
            for (Index i0 = 0; i0 < m; i0 += IB) {
                const Index i1 = std::min(m, i0 + IB);
                for (Index k = k0; k < k1; ++k) {
                    const double* s = S + k * m;
                    if (jn == 4) {
                        const double a0 = A[k + (j0 + 0) * lda], a1 = A[k + (j0 + 1) * lda];
                        const double a2 = A[k + (j0 + 2) * lda], a3 = A[k + (j0 + 3) * lda];
                        double* c0 = C + (j0 + 0) * m; double* c1 = C + (j0 + 1) * m;
                        double* c2 = C + (j0 + 2) * m; double* c3 = C + (j0 + 3) * m;
                        for (Index i = i0; i < i1; ++i) {
                            const double si = s[i];
                            c0[i] += si * a0; c1[i] += si * a1; c2[i] += si * a2; c3[i] += si * a3;
                        }
                    } else {
                        for (Index jj = 0; jj < jn; ++jj) {
                            const double a = A[k + (j0 + jj) * lda];
                            double* c = C + (j0 + jj) * m;
                            for (Index i = i0; i < i1; ++i) c[i] += s[i] * a;
                        }
                    }
                }
            }
        }
    }
}

Mat gaussian_sketch(const Mat& A, Index m, std::uint64_t seed, CostCounters* counters) {  // sketch.hpp:58-69
    if (m < 1) throw InvalidInput("gaussian_sketch: m must be >= 1");
    const Index n = A.rows;
    auto gen = make_stream(seed, 0);
    Mat S(m, n);
    fill_gaussian(S.a.data(), m, n, gen, 1.0 / std::sqrt(static_cast<double>(m)));
    if (counters)
        counters->sketch += static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(n) *
                            static_cast<std::uint64_t>(A.cols);
    Mat SA(m, A.cols);
    gemm_nn(S.a.data(), m, n, A.a.data(), A.rows, A.cols, SA.a.data());
    return SA;
}

Mat srht_sketch(const Mat& A, Index m, std::uint64_t seed, CostCounters* counters) {  // sketch.hpp:77-108
    if (m < 1) throw InvalidInput("srht_sketch: m must be >= 1");
    const Index n = A.rows;
    const Index d = A.cols;
    const Index n_pad = next_pow2(n);
    if (m > n_pad) throw SketchTooLarge("srht_sketch: m exceeds padded row count");

    auto sign_stream = make_stream(seed, 1);
    auto row_stream = make_stream(seed, 2);
    const std::vector<double> eps = rademacher(n_pad, sign_stream);
    const std::vector<Index> rows = sample_without_replacement(n_pad, m, row_stream);

    Mat B(n_pad, d, 0.0);  // full padded copy, as in the reference (:90)
    for (Index j = 0; j < d; ++j)
        for (Index i = 0; i < n; ++i) B(i, j) = eps[static_cast<std::size_t>(i)] * A(i, j);
    for (Index j = 0; j < d; ++j) fwht_inplace(B.col(j), static_cast<std::size_t>(n_pad));

    const double scale = std::sqrt(static_cast<double>(n_pad) / static_cast<double>(m));
    Mat SA(m, d);
    for (Index j = 0; j < d; ++j)
        for (Index k = 0; k < m; ++k) SA(k, j) = scale * B(rows[static_cast<std::size_t>(k)], j);

    if (counters) {
        const auto np = static_cast<std::uint64_t>(n_pad);
        const auto dd = static_cast<std::uint64_t>(d);
        const auto log2np = static_cast<std::uint64_t>(std::bit_width(static_cast<std::uint64_t>(n_pad)) - 1);
        counters->sketch += dd * np * log2np + static_cast<std::uint64_t>(n) * dd + static_cast<std::uint64_t>(m) * dd;
    }
    return SA;
}

Mat apply_sketch(const Mat& A, SketchKind kind, Index m, std::uint64_t seed, CostCounters* c) {  // :110-117
    if (kind == SketchKind::Gaussian) return gaussian_sketch(A, m, seed, c);
    return srht_sketch(A, m, seed, c);
}

// =============================================================== problem.hpp
Problem::Problem(Mat A_, Vec b_, double nu_, bool underdetermined)
    : A(std::move(A_)), b(std::move(b_)), nu(nu_), underdetermined(underdetermined) {  // :22-33
    if (!(nu > 0.0)) throw InvalidInput("ProblemInstance: nu must be strictly positive");
    if (A.rows < 1 || A.cols < 1) throw InvalidInput("ProblemInstance: empty matrix");
    if (static_cast<Index>(b.size()) != A.rows) throw InvalidInput("ProblemInstance: size of b must match rows of A");
    for (double v : A.a) if (!std::isfinite(v)) throw InvalidInput("ProblemInstance: non-finite input");
    for (double v : b) if (!std::isfinite(v)) throw InvalidInput("ProblemInstance: non-finite input");
    if (!std::isfinite(nu)) throw InvalidInput("ProblemInstance: non-finite input");
    if (!underdetermined && A.rows < A.cols)
        throw InvalidInput("ProblemInstance: overdetermined orientation requires n >= d");
    if (underdetermined && A.cols < A.rows)
        throw InvalidInput("ProblemInstance: underdetermined orientation requires d >= n");
}

static double dot4(const double* a, const double* b, Index n) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    Index i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 += a[i] * b[i]; s1 += a[i + 1] * b[i + 1]; s2 += a[i + 2] * b[i + 2]; s3 += a[i + 3] * b[i + 3];
    }
    for (; i < n; ++i) s0 += a[i] * b[i];
    return (s0 + s1) + (s2 + s3);
}

Vec gradient(const Problem& p, const Vec& x, CostCounters* counters) {  // problem.hpp:59-69
    const Index n = p.A.rows, d = p.A.cols;
    if (static_cast<Index>(x.size()) != d) throw InvalidInput("gradient: dimension mismatch");
    Vec r(static_cast<size_t>(n), 0.0);
    for (Index j = 0; j < d; ++j) {  // r = A x  (column axpy)
        const double xj = x[static_cast<size_t>(j)];
        const double* a = p.A.col(j);
        for (Index i = 0; i < n; ++i) r[static_cast<size_t>(i)] += a[i] * xj;
    }
    for (Index i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= p.b[static_cast<size_t>(i)];
    const double nu2 = p.nu * p.nu;
    Vec g(static_cast<size_t>(d));
    for (Index j = 0; j < d; ++j) g[static_cast<size_t>(j)] = dot4(p.A.col(j), r.data(), n) + nu2 * x[static_cast<size_t>(j)];
    if (counters) {
        const auto nn = static_cast<std::uint64_t>(n), dd = static_cast<std::uint64_t>(d);
        counters->matvec += 2 * nn * dd + nn + 2 * dd;
    }
    return g;
}

// lower Cholesky in place (left-looking); returns false on a non-positive pivot
static bool cholesky_lower(Mat& H) {
    const Index n = H.rows;
    for (Index j = 0; j < n; ++j) {
        double s = H(j, j);
        for (Index k = 0; k < j; ++k) s -= H(j, k) * H(j, k);
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        const double ljj = std::sqrt(s);
        H(j, j) = ljj;
        for (Index i = j + 1; i < n; ++i) {
            double t = H(i, j);
            for (Index k = 0; k < j; ++k) t -= H(i, k) * H(j, k);
            H(i, j) = t / ljj;
        }
        for (Index i = 0; i < j; ++i) H(i, j) = 0.0;
    }
    return true;
}

static void chol_solve(const Mat& L, double* z) {  // L L^T z = rhs, in place
    const Index n = L.rows;
    for (Index i = 0; i < n; ++i) {
        double s = z[i];
        for (Index k = 0; k < i; ++k) s -= L(i, k) * z[k];
        z[i] = s / L(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (Index k = i + 1; k < n; ++k) s -= L(k, i) * z[k];
        z[i] = s / L(i, i);
    }
}

Vec direct_solve(const Problem& p) {
    const Index d = p.A.cols, n = p.A.rows;
    Mat H(d, d);
    for (Index j = 0; j < d; ++j)
        for (Index i = j; i < d; ++i) H(i, j) = H(j, i) = dot4(p.A.col(i), p.A.col(j), n);
    for (Index j = 0; j < d; ++j) H(j, j) += p.nu * p.nu;
    if (!cholesky_lower(H)) throw NumericalBreakdown("direct_solve: Cholesky failed");
    Vec z(static_cast<size_t>(d));
    for (Index j = 0; j < d; ++j) z[static_cast<size_t>(j)] = dot4(p.A.col(j), p.b.data(), n);
    chol_solve(H, z.data());
    return z;
}

double prediction_error(const Problem& p, const Vec& x, const Vec& xs) {  // problem.hpp:104-109
    const Index n = p.A.rows, d = p.A.cols;
    Vec diff(static_cast<size_t>(d));
    for (Index j = 0; j < d; ++j) diff[static_cast<size_t>(j)] = x[static_cast<size_t>(j)] - xs[static_cast<size_t>(j)];
    Vec Ad(static_cast<size_t>(n), 0.0);
    for (Index j = 0; j < d; ++j)
        for (Index i = 0; i < n; ++i) Ad[static_cast<size_t>(i)] += p.A(i, j) * diff[static_cast<size_t>(j)];
    double a = 0, q = 0;
    for (double v : Ad) a += v * v;
    for (double v : diff) q += v * v;
    return 0.5 * a + 0.5 * p.nu * p.nu * q;
}

// =============================================================== sketched_system.hpp
SketchedSystem::SketchedSystem(Mat SA, double nu)  // :69-84
    : SA_(std::move(SA)), nu_(nu), kind_(SA_.rows < SA_.cols ? FactorKind::WoodburyInner : FactorKind::DirectGram) {
    const double nu2 = nu_ * nu_;
    const Index m = SA_.rows, d = SA_.cols;
    // Both products are full dense GEMMs like Eigen's `SA_ * SA_.transpose()` / `SA_.transpose() * SA_` (the
    // counted m^2 d / d^2 m multiply-adds), formed by the blocked axpy-form gemm_nn over a transposed copy so
    // every entry accumulates its inner index in ascending order.
    Mat SAT(d, m);
    for (Index j = 0; j < d; ++j)
        for (Index i = 0; i < m; ++i) SAT(j, i) = SA_(i, j);
    if (kind_ == FactorKind::WoodburyInner) {  // inner = SA SA^T + nu^2 I_m
        L_ = Mat(m, m);
        gemm_nn(SA_.a.data(), m, d, SAT.a.data(), d, m, L_.a.data());
        for (Index j = 0; j < m; ++j) L_(j, j) += nu2;
    } else {  // gram = SA^T SA + nu^2 I_d
        L_ = Mat(d, d);
        gemm_nn(SAT.a.data(), d, m, SA_.a.data(), m, d, L_.a.data());
        for (Index j = 0; j < d; ++j) L_(j, j) += nu2;
    }
    if (!cholesky_lower(L_)) throw NumericalBreakdown("SketchedSystem: Cholesky factorization failed");
}

SketchedSystem SketchedSystem::factorize(Mat SA, double nu, CostCounters* counters) {  // :25-31
    if (!(nu > 0.0)) throw InvalidInput("SketchedSystem: nu must be positive");
    for (double v : SA.a) if (!std::isfinite(v)) throw InvalidInput("SketchedSystem: non-finite sketched matrix");
    SketchedSystem sys(std::move(SA), nu);
    if (counters) counters->factor += sys.factor_flops();
    return sys;
}

Vec SketchedSystem::solve(const Vec& g, CostCounters* counters) const {  // :40-49
    const Index m = SA_.rows, d = SA_.cols;
    if (static_cast<Index>(g.size()) != d) throw InvalidInput("SketchedSystem::solve: dimension mismatch");
    if (counters) counters->solve += flops_per_solve();
    if (kind_ == FactorKind::WoodburyInner) {
        Vec u(static_cast<size_t>(m), 0.0);
        for (Index k = 0; k < d; ++k)
            for (Index i = 0; i < m; ++i) u[static_cast<size_t>(i)] += SA_(i, k) * g[static_cast<size_t>(k)];
        chol_solve(L_, u.data());
        Vec z(static_cast<size_t>(d));
        const double nu2 = nu_ * nu_;
        for (Index k = 0; k < d; ++k) z[static_cast<size_t>(k)] = (g[static_cast<size_t>(k)] - dot4(SA_.col(k), u.data(), m)) / nu2;
        return z;
    }
    Vec z = g;
    chol_solve(L_, z.data());
    return z;
}

std::uint64_t SketchedSystem::factor_flops() const {  // :52-57
    const auto mm = static_cast<std::uint64_t>(m()), dd = static_cast<std::uint64_t>(d());
    if (kind_ == FactorKind::WoodburyInner) return mm * mm * dd + mm * mm * mm / 3;
    return dd * dd * mm + dd * dd * dd / 3;
}
std::uint64_t SketchedSystem::flops_per_solve() const {  // :61-66
    const auto mm = static_cast<std::uint64_t>(m()), dd = static_cast<std::uint64_t>(d());
    if (kind_ == FactorKind::WoodburyInner) return 2 * mm * dd + mm * mm + 2 * dd;
    return dd * dd + dd;
}

double newton_decrement(const Vec& g, const Vec& gt) {  // :95-101
    if (g.size() != gt.size()) throw InvalidInput("newton_decrement: dimension mismatch");
    double dot = 0, sq = 0;
    for (size_t i = 0; i < g.size(); ++i) { dot += g[i] * gt[i]; sq += g[i] * g[i]; }
    const double r = 0.5 * dot;
    if (r < -1e-12 * (1.0 + sq)) throw NumericalBreakdown("newton_decrement: negative decrement");
    return r < 0.0 ? 0.0 : r;
}

// =============================================================== tuning.hpp
TuningParams rates_from_bounds(double lam, double Lam) {  // :25-38
    if (!(lam > 0.0) || !(lam <= Lam)) throw InvalidInput("rates_from_bounds: need 0 < lam <= Lam");
    TuningParams tp;
    tp.lam = lam;
    tp.Lam = Lam;
    tp.mu_gd = 2.0 / (1.0 / lam + 1.0 / Lam);
    const double r = (Lam - lam) / (Lam + lam);
    tp.c_gd = r * r;
    const double sl = std::sqrt(lam), sL = std::sqrt(Lam);
    tp.mu_p = 4.0 / ((1.0 / sl + 1.0 / sL) * (1.0 / sl + 1.0 / sL));
    const double q = (sL - sl) / (sL + sl);
    tp.beta_p = tp.c_p = q * q;
    return tp;
}

std::pair<double, double> gaussian_targets(double rho, double eta, bool enforce_validity) {  // :47-56
    if (!(rho > 0.0) || !(eta > 0.0)) throw InvalidInput("gaussian_targets: rho, eta must be positive");
    if (enforce_validity && (rho > 0.18 || eta > 0.01))
        throw OutOfValidityRange("gaussian_targets: proven region is rho <= 0.18, eta <= 0.01");
    const double ce = (1.0 + 3.0 * std::sqrt(eta)) * (1.0 + 3.0 * std::sqrt(eta));
    const double s = std::sqrt(ce * rho);
    if (s >= 1.0) throw OutOfValidityRange("gaussian_targets: c_eta * rho must be < 1");
    return {(1.0 - s) * (1.0 - s), (1.0 + s) * (1.0 + s)};
}

std::pair<double, double> srht_targets(double rho) {  // :59-63
    if (!(rho > 0.0 && rho < 1.0)) throw InvalidInput("srht_targets: rho must be in (0,1)");
    const double s = std::sqrt(rho);
    return {1.0 - s, 1.0 + s};
}

// =============================================================== solver.hpp
namespace {
struct Candidate { Vec x, g, gt; double r; };
}

SolveReport adaptive_solve_core(const Mat& A, double nu, const GradFn& grad, const SolverConfig& cfg) {  // :106-232
    if (!(cfg.eps > 0.0 && cfg.eps < 1.0)) throw InvalidInput("adaptive_solve: eps must be in (0,1)");
    if (cfg.m_initial < 1) throw InvalidInput("adaptive_solve: m_initial must be >= 1");
    if (cfg.max_iters < 1) throw InvalidInput("adaptive_solve: max_iters must be >= 1");

    const auto t_start = std::chrono::steady_clock::now();
    const Index dim = A.cols, n_rows = A.rows;

    TuningParams tp;
    if (cfg.tuning_override) tp = *cfg.tuning_override;
    else if (cfg.sketch_kind == SketchKind::Gaussian) {
        auto [lam, Lam] = gaussian_targets(cfg.rho, cfg.eta, cfg.enforce_validity);
        tp = rates_from_bounds(lam, Lam);
    } else {
        auto [lam, Lam] = srht_targets(cfg.rho);
        tp = rates_from_bounds(lam, Lam);
    }
    Index cap = cfg.sketch_kind == SketchKind::SRHT ? next_pow2(n_rows) : n_rows;  // :128-130
    if (cfg.max_sketch) cap = std::min(cap, *cfg.max_sketch);
    cap = std::max(cap, cfg.m_initial);

    SolveReport rep;
    rep.tuning = tp;
    rep.recompute_r_after_resketch = cfg.recompute_r_after_resketch;
    Index m = cfg.m_initial, K = 0;

    auto core_sketch = [&](Index mm, std::uint64_t sub_seed) -> Mat {  // :100-104
        if (cfg.sketch_override) return cfg.sketch_override(A, mm, sub_seed);
        return apply_sketch(A, cfg.sketch_kind, mm, sub_seed, &rep.counters);
    };
    SketchedSystem sys = SketchedSystem::factorize(core_sketch(m, derive_seed(cfg.seed, 0)), nu, &rep.counters);

    Vec x_cur = cfg.warm_start ? *cfg.warm_start : Vec(static_cast<size_t>(dim), 0.0);
    if (static_cast<Index>(x_cur.size()) != dim) throw InvalidInput("adaptive_solve: warm start has wrong dimension");
    Vec x_prev = x_cur;

    Vec g = grad(x_cur, &rep.counters);
    Vec gt = sys.solve(g, &rep.counters);
    double r = newton_decrement(g, gt);
    const double r1 = r;
    rep.r1 = r1;
    if (cfg.record_iterates) rep.iterates.push_back(x_cur);

    Index t = 1;
    bool converged = !(r > cfg.eps * r1) || r1 == 0.0;
    bool checks_enabled = true;

    auto evaluate = [&](Vec xc) -> Candidate {  // :161-166
        Vec gc = grad(xc, &rep.counters);
        Vec gtc = sys.solve(gc, &rep.counters);
        const double rc = newton_decrement(gc, gtc);
        return {std::move(xc), std::move(gc), std::move(gtc), rc};
    };
    auto accept = [&](Candidate&& c, StepKind kind) {  // :167-178
        const double r_prev = r;
        x_prev = std::move(x_cur);
        x_cur = std::move(c.x);
        g = std::move(c.g);
        gt = std::move(c.gt);
        r = c.r;
        ++t;
        rep.log.push_back({t, m, r, r_prev, kind});
        if (cfg.record_iterates) rep.iterates.push_back(x_cur);
        converged = r <= cfg.eps * r1;
    };

    while (!converged && t < cfg.max_iters) {  // :180-221
        if (checks_enabled && cfg.mode == SolveMode::PolyakThenGradient) {
            Vec xc(static_cast<size_t>(dim));
            // x_cur - mu_p * gt + beta_p * (x_cur - x_prev), evaluated as Eigen does
            // elementwise: (x - mu*gt) + beta*(x - xp)
            for (Index i = 0; i < dim; ++i) {
                const size_t u = static_cast<size_t>(i);
                xc[u] = (x_cur[u] - tp.mu_p * gt[u]) + tp.beta_p * (x_cur[u] - x_prev[u]);
            }
            Candidate cand = evaluate(std::move(xc));
            const double ratio = std::pow(cand.r / r1, 1.0 / static_cast<double>(t));
            if (ratio <= tp.c_p || cand.r <= cfg.eps * r1) {
                accept(std::move(cand), StepKind::Polyak);
                continue;
            }
        }
        Vec xg(static_cast<size_t>(dim));
        for (Index i = 0; i < dim; ++i) xg[static_cast<size_t>(i)] = x_cur[static_cast<size_t>(i)] - tp.mu_gd * gt[static_cast<size_t>(i)];
        Candidate cand = evaluate(std::move(xg));
        const bool pass = checks_enabled ? (cand.r <= tp.c_gd * r || cand.r <= cfg.eps * r1) : cand.r <= r;
        if (pass) {
            accept(std::move(cand), StepKind::Gradient);
            continue;
        }
        if (!checks_enabled) break;
        if (2 * m > cap) {
            rep.sketch_exhausted = true;
            checks_enabled = false;
            if (cand.r <= r) {
                accept(std::move(cand), StepKind::Gradient);
                continue;
            }
            break;
        }
        m *= 2;
        ++K;
        sys = SketchedSystem::factorize(core_sketch(m, derive_seed(cfg.seed, static_cast<std::uint64_t>(K))), nu, &rep.counters);
        gt = sys.solve(g, &rep.counters);
        const double r_old = r;
        if (cfg.recompute_r_after_resketch) {
            r = newton_decrement(g, gt);
            converged = r <= cfg.eps * r1;
        }
        rep.log.push_back({t, m, r, r_old, StepKind::Resketch});
    }
    rep.x = std::move(x_cur);
    rep.iterations = t;
    rep.rejections = K;
    rep.final_m = m;
    rep.r_final = r;
    rep.converged = converged;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return rep;
}

SolveReport adaptive_solve(const Problem& p, const SolverConfig& cfg) {  // :242-250
    return adaptive_solve_core(p.A, p.nu, [&p](const Vec& x, CostCounters* c) { return gradient(p, x, c); }, cfg);
}

// dual.hpp:13-33: the dual ridge problem in A^T, gradient A(A^T z) - b + nu^2 z, x = A^T z
SolveReport solve_underdetermined(const Problem& p, const SolverConfig& cfg) {
    if (p.A.rows > p.A.cols) throw InvalidInput("solve_underdetermined: expects an underdetermined instance");
    // (an n == d instance is both; the caller constructs it with the underdetermined orientation)
    const Index n = p.A.rows, d = p.A.cols;
    Mat At(d, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < d; ++i) At(i, j) = p.A(j, i);
    const double nu2 = p.nu * p.nu;
    GradFn grad = [&p, n, d, nu2](const Vec& z, CostCounters* c) -> Vec {
        Vec u(static_cast<size_t>(d), 0.0);  // u = A^T z
        for (Index i = 0; i < d; ++i) {
            double s = 0.0;
            for (Index r = 0; r < n; ++r) s += p.A(r, i) * z[static_cast<size_t>(r)];
            u[static_cast<size_t>(i)] = s;
        }
        Vec g(static_cast<size_t>(n), 0.0);  // g = A u - b + nu^2 z
        for (Index i = 0; i < d; ++i) {
            const double ui = u[static_cast<size_t>(i)];
            for (Index r = 0; r < n; ++r) g[static_cast<size_t>(r)] += p.A(r, i) * ui;
        }
        for (Index r = 0; r < n; ++r) {
            const size_t q = static_cast<size_t>(r);
            g[q] = (g[q] - p.b[q]) + nu2 * z[q];
        }
        if (c) c->matvec += 2 * static_cast<std::uint64_t>(n) * static_cast<std::uint64_t>(d) +
                            static_cast<std::uint64_t>(d) + 2 * static_cast<std::uint64_t>(n);
        return g;
    };
    SolveReport rep = adaptive_solve_core(At, p.nu, grad, cfg);
    rep.dual_final = rep.x;
    Vec x(static_cast<size_t>(d), 0.0);  // x = A^T z
    for (Index i = 0; i < d; ++i) {
        double s = 0.0;
        for (Index r = 0; r < n; ++r) s += p.A(r, i) * rep.dual_final[static_cast<size_t>(r)];
        x[static_cast<size_t>(i)] = s;
    }
    rep.x = std::move(x);
    return rep;
}

std::vector<Vec> fixed_sketch_ihs(const Problem& p, const SketchedSystem& sys, const TuningParams& tp, Index T,
                                  FixedMode mode, const Vec* x_start) {  // :258-276
    const double mu = mode == FixedMode::Gradient ? tp.mu_gd : tp.mu_p;
    const double beta = mode == FixedMode::Gradient ? 0.0 : tp.beta_p;
    const size_t d = static_cast<size_t>(p.A.cols);
    Vec x = x_start ? *x_start : Vec(d, 0.0);
    Vec x_prev = x;
    std::vector<Vec> its;
    its.push_back(x);
    for (Index t = 0; t < T; ++t) {
        Vec step = sys.solve(gradient(p, x));
        Vec xn(d);
        for (size_t i = 0; i < d; ++i) xn[i] = (x[i] - mu * step[i]) + beta * (x[i] - x_prev[i]);
        x_prev = std::move(x);
        x = std::move(xn);
        its.push_back(x);
    }
    return its;
}

// =============================================================== baselines.hpp
namespace {
double sq_norm(const Vec& v) {
    double s = 0;
    for (double x : v) s += x * x;
    return s;
}
double dotv(const Vec& a, const Vec& b) {
    double s = 0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
// H v = A^T (A v) + nu^2 v (baselines.hpp:50-53, :115-118), counted as 2nd + 2d
Vec apply_h(const Problem& p, const Vec& v, CostCounters& c) {
    const Index n = p.A.rows, d = p.A.cols;
    Vec r(static_cast<size_t>(n), 0.0);
    for (Index j = 0; j < d; ++j) {
        const double vj = v[static_cast<size_t>(j)];
        const double* a = p.A.col(j);
        for (Index i = 0; i < n; ++i) r[static_cast<size_t>(i)] += a[i] * vj;
    }
    const double nu2 = p.nu * p.nu;
    Vec h(static_cast<size_t>(d));
    for (Index j = 0; j < d; ++j) h[static_cast<size_t>(j)] = dot4(p.A.col(j), r.data(), n) + nu2 * v[static_cast<size_t>(j)];
    c.matvec += 2 * static_cast<std::uint64_t>(n) * static_cast<std::uint64_t>(d) + 2 * static_cast<std::uint64_t>(d);
    return h;
}
Vec atb_of(const Problem& p) {
    Vec z(static_cast<size_t>(p.A.cols));
    for (Index j = 0; j < p.A.cols; ++j) z[static_cast<size_t>(j)] = dot4(p.A.col(j), p.b.data(), p.A.rows);
    return z;
}
// r = A^T b - H x; x = x0 or 0 (baselines.hpp:55-58, :126-129)
Vec cg_start(const Problem& p, CgResult& res, const Vec* x0, const Vec& atb) {
    const size_t d = static_cast<size_t>(p.A.cols);
    if (x0 && x0->size() != d) throw InvalidInput("cg_solve: dimension mismatch");
    res.x = x0 ? *x0 : Vec(d, 0.0);
    Vec hx = apply_h(p, res.x, res.counters);
    Vec r(d);
    for (size_t i = 0; i < d; ++i) r[i] = atb[i] - hx[i];
    res.residuals.push_back(std::sqrt(sq_norm(r)));
    return r;
}
}  // namespace

CgResult cg_solve(const Problem& p, double tol, Index max_iters, const Vec* x0) {  // baselines.hpp:40-92
    if (p.underdetermined) throw InvalidInput("cg_solve: expects an overdetermined instance");
    const size_t d = static_cast<size_t>(p.A.cols);
    CgResult res;
    const Vec atb = atb_of(p);
    const double target = tol * std::sqrt(sq_norm(atb));
    Vec r = cg_start(p, res, x0, atb);
    if (res.residuals.back() <= target) {
        res.converged = true;
        return res;
    }
    Vec pdir = r;
    double rr = sq_norm(r);
    for (Index k = 0; k < max_iters; ++k) {
        Vec hp = apply_h(p, pdir, res.counters);
        const double alpha = rr / dotv(pdir, hp);
        for (size_t i = 0; i < d; ++i) res.x[i] += alpha * pdir[i];
        for (size_t i = 0; i < d; ++i) r[i] -= alpha * hp[i];
        ++res.iterations;
        const double rr_new = sq_norm(r);
        res.residuals.push_back(std::sqrt(rr_new));
        if (res.residuals.back() <= target) {
            res.converged = true;
            break;
        }
        const double beta = rr_new / rr;
        for (size_t i = 0; i < d; ++i) pdir[i] = r[i] + beta * pdir[i];
        rr = rr_new;
    }
    return res;
}

CgResult pcg_solve_with(const Problem& p, const Mat& SA, double tol, Index max_iters, CgResult res,
                        const Vec* x0) {  // baselines.hpp:98-165
    if (p.underdetermined) throw InvalidInput("pcg_solve: expects an overdetermined instance");
    const Index d = p.A.cols, m = SA.rows;
    if (SA.cols != d) throw InvalidInput("pcg_solve: dimension mismatch");
    const auto dd = static_cast<std::uint64_t>(d), mm = static_cast<std::uint64_t>(m);
    res.m = m;
    // gram = SA^T SA + nu^2 I_d, lower Cholesky; applied by two triangular substitutions
    Mat L(d, d);
    for (Index j = 0; j < d; ++j)
        for (Index i = j; i < d; ++i) L(i, j) = L(j, i) = dot4(SA.col(i), SA.col(j), m);
    for (Index j = 0; j < d; ++j) L(j, j) += p.nu * p.nu;
    if (!cholesky_lower(L)) throw NumericalBreakdown("pcg_solve: preconditioner factorization failed");
    res.setup_flops += dd * dd * mm + dd * dd * dd / 3;
    res.counters.factor += dd * dd * mm + dd * dd * dd / 3;
    auto apply_minv = [&](const Vec& v) {
        res.counters.solve += 2 * dd * dd;
        Vec z = v;
        chol_solve(L, z.data());
        return z;
    };
    const size_t du = static_cast<size_t>(d);
    const Vec atb = atb_of(p);
    const double target = tol * std::sqrt(sq_norm(atb));
    Vec r = cg_start(p, res, x0, atb);
    if (res.residuals.back() <= target) {
        res.converged = true;
        return res;
    }
    Vec z = apply_minv(r);
    Vec pdir = z;
    double rz = dotv(r, z);
    for (Index k = 0; k < max_iters; ++k) {
        Vec hp = apply_h(p, pdir, res.counters);
        const double alpha = rz / dotv(pdir, hp);
        for (size_t i = 0; i < du; ++i) res.x[i] += alpha * pdir[i];
        for (size_t i = 0; i < du; ++i) r[i] -= alpha * hp[i];
        ++res.iterations;
        res.residuals.push_back(std::sqrt(sq_norm(r)));
        if (res.residuals.back() <= target) {
            res.converged = true;
            break;
        }
        z = apply_minv(r);
        const double rz_new = dotv(r, z);
        const double beta = rz_new / rz;
        for (size_t i = 0; i < du; ++i) pdir[i] = z[i] + beta * pdir[i];
        rz = rz_new;
    }
    return res;
}

std::pair<Index, bool> pcg_sketch_size(Index n, Index d, SketchKind kind, double rho) {  // baselines.hpp:170-187
    if (!(rho > 0.0 && rho < 1.0)) throw InvalidInput("pcg_sketch_size: rho must be in (0,1)");
    const double m_raw = kind == SketchKind::Gaussian
                             ? static_cast<double>(d) / rho
                             : static_cast<double>(d) * std::log(static_cast<double>(d)) / rho;
    Index m = std::max<Index>(static_cast<Index>(std::ceil(m_raw)), 1);
    bool capped = false;
    if (kind == SketchKind::SRHT) {
        const Index n_pad = next_pow2(n);
        if (m > n_pad) {
            m = n_pad;
            capped = true;
        }
    }
    return {m, capped};
}

CgResult pcg_solve(const Problem& p, SketchKind kind, std::uint64_t seed, double rho, double tol, Index max_iters,
                   const Vec* x0) {  // baselines.hpp:190-200
    auto [m, capped] = pcg_sketch_size(p.A.rows, p.A.cols, kind, rho);
    CgResult res;
    res.m_capped = capped;
    Mat SA = apply_sketch(p.A, kind, m, seed, &res.counters);
    res.setup_flops += res.counters.sketch;
    return pcg_solve_with(p, SA, tol, max_iters, std::move(res), x0);
}

// =============================================================== synthetic data
void synth_generate(const SynthSpec& s, Mat& A, Vec& b, Vec& x_true) {
    const Index n = s.n, d = s.d;
    const Index n_pad = next_pow2(n);
    const Index B = std::min<Index>(Index{1} << 16, n_pad);
    const Index nb = (n + B - 1) / B;
    A = Mat(n, d);
    for (Index j = 0; j < d; ++j) {
        const double sigma = s.spectrum == 0 ? std::pow(s.decay, static_cast<double>(j + 1))
                                             : 1.0 / static_cast<double>(j + 1);
        for (Index q = 0; q < nb; ++q) {
            auto gen = make_stream(s.data_seed, static_cast<std::uint64_t>(1000 + j * nb + q));
            const Index r0 = q * B, r1 = std::min(n, r0 + B);
            fill_gaussian(A.col(j) + r0, r1 - r0, 1, gen, 1.0);
            for (Index i = r0; i < r1; ++i) A(i, j) *= sigma;
        }
    }
    if (s.outlier_frac > 0.0) {
        const Index k = static_cast<Index>(static_cast<double>(n) * s.outlier_frac);
        auto gen = make_stream(s.data_seed, 14);
        auto rows = sample_without_replacement(n, k, gen);
        for (Index r : rows)
            for (Index j = 0; j < d; ++j) A(r, j) *= s.outlier_scale;
    }
    x_true.assign(static_cast<size_t>(d), 0.0);
    {
        auto gen = make_stream(s.data_seed, 12);
        fill_gaussian(x_true.data(), d, 1, gen, 1.0);
    }
    Vec noise(static_cast<size_t>(n));
    {
        auto gen = make_stream(s.data_seed, 13);
        fill_gaussian(noise.data(), n, 1, gen, s.noise_std);
    }
    b.assign(static_cast<size_t>(n), 0.0);
    for (Index i = 0; i < n; ++i) {
        double acc = 0.0;
        for (Index j = 0; j < d; ++j) acc += A(i, j) * x_true[static_cast<size_t>(j)];
        b[static_cast<size_t>(i)] = acc + noise[static_cast<size_t>(i)];
    }
}

}  // namespace ihs_oracle
