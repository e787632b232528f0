// Reference unit tests re-targeted at the C++ drop-in (include/ihs_b200.hpp):
// the hot-path cases of proj/tests/test_sketch.cpp, test_sketched_system.cpp,
// test_problem.cpp, test_tuning.cpp and test_solver.cpp, written against the
// same API names. Prints one line per check; exit status = failures.
#include "ihs_b200.hpp"

#include <cmath>
#include <cstdio>
#include <random>

using namespace ihs;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (cond) ++g_pass;                                                \
        else { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
    do {                                                                   \
        bool ok = false;                                                   \
        try { (void)(expr); } catch (const T&) { ok = true; } catch (...) {} \
        CHECK(ok && #T);                                                   \
    } while (0)

static Matrix random_matrix(Index r, Index c, std::mt19937_64& gen) {  // support.hpp:34-40
    std::normal_distribution<double> dist;
    Matrix M(r, c);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) M(i, j) = dist(gen);
    return M;
}
static Vector random_vector(Index n, std::mt19937_64& gen) {
    std::normal_distribution<double> dist;
    Vector v(n);
    for (Index i = 0; i < n; ++i) v(i) = dist(gen);
    return v;
}

// x = A^T (A A^T + nu^2 I)^{-1} b (support.hpp ridge_kernel_form), Gauss-Jordan on the small n x n system
static Vector ridge_kernel_form(const Matrix& A, const Vector& b, double nu) {
    const Index n = A.rows(), d = A.cols();
    std::vector<double> K(static_cast<size_t>(n * n)), rhs(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) {
        for (Index j = 0; j < n; ++j) {
            double s = 0.0;
            for (Index k = 0; k < d; ++k) s += A(i, k) * A(j, k);
            K[static_cast<size_t>(i + j * n)] = s + (i == j ? nu * nu : 0.0);
        }
        rhs[static_cast<size_t>(i)] = b(i);
    }
    for (Index c = 0; c < n; ++c) {
        const double piv = K[static_cast<size_t>(c + c * n)];
        for (Index j = 0; j < n; ++j) K[static_cast<size_t>(c + j * n)] /= piv;
        rhs[static_cast<size_t>(c)] /= piv;
        for (Index r = 0; r < n; ++r) {
            if (r == c) continue;
            const double f = K[static_cast<size_t>(r + c * n)];
            for (Index j = 0; j < n; ++j) K[static_cast<size_t>(r + j * n)] -= f * K[static_cast<size_t>(c + j * n)];
            rhs[static_cast<size_t>(r)] -= f * rhs[static_cast<size_t>(c)];
        }
    }
    Vector x(d);
    for (Index k = 0; k < d; ++k) {
        double s = 0.0;
        for (Index i = 0; i < n; ++i) s += A(i, k) * rhs[static_cast<size_t>(i)];
        x(k) = s;
    }
    return x;
}

int main() {
    // ---- test_sketch.cpp
    {
        Vector v{1.0, 0.0, 0.0, 0.0};
        fwht_inplace(v);
        for (Index i = 0; i < 4; ++i) CHECK(std::abs(v(i) - 0.5) <= 1e-15);
        std::mt19937_64 gen(2);
        Vector x = random_vector(64, gen), w = x;
        fwht_inplace(w);
        CHECK(std::abs(w.norm() - x.norm()) <= 1e-12 * x.norm());
        fwht_inplace(w);
        double mx = 0;
        for (Index i = 0; i < 64; ++i) mx = std::max(mx, std::abs(w(i) - x(i)));
        CHECK(mx <= 1e-12);
        Vector twelve(12);
        CHECK_THROWS_AS(fwht_inplace(twelve), InvalidInput);
    }
    {
        CHECK(gaussian_sketch(Matrix::Zero(10, 3), 4, 7).norm() == 0.0);
        std::mt19937_64 gen(4);
        Matrix A = random_matrix(12, 5, gen);
        CHECK((gaussian_sketch(A, 6, 123) - gaussian_sketch(A, 6, 123)).norm() == 0.0);
        CHECK((gaussian_sketch(A, 6, 123) - gaussian_sketch(A, 6, 124)).norm() > 0.0);
        CostCounters c;
        gaussian_sketch(Matrix::Zero(10, 3), 4, 7, &c);
        CHECK(c.sketch == 4u * 10u * 3u);
    }
    {
        CHECK(srht_sketch(Matrix::Zero(10, 3), 4, 7).norm() == 0.0);
        Matrix S = srht_sketch(Matrix::Identity(16, 16), 16, 3);
        CHECK((S.transpose() * S - Matrix::Identity(16, 16)).norm() <= 1e-10);
        CHECK_THROWS_AS(srht_sketch(Matrix::Zero(12, 2), 17, 0), SketchTooLarge);
        std::mt19937_64 gen(6);
        Matrix A = random_matrix(20, 3, gen);
        CHECK((srht_sketch(A, 8, 42) - srht_sketch(A, 8, 42)).norm() == 0.0);
        CHECK((srht_sketch(A, 8, 42) - srht_sketch(A, 8, 43)).norm() > 0.0);
        CostCounters c16, c256;
        srht_sketch(Matrix::Zero(1000, 2), 16, 0, &c16);
        srht_sketch(Matrix::Zero(1000, 2), 256, 0, &c256);
        const std::uint64_t fw = 2ull * 1024ull * 10ull;
        CHECK(c16.sketch == fw + 2ull * 1000ull + 2ull * 16ull);
        CHECK(c256.sketch == fw + 2ull * 1000ull + 2ull * 256ull);
        CHECK(next_pow2(1000) == 1024 && next_pow2(1) == 1);
    }
    // ---- test_sketched_system.cpp
    {
        auto sys = SketchedSystem::factorize(Matrix::Zero(3, 4), 2.0);
        Vector g{4.0, -8.0, 0.0, 2.0};
        Vector z = sys.solve(g);
        for (Index i = 0; i < 4; ++i) CHECK(std::abs(z(i) - g(i) / 4.0) <= 1e-14);
        Matrix SA(1, 3);
        SA(0, 0) = 1.0;
        auto s2 = SketchedSystem::factorize(SA, 1.0);
        CHECK(s2.kind() == FactorKind::WoodburyInner);
        Vector z2 = s2.solve(Vector::Ones(3));
        CHECK(std::abs(z2(0) - 0.5) <= 1e-14 && std::abs(z2(1) - 1.0) <= 1e-14 && std::abs(z2(2) - 1.0) <= 1e-14);
        std::mt19937_64 gen(15);
        CHECK(SketchedSystem::factorize(random_matrix(5, 5, gen), 1.0).kind() == FactorKind::DirectGram);
        CHECK(SketchedSystem::factorize(random_matrix(4, 5, gen), 1.0).kind() == FactorKind::WoodburyInner);
        Matrix bad = Matrix::Zero(2, 3);
        bad(1, 1) = INFINITY;
        CHECK_THROWS_AS(SketchedSystem::factorize(bad, 1.0), InvalidInput);
        CHECK_THROWS_AS(SketchedSystem::factorize(Matrix::Zero(2, 3), 0.0), InvalidInput);
        CHECK_THROWS_AS(newton_decrement(Vector::Ones(3), (-1.0) * Vector::Ones(3)), NumericalBreakdown);
        std::mt19937_64 g23(23);
        CostCounters c;
        auto s3 = SketchedSystem::factorize(random_matrix(8, 32, g23), 1.0, &c);
        CHECK(c.factor == 8u * 8u * 32u + 8u * 8u * 8u / 3u);
        s3.solve(Vector::Zero(32), &c);
        CHECK(c.solve == 2u * 8u * 32u + 8u * 8u + 2u * 32u);
    }
    // ---- test_problem.cpp
    {
        Vector b{1.0, 2.0};
        ProblemInstance p(Matrix::Identity(2, 2), b, 1.0, Orientation::Overdetermined);
        Vector g = gradient(p, Vector{1.0, 1.0});
        CHECK(std::abs(g(0) - 1.0) <= 1e-15 && std::abs(g(1)) <= 1e-15);
        CostCounters c;
        gradient(p, Vector::Zero(2), &c);
        CHECK(c.matvec == 2 * 2 * 2 + 2 + 2 * 2);
        CHECK_THROWS_AS(ProblemInstance(Matrix::Identity(3, 2), Vector::Ones(3), 0.0, Orientation::Overdetermined), InvalidInput);
        CHECK_THROWS_AS(ProblemInstance(Matrix::Identity(3, 2), Vector::Ones(2), 1.0, Orientation::Overdetermined), InvalidInput);
    }
    // ---- test_tuning.cpp
    {
        TuningParams tp = rates_from_bounds(0.5, 2.0);
        CHECK(std::abs(tp.mu_gd - 0.8) <= 1e-14 && std::abs(tp.c_gd - 0.36) <= 1e-14);
        auto [l, L] = srht_targets(0.04);
        CHECK(std::abs(l - 0.8) <= 1e-14 && std::abs(L - 1.2) <= 1e-14);
        CHECK_THROWS_AS(gaussian_targets(0.19, 0.01), OutOfValidityRange);
        CHECK_THROWS_AS(rates_from_bounds(0.0, 1.0), InvalidInput);
    }
    // ---- test_solver.cpp
    {
        std::mt19937_64 gen(52);
        ProblemInstance p(random_matrix(10, 3, gen), Vector::Zero(10), 1.0, Orientation::Overdetermined);
        SolverConfig cfg;
        SolveReport rep = adaptive_solve(p, cfg);
        CHECK(rep.converged && rep.iterations == 1 && rep.r1 == 0.0 && rep.x.norm() == 0.0);
    }
    {
        std::mt19937_64 gen(53);
        ProblemInstance p(random_matrix(6, 3, gen), random_vector(6, gen), 1.0, Orientation::Overdetermined);
        SolverConfig cfg;
        cfg.eps = 0.0;
        CHECK_THROWS_AS(adaptive_solve(p, cfg), InvalidInput);
        cfg = SolverConfig{};
        cfg.rho = 0.5;
        CHECK_THROWS_AS(adaptive_solve(p, cfg), OutOfValidityRange);
        cfg.enforce_validity = false;
        adaptive_solve(p, cfg);
        ++g_pass;
    }
    {
        std::mt19937_64 gen(9);
        Matrix A = random_matrix(256, 8, gen);
        Vector b = random_vector(256, gen);
        ProblemInstance p(A, b, 0.2, Orientation::Overdetermined);
        for (SketchKind k : {SketchKind::Gaussian, SketchKind::SRHT}) {
            SolverConfig cfg;
            cfg.sketch_kind = k;
            cfg.rho = 0.15;
            cfg.seed = 7;
            cfg.record_iterates = true;
            SolveReport a = adaptive_solve(p, cfg), c = adaptive_solve(p, cfg);
            CHECK(a.converged && a.iterations == c.iterations && a.rejections == c.rejections);
            CHECK((a.x - c.x).norm() == 0.0);
            CHECK(a.final_m == cfg.m_initial * (Index{1} << a.rejections));
            CHECK(static_cast<Index>(a.iterates.size()) == a.iterations);
            Index accepted = 0, resk = 0;
            for (const auto& e : a.log) (e.branch == StepKind::Resketch ? resk : accepted)++;
            CHECK(accepted == a.iterations - 1 && resk == a.rejections);
        }
        // sketch_override hook: an exact sketch (SA = A itself) converges immediately
        SolverConfig cfg;
        cfg.m_initial = 256;
        cfg.tuning_override = rates_from_bounds(1.0, 1.0);
        cfg.sketch_override = [](const Matrix& M, Index, std::uint64_t) { return M; };
        SolveReport r = adaptive_solve(p, cfg);
        CHECK(r.converged && r.rejections == 0 && r.iterations == 2 && r.counters.sketch == 0);
    }
    // ---- test_dual.cpp (solve_underdetermined, dual.hpp:13-33)
    {
        Matrix A(1, 2);
        A(0, 0) = 1.0;
        A(0, 1) = 1.0;
        ProblemInstance p(A, Vector{2.0}, 1.0, Orientation::Underdetermined);
        SolverConfig cfg;
        cfg.eps = 1e-14;
        SolveReport rep = solve_underdetermined(p, cfg);
        CHECK(rep.converged);
        CHECK(std::abs(rep.x(0) - 2.0 / 3.0) <= 1e-8 && std::abs(rep.x(1) - 2.0 / 3.0) <= 1e-8);
        CHECK(rep.dual_final.size() == 1 && std::abs(rep.dual_final(0) - 2.0 / 3.0) <= 1e-8);
    }
    {
        std::mt19937_64 gen(61);
        ProblemInstance p(random_matrix(4, 12, gen), Vector::Zero(4), 0.5, Orientation::Underdetermined);
        SolveReport rep = solve_underdetermined(p, SolverConfig{});
        CHECK(rep.converged && rep.x.norm() == 0.0);
    }
    {
        std::mt19937_64 gen(62);
        Matrix A = random_matrix(16, 64, gen);
        Vector b = random_vector(16, gen);
        ProblemInstance p(A, b, 0.8, Orientation::Underdetermined);
        Vector x_ref = ridge_kernel_form(A, b, 0.8);
        for (SketchKind k : {SketchKind::Gaussian, SketchKind::SRHT}) {
            SolverConfig cfg;
            cfg.eps = 1e-18;
            cfg.sketch_kind = k;
            if (k == SketchKind::SRHT) cfg.rho = 0.25;
            SolveReport rep = solve_underdetermined(p, cfg);
            CHECK(rep.converged);
            CHECK(rep.final_m <= next_pow2(64));
            CHECK((rep.x - x_ref).norm() <= 1e-8 * (1.0 + x_ref.norm()));
        }
    }
    {
        std::mt19937_64 gen(64);
        ProblemInstance p(random_matrix(8, 3, gen), random_vector(8, gen), 1.0, Orientation::Overdetermined);
        CHECK_THROWS_AS(solve_underdetermined(p, SolverConfig{}), InvalidInput);
    }
    // ---------------------------------------------------- baselines.hpp (test_baselines.cpp:10-99)
    {
        Vector b2(2);
        b2(0) = 1.0;
        b2(1) = 2.0;
        ProblemInstance p(Matrix::Identity(2, 2), b2, 1.0, Orientation::Overdetermined);
        CgResult r = cg_solve(p, 1e-12, 10);
        CHECK(r.converged && r.iterations <= 2);
        CHECK(std::abs(r.x(0) - 0.5) <= 1e-10 && std::abs(r.x(1) - 1.0) <= 1e-10);
        CHECK(static_cast<Index>(r.residuals.size()) == r.iterations + 1);
    }
    {
        std::mt19937_64 gen(71);
        Matrix A = random_matrix(12, 4, gen);
        Vector b = random_vector(12, gen);
        ProblemInstance p(A, b, 0.6, Orientation::Overdetermined);
        Vector xs = direct_solve(p);
        CgResult r = cg_solve(p, 1e-10, 50, &xs);
        CHECK(r.converged && r.iterations == 0);
    }
    {
        std::mt19937_64 gen(72);
        Matrix A = random_matrix(30, 6, gen);
        Vector b = random_vector(30, gen);
        ProblemInstance p(A, b, 1.0, Orientation::Overdetermined);
        CgResult r = cg_solve(p, 1e-12, 200);
        CHECK(r.converged && (r.x - direct_solve(p)).norm() <= 1e-10 * (1.0 + r.x.norm()));
    }
    {
        std::mt19937_64 gen(73);
        ProblemInstance p(random_matrix(40, 20, gen), random_vector(40, gen), 1e-3, Orientation::Overdetermined);
        CHECK(!cg_solve(p, 1e-14, 1).converged);
    }
    {
        // an exact preconditioner (SA^T SA = A^T A; the reference uses an orthogonal sketch) converges in one step
        std::mt19937_64 gen(74);
        Matrix A = random_matrix(16, 5, gen);
        Vector b = random_vector(16, gen);
        ProblemInstance p(A, b, 0.7, Orientation::Overdetermined);
        PcgResult r = pcg_solve_with(p, A, 1e-10, 20);
        CHECK(r.converged && r.iterations == 1 && r.m == 16);
        CHECK((r.x - direct_solve(p)).norm() <= 1e-8 * (1.0 + r.x.norm()));
    }
    {
        auto [mg, cg_capped] = pcg_sketch_size(4096, 32, SketchKind::Gaussian, 0.25);
        CHECK(mg == 128 && !cg_capped);
        auto [ms, cs] = pcg_sketch_size(4096, 32, SketchKind::SRHT, 0.25);
        CHECK(ms == static_cast<Index>(std::ceil(32.0 * std::log(32.0) / 0.25)) && !cs);
        auto [mc, cc] = pcg_sketch_size(64, 32, SketchKind::SRHT, 0.25);
        CHECK(mc == 64 && cc);
        CHECK_THROWS_AS(pcg_sketch_size(64, 32, SketchKind::Gaussian, 1.0), InvalidInput);
    }
    {
        std::mt19937_64 gen(75);
        Matrix A = random_matrix(64, 8, gen);
        Vector b = random_vector(64, gen);
        ProblemInstance p(A, b, 0.5, Orientation::Overdetermined);
        PcgResult r = pcg_solve(p, SketchKind::Gaussian, 1, 0.25, 1e-8, 50);
        const std::uint64_t m = static_cast<std::uint64_t>(r.m);
        CHECK(r.converged && r.setup_flops == m * 64 * 8 + 8 * 8 * m + 8 * 8 * 8 / 3);
        CHECK((r.x - direct_solve(p)).norm() <= 1e-6 * (1.0 + r.x.norm()));
    }
    {
        std::mt19937_64 gen(62);
        Matrix A = random_matrix(16, 64, gen);
        Vector b = random_vector(16, gen);
        ProblemInstance p(A, b, 0.8, Orientation::Underdetermined);
        Vector x_ref = ridge_kernel_form(A, b, 0.8);
        CHECK((direct_solve(p) - x_ref).norm() <= 1e-10 * (1.0 + x_ref.norm()));
        CHECK_THROWS_AS(cg_solve(p, 1e-8, 5), InvalidInput);
    }
    std::printf("shim tests: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
