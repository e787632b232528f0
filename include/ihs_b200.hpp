// ihs_b200.hpp — header-only C++ drop-in for the reference solver API.
//
// Replaces #include <ihs/ihs.hpp> (reference proj/include/ihs/ihs.hpp:6-19)
// for the hot path: same namespace, type and function names, argument
// meaning and exception types; every numerical call goes through the C-ABI
// of libihs_b200.so (include/ihs_gpu.h) and runs on the B200. Link with
// -lihs_b200 (and -Wl,-rpath to the package directory).
//
// Matrix/Vector: the reference uses Eigen::MatrixXd / VectorXd (types.hpp:
// 9-11). Define IHS_B200_USE_EIGEN before including this header to use Eigen
// types directly; otherwise a minimal column-major ihs::Matrix / ihs::Vector
// with the members the reference API and its tests use is provided.
#pragma once

#include "ihs_gpu.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <type_traits>
#include <vector>

#ifdef IHS_B200_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace ihs {

// ------------------------------------------------------------ errors.hpp:9-57
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class InvalidInput : public Error { public: using Error::Error; };
class OutOfValidityRange : public Error { public: using Error::Error; };
class SketchTooLarge : public Error { public: using Error::Error; };
class NumericalBreakdown : public Error { public: using Error::Error; };
class DeviceError : public Error { public: using Error::Error; };

namespace detail {
inline void check(ihs_status s) {
    if (s == IHS_OK) return;
    const std::string msg = ihs_gpu_last_error();
    switch (s) {
        case IHS_INVALID_INPUT: throw InvalidInput(msg);
        case IHS_OUT_OF_VALIDITY_RANGE: throw OutOfValidityRange(msg);
        case IHS_SKETCH_TOO_LARGE: throw SketchTooLarge(msg);
        case IHS_NUMERICAL_BREAKDOWN: throw NumericalBreakdown(msg);
        case IHS_CUDA_ERROR:
        case IHS_NCCL_ERROR: throw DeviceError(msg);
        default: throw Error(msg);
    }
}
}  // namespace detail

// ------------------------------------------------------------ types.hpp
#ifdef IHS_B200_USE_EIGEN
using Index = Eigen::Index;
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
#else
using Index = std::ptrdiff_t;
class Vector {
public:
    Vector() = default;
    explicit Vector(Index n, double v = 0.0) : a_(static_cast<size_t>(n), v) {}
    Vector(std::initializer_list<double> l) : a_(l) {}
    static Vector Zero(Index n) { return Vector(n, 0.0); }
    static Vector Ones(Index n) { return Vector(n, 1.0); }
    Index size() const { return static_cast<Index>(a_.size()); }
    double& operator()(Index i) { return a_[static_cast<size_t>(i)]; }
    double operator()(Index i) const { return a_[static_cast<size_t>(i)]; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double dot(const Vector& o) const { double s = 0; for (size_t i = 0; i < a_.size(); ++i) s += a_[i] * o.a_[i]; return s; }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Vector eval() const { return *this; }
    friend Vector operator-(const Vector& x, const Vector& y) { Vector r(x.size()); for (Index i = 0; i < x.size(); ++i) r(i) = x(i) - y(i); return r; }
    friend Vector operator+(const Vector& x, const Vector& y) { Vector r(x.size()); for (Index i = 0; i < x.size(); ++i) r(i) = x(i) + y(i); return r; }
    friend Vector operator*(double s, const Vector& x) { Vector r(x.size()); for (Index i = 0; i < x.size(); ++i) r(i) = s * x(i); return r; }
    friend Vector operator/(const Vector& x, double s) { Vector r(x.size()); for (Index i = 0; i < x.size(); ++i) r(i) = x(i) / s; return r; }
private:
    std::vector<double> a_;
};
class Matrix {  // column-major like Eigen::MatrixXd
public:
    Matrix() = default;
    Matrix(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) { Matrix m(r, c); for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0; return m; }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * r_)]; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    Matrix transpose() const { Matrix t(c_, r_); for (Index j = 0; j < c_; ++j) for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j); return t; }
    friend Vector operator*(const Matrix& A, const Vector& x) { Vector y(A.rows()); for (Index j = 0; j < A.cols(); ++j) for (Index i = 0; i < A.rows(); ++i) y(i) += A(i, j) * x(j); return y; }
    friend Matrix operator*(const Matrix& A, const Matrix& B) { Matrix C(A.rows(), B.cols()); for (Index j = 0; j < B.cols(); ++j) for (Index k = 0; k < A.cols(); ++k) for (Index i = 0; i < A.rows(); ++i) C(i, j) += A(i, k) * B(k, j); return C; }
    friend Matrix operator-(const Matrix& A, const Matrix& B) { Matrix C(A.rows(), A.cols()); for (size_t e = 0; e < A.a_.size(); ++e) C.a_[e] = A.a_[e] - B.a_[e]; return C; }
    double norm() const { double s = 0; for (double v : a_) s += v * v; return std::sqrt(s); }
private:
    Index r_ = 0, c_ = 0;
    std::vector<double> a_;
};
#endif

struct CostCounters {  // types.hpp:18-33
    std::uint64_t sketch = 0, factor = 0, solve = 0, matvec = 0;
    std::uint64_t total() const noexcept { return sketch + factor + solve + matvec; }
    CostCounters& operator+=(const CostCounters& o) noexcept {
        sketch += o.sketch; factor += o.factor; solve += o.solve; matvec += o.matvec;
        return *this;
    }
};

namespace detail {
struct CounterArg {  // CostCounters* <-> ihs_counters*
    CostCounters* user;
    ihs_counters c{};
    explicit CounterArg(CostCounters* u) : user(u) { if (u) c = {u->sketch, u->factor, u->solve, u->matvec}; }
    ihs_counters* ptr() { return user ? &c : nullptr; }
    ~CounterArg() { if (user) { user->sketch = c.sketch; user->factor = c.factor; user->solve = c.solve; user->matvec = c.matvec; } }
};
}  // namespace detail

// ------------------------------------------------------------ rng.hpp (seeds)
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) { return ihs_derive_seed(seed, tag); }

// ------------------------------------------------------------ tuning.hpp:13-63
struct TuningParams { double lam = 1.0, Lam = 1.0, mu_gd = 1.0, c_gd = 0.0, mu_p = 1.0, beta_p = 0.0, c_p = 0.0; };
inline TuningParams rates_from_bounds(double lam, double Lam) {
    ihs_tuning t{};
    detail::check(ihs_rates_from_bounds(lam, Lam, &t));
    return {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
}
inline std::pair<double, double> gaussian_targets(double rho, double eta, bool enforce_validity = true) {
    double a = 0, b = 0;
    detail::check(ihs_gaussian_targets(rho, eta, enforce_validity ? 1 : 0, &a, &b));
    return {a, b};
}
inline std::pair<double, double> srht_targets(double rho) {
    double a = 0, b = 0;
    detail::check(ihs_srht_targets(rho, &a, &b));
    return {a, b};
}

// ------------------------------------------------------------ problem.hpp
enum class Orientation { Overdetermined, Underdetermined };

class ProblemInstance {
public:
    ProblemInstance(Matrix A, Vector b, double nu, Orientation o, int device = 0)
        : A_(std::move(A)), b_(std::move(b)), nu_(nu), o_(o) {
        if (!(nu_ > 0.0)) throw InvalidInput("ProblemInstance: nu must be strictly positive");
        if (A_.rows() < 1 || A_.cols() < 1) throw InvalidInput("ProblemInstance: empty matrix");
        if (b_.size() != A_.rows()) throw InvalidInput("ProblemInstance: size of b must match rows of A");
        ihs_gpu_options opts{};
        opts.device = device;
        opts.world_size = 1;
        opts.n_global = A_.rows();
        ihs_gpu_problem* h = nullptr;
        detail::check(ihs_gpu_problem_create(A_.data(), A_.rows(), A_.cols(), A_.rows(), b_.data(), nu_,
                                             o == Orientation::Overdetermined ? IHS_OVERDETERMINED : IHS_UNDERDETERMINED,
                                             &opts, &h));
        h_.reset(h, ihs_gpu_problem_destroy);
    }
    static ProblemInstance make(Matrix A, Vector b, double nu) {
        const Orientation o = A.rows() >= A.cols() ? Orientation::Overdetermined : Orientation::Underdetermined;
        return ProblemInstance(std::move(A), std::move(b), nu, o);
    }
    const Matrix& A() const noexcept { return A_; }
    const Vector& b() const noexcept { return b_; }
    double nu() const noexcept { return nu_; }
    Orientation orientation() const noexcept { return o_; }
    Index rows() const noexcept { return A_.rows(); }
    Index cols() const noexcept { return A_.cols(); }
    ihs_gpu_problem* handle() const noexcept { return h_.get(); }

private:
    Matrix A_;
    Vector b_;
    double nu_;
    Orientation o_;
    std::shared_ptr<ihs_gpu_problem> h_;
};

inline Vector gradient(const ProblemInstance& p, const Vector& x, CostCounters* counters = nullptr) {
    if (x.size() != p.cols()) throw InvalidInput("gradient: dimension mismatch");
    Vector g(p.cols());
    detail::CounterArg c(counters);
    detail::check(ihs_gpu_gradient(p.handle(), x.data(), g.data(), c.ptr()));
    return g;
}

// problem.hpp:104-109
inline double prediction_error(const ProblemInstance& p, const Vector& x, const Vector& x_star) {
    if (x.size() != p.cols() || x_star.size() != p.cols()) throw InvalidInput("prediction_error: dimension mismatch");
    double out = 0.0;
    detail::check(ihs_gpu_prediction_error(p.handle(), x.data(), x_star.data(), &out));
    return out;
}

// problem.hpp:73-82: the exact minimizer (device Gram + Cholesky + iterative refinement; the kernel form
// through the dual for underdetermined instances)
inline Vector direct_solve(const ProblemInstance& p) {
    Vector x(p.cols());
    detail::check(ihs_gpu_direct_solve(p.handle(), x.data()));
    return x;
}

// ------------------------------------------------------------ sketch.hpp
enum class SketchKind { Gaussian, SRHT };
struct SketchConfig { SketchKind kind = SketchKind::Gaussian; Index m = 1; std::uint64_t seed = 0; };
inline Index next_pow2(Index n) { return static_cast<Index>(ihs_next_pow2(n)); }

inline void fwht_inplace(Vector& v) { detail::check(ihs_gpu_fwht(v.size() ? v.data() : nullptr, v.size())); }

inline Matrix apply_sketch(const Matrix& A, const SketchConfig& cfg, CostCounters* counters = nullptr) {
    if (cfg.m < 1)
        throw InvalidInput(cfg.kind == SketchKind::SRHT ? "srht_sketch: m must be >= 1" : "gaussian_sketch: m must be >= 1");
    Matrix SA(cfg.m, A.cols());
    detail::CounterArg c(counters);
    detail::check(ihs_gpu_sketch_matrix(A.data(), A.rows(), A.cols(), A.rows(),
                                        cfg.kind == SketchKind::SRHT ? IHS_SKETCH_SRHT : IHS_SKETCH_GAUSSIAN, cfg.m,
                                        cfg.seed, SA.data(), c.ptr()));
    return SA;
}
inline Matrix gaussian_sketch(const Matrix& A, Index m, std::uint64_t seed, CostCounters* c = nullptr) {
    return apply_sketch(A, {SketchKind::Gaussian, m, seed}, c);
}
inline Matrix srht_sketch(const Matrix& A, Index m, std::uint64_t seed, CostCounters* c = nullptr) {
    return apply_sketch(A, {SketchKind::SRHT, m, seed}, c);
}

// ------------------------------------------------------------ sketched_system.hpp
enum class FactorKind { WoodburyInner, DirectGram };

class SketchedSystem {
public:
    static SketchedSystem factorize(Matrix SA, double nu, CostCounters* counters = nullptr, int device = 0) {
        if (!(nu > 0.0)) throw InvalidInput("SketchedSystem: nu must be positive");
        SketchedSystem s;
        s.SA_ = std::move(SA);
        s.nu_ = nu;
        ihs_gpu_system* h = nullptr;
        detail::CounterArg c(counters);
        detail::check(ihs_gpu_system_factorize(s.SA_.data(), s.SA_.rows(), s.SA_.cols(), std::max<Index>(1, s.SA_.rows()),
                                               nu, device, c.ptr(), &h));
        s.h_.reset(h, ihs_gpu_system_destroy);
        return s;
    }
    Index m() const noexcept { return SA_.rows(); }
    Index d() const noexcept { return SA_.cols(); }
    double nu() const noexcept { return nu_; }
    FactorKind kind() const { return ihs_gpu_system_kind(h_.get()) == IHS_FACTOR_WOODBURY_INNER ? FactorKind::WoodburyInner : FactorKind::DirectGram; }
    const Matrix& SA() const noexcept { return SA_; }
    Vector solve(const Vector& g, CostCounters* counters = nullptr) const {
        if (g.size() != d()) throw InvalidInput("SketchedSystem::solve: dimension mismatch");
        Vector z(d());
        detail::CounterArg c(counters);
        detail::check(ihs_gpu_system_solve(h_.get(), g.data(), z.data(), c.ptr()));
        return z;
    }
    std::uint64_t factor_flops() const noexcept { return ihs_gpu_system_factor_flops(h_.get()); }
    std::uint64_t flops_per_solve() const noexcept { return ihs_gpu_system_flops_per_solve(h_.get()); }
    ihs_gpu_system* handle() const noexcept { return h_.get(); }

private:
    SketchedSystem() = default;
    Matrix SA_;
    double nu_ = 0;
    std::shared_ptr<ihs_gpu_system> h_;
};

inline double newton_decrement(const Vector& g, const Vector& gt) {
    if (g.size() != gt.size()) throw InvalidInput("newton_decrement: dimension mismatch");
    double r = 0;
    detail::check(ihs_newton_decrement(g.data(), gt.data(), g.size(), &r));
    return r;
}

// ------------------------------------------------------------ solver.hpp
enum class SolveMode { PolyakThenGradient, GradientOnly };
enum class StepKind { Polyak, Gradient, Resketch };

struct SolverConfig {  // solver.hpp:28-57
    double rho = 0.1;
    double eta = 0.01;
    SketchKind sketch_kind = SketchKind::Gaussian;
    Index m_initial = 1;
    double eps = 1e-10;
    Index max_iters = 500;
    std::optional<Index> max_sketch;
    SolveMode mode = SolveMode::PolyakThenGradient;
    std::uint64_t seed = 0;
    bool enforce_validity = true;
    bool recompute_r_after_resketch = true;
    bool record_iterates = false;
    std::optional<Vector> warm_start;
    std::optional<TuningParams> tuning_override;
    std::function<Matrix(const Matrix&, Index, std::uint64_t)> sketch_override;
};

struct IterationRecord { Index t = 0; Index m = 0; double r = 0.0; double r_prev = 0.0; StepKind branch = StepKind::Gradient; };

struct SolveReport {  // solver.hpp:70-87
    Vector x;
    Index iterations = 1;
    Index rejections = 0;
    Index final_m = 0;
    double r1 = 0.0;
    double r_final = 0.0;
    bool converged = false;
    bool sketch_exhausted = false;
    std::vector<IterationRecord> log;
    std::vector<Vector> iterates;
    CostCounters counters;
    double wall_seconds = 0.0;
    TuningParams tuning;
    bool recompute_r_after_resketch = true;
    Vector dual_final;  ///< final dual iterate z_T (underdetermined solves only, solver.hpp:82)
    ihs_phase_times device_times{};
};

namespace detail {
struct OverrideCtx { const SolverConfig* cfg; const Matrix* A; };
inline int override_tramp(void* user, int64_t m, uint64_t sub_seed, double* out) {
    auto* ctx = static_cast<OverrideCtx*>(user);
    try {
        Matrix SA = ctx->cfg->sketch_override(*ctx->A, static_cast<Index>(m), sub_seed);
        if (SA.rows() != m || SA.cols() != ctx->A->cols()) return 1;
        std::memcpy(out, SA.data(), sizeof(double) * static_cast<size_t>(SA.rows() * SA.cols()));
        return 0;
    } catch (...) {
        return 1;
    }
}
}  // namespace detail

namespace detail {
// adaptive_solve / solve_underdetermined through the C-ABI; dual: the iterates, warm start and
// sketch_override live in the dual space (n), x is the primal d-vector
inline SolveReport run_solve(const ProblemInstance& p, const SolverConfig& cfg, bool dual) {
    ihs_solver_config c;
    ihs_solver_config_default(&c);
    c.rho = cfg.rho;
    c.eta = cfg.eta;
    c.sketch_kind = cfg.sketch_kind == SketchKind::SRHT ? IHS_SKETCH_SRHT : IHS_SKETCH_GAUSSIAN;
    c.mode = cfg.mode == SolveMode::GradientOnly ? IHS_MODE_GRADIENT_ONLY : IHS_MODE_POLYAK_THEN_GRADIENT;
    c.m_initial = cfg.m_initial;
    c.eps = cfg.eps;
    c.max_iters = cfg.max_iters;
    c.max_sketch = cfg.max_sketch ? *cfg.max_sketch : 0;
    c.seed = cfg.seed;
    c.enforce_validity = cfg.enforce_validity;
    c.recompute_r_after_resketch = cfg.recompute_r_after_resketch;
    c.record_iterates = cfg.record_iterates;
    if (cfg.warm_start) {
        if (cfg.warm_start->size() != (dual ? p.rows() : p.cols()))
            throw InvalidInput("adaptive_solve: warm start has wrong dimension");
        c.warm_start = cfg.warm_start->data();
    }
    if (cfg.tuning_override) {
        const auto& t = *cfg.tuning_override;
        c.has_tuning_override = 1;
        c.tuning_override = {t.lam, t.Lam, t.mu_gd, t.c_gd, t.mu_p, t.beta_p, t.c_p};
    }
    Matrix At;
    if (dual && cfg.sketch_override) {
        At = Matrix(p.cols(), p.rows());
        for (Index j = 0; j < p.rows(); ++j)
            for (Index i = 0; i < p.cols(); ++i) At(i, j) = p.A()(j, i);
    }
    detail::OverrideCtx ctx{&cfg, dual ? &At : &p.A()};
    if (cfg.sketch_override) {
        c.sketch_override = &detail::override_tramp;
        c.sketch_override_user = &ctx;
    }
    const Index d = dual ? p.rows() : p.cols();  // iterate dimension
    SolveReport out;
    out.x = Vector(p.cols());
    if (dual) out.dual_final = Vector(p.rows());
    std::vector<ihs_iteration_record> log(4096);
    std::vector<double> its;
    ihs_solve_report r{};
    r.x = out.x.data();
    if (dual) r.dual_final = out.dual_final.data();
    auto call = [&] {
        detail::check(dual ? ihs_gpu_solve_underdetermined(p.handle(), &c, &r) : ihs_gpu_adaptive_solve(p.handle(), &c, &r));
    };
    r.log = log.data();
    r.log_capacity = static_cast<int64_t>(log.size());
    if (cfg.record_iterates) {
        its.resize(static_cast<size_t>((cfg.max_iters + 1) * d));
        r.iterates = its.data();
        r.iterates_capacity = cfg.max_iters + 1;
    }
    call();
    if (r.log_size > r.log_capacity) {  // rare: rerun with a larger audit buffer
        log.resize(static_cast<size_t>(r.log_size));
        r.log = log.data();
        r.log_capacity = r.log_size;
        call();
    }
    out.iterations = r.iterations;
    out.rejections = r.rejections;
    out.final_m = r.final_m;
    out.r1 = r.r1;
    out.r_final = r.r_final;
    out.converged = r.converged != 0;
    out.sketch_exhausted = r.sketch_exhausted != 0;
    for (int64_t i = 0; i < r.log_size; ++i) {
        const auto& e = log[static_cast<size_t>(i)];
        out.log.push_back({e.t, e.m, e.r, e.r_prev,
                           e.branch == IHS_STEP_POLYAK ? StepKind::Polyak
                           : e.branch == IHS_STEP_GRADIENT ? StepKind::Gradient : StepKind::Resketch});
    }
    for (int64_t i = 0; i < r.iterates_size && i < r.iterates_capacity; ++i) {
        Vector v(d);
        std::memcpy(v.data(), its.data() + i * d, sizeof(double) * static_cast<size_t>(d));
        out.iterates.push_back(std::move(v));
    }
    out.counters = {r.counters.sketch, r.counters.factor, r.counters.solve, r.counters.matvec};
    out.wall_seconds = r.wall_seconds;
    out.tuning = {r.tuning.lam, r.tuning.Lam, r.tuning.mu_gd, r.tuning.c_gd, r.tuning.mu_p, r.tuning.beta_p, r.tuning.c_p};
    out.recompute_r_after_resketch = r.recompute_r_after_resketch != 0;
    out.device_times = r.times;
    return out;
}
}  // namespace detail

inline SolveReport adaptive_solve(const ProblemInstance& p, const SolverConfig& cfg) {  // solver.hpp:242-250
    if (p.orientation() != Orientation::Overdetermined)
        throw InvalidInput("adaptive_solve: expects an overdetermined instance (use solve_underdetermined for d > n)");
    return detail::run_solve(p, cfg, false);
}

// dual.hpp:13-33: the dual ridge problem in A^T; x = A^T z_T, dual_final = z_T, iterates = dual trace
inline SolveReport solve_underdetermined(const ProblemInstance& p, const SolverConfig& cfg) {
    if (p.orientation() != Orientation::Underdetermined)
        throw InvalidInput("solve_underdetermined: expects an underdetermined instance");
    return detail::run_solve(p, cfg, true);
}


enum class FixedMode { Gradient, Polyak };

inline std::vector<Vector> fixed_sketch_ihs(const ProblemInstance& p, const SketchedSystem& sys, const TuningParams& tp,
                                            Index T, FixedMode mode, const Vector* x_start = nullptr) {
    const Index d = p.cols();
    std::vector<double> buf(static_cast<size_t>((T + 1) * d));
    ihs_tuning t{tp.lam, tp.Lam, tp.mu_gd, tp.c_gd, tp.mu_p, tp.beta_p, tp.c_p};
    detail::check(ihs_gpu_fixed_sketch_ihs(p.handle(), sys.handle(), &t, T,
                                           mode == FixedMode::Polyak ? IHS_FIXED_POLYAK : IHS_FIXED_GRADIENT,
                                           x_start ? x_start->data() : nullptr, buf.data()));
    std::vector<Vector> out;
    for (Index k = 0; k <= T; ++k) {
        Vector v(d);
        std::memcpy(v.data(), buf.data() + k * d, sizeof(double) * static_cast<size_t>(d));
        out.push_back(std::move(v));
    }
    return out;
}

// ------------------------------------------------------------ baselines.hpp
struct CgResult {  // baselines.hpp:16-23
    Vector x;
    Index iterations = 0;
    std::vector<double> residuals;
    bool converged = false;
    CostCounters counters;
    double wall_seconds = 0.0;
};
struct PcgResult {  // baselines.hpp:25-36
    Vector x;
    Index iterations = 0;
    std::vector<double> residuals;
    bool converged = false;
    Index m = 0;
    bool m_capped = false;
    std::uint64_t setup_flops = 0;
    CostCounters counters;
    double wall_seconds = 0.0;
};

namespace detail {
template <class R, class F>
R run_cg(const ProblemInstance& p, Index max_iters, const Vector* x0, F&& call) {
    if (x0 && x0->size() != p.cols()) throw InvalidInput("cg_solve: dimension mismatch");
    R res;
    res.x = Vector(p.cols());
    const Index cap = (max_iters > 0 ? max_iters : 0) + 1;
    res.residuals.assign(static_cast<size_t>(cap), 0.0);
    ihs_cg_report rep{};
    rep.x = res.x.data();
    rep.residuals = res.residuals.data();
    rep.residuals_capacity = cap;
    check(call(x0 ? x0->data() : nullptr, &rep));
    res.residuals.resize(static_cast<size_t>(std::min<int64_t>(rep.residuals_size, cap)));
    res.iterations = rep.iterations;
    res.converged = rep.converged != 0;
    res.counters = CostCounters{rep.counters.sketch, rep.counters.factor, rep.counters.solve, rep.counters.matvec};
    res.wall_seconds = rep.wall_seconds;
    if constexpr (std::is_same_v<R, PcgResult>) {
        res.m = rep.m;
        res.m_capped = rep.m_capped != 0;
        res.setup_flops = rep.setup_flops;
    }
    return res;
}
}  // namespace detail

inline CgResult cg_solve(const ProblemInstance& p, double tol, Index max_iters, const Vector* x0 = nullptr) {
    return detail::run_cg<CgResult>(p, max_iters, x0, [&](const double* x0p, ihs_cg_report* r) {
        return ihs_gpu_cg_solve(p.handle(), tol, max_iters, x0p, r);
    });
}

inline PcgResult pcg_solve_with(const ProblemInstance& p, const Matrix& SA, double tol, Index max_iters,
                                const Vector* x0 = nullptr) {
    if (SA.cols() != p.cols()) throw InvalidInput("pcg_solve: dimension mismatch");
    return detail::run_cg<PcgResult>(p, max_iters, x0, [&](const double* x0p, ihs_cg_report* r) {
        return ihs_gpu_pcg_solve_with(p.handle(), SA.data(), SA.rows(), SA.rows(), tol, max_iters, x0p, r);
    });
}

inline std::pair<Index, bool> pcg_sketch_size(Index n, Index d, SketchKind kind, double rho) {
    int64_t m = 0;
    int32_t capped = 0;
    detail::check(ihs_pcg_sketch_size(n, d, kind == SketchKind::SRHT ? IHS_SKETCH_SRHT : IHS_SKETCH_GAUSSIAN, rho,
                                      &m, &capped));
    return {static_cast<Index>(m), capped != 0};
}

inline PcgResult pcg_solve(const ProblemInstance& p, SketchKind kind, std::uint64_t seed, double rho, double tol,
                           Index max_iters, const Vector* x0 = nullptr) {
    return detail::run_cg<PcgResult>(p, max_iters, x0, [&](const double* x0p, ihs_cg_report* r) {
        return ihs_gpu_pcg_solve(p.handle(), kind == SketchKind::SRHT ? IHS_SKETCH_SRHT : IHS_SKETCH_GAUSSIAN, seed,
                                 rho, tol, max_iters, x0p, r);
    });
}

}  // namespace ihs
