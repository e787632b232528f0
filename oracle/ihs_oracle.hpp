// ihs_oracle.hpp — CPU ORACLE (test infrastructure only).
//
// A plain C++20 restatement of the reference's hot path, written without
// Eigen (which is absent from this image, so the reference itself cannot be
// compiled here — see DESIGN.md §Oracle). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it, and only
// as the checker or the timed CPU baseline. The product
// (paper_2006_05874_b200/) never links or calls anything in this directory.
//
// Every function cites the reference file:line it follows
// (/root/reference/proj/include/ihs/...). RNG streams use the very same
// libstdc++ types as the reference (std::mt19937_64, normal_distribution,
// uniform_int_distribution), so D, P and S are the reference's values
// bit-for-bit. Dense linear algebra (GEMV/GEMM/LLT) replaces Eigen calls and
// matches them to floating-point tolerance only (different summation order).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace ihs_oracle {

using Index = long;  // Eigen::Index == std::ptrdiff_t (types.hpp:9)

// ---------------------------------------------------------------- errors.hpp:9-40
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidInput : Error { using Error::Error; };
struct OutOfValidityRange : Error { using Error::Error; };
struct SketchTooLarge : Error { using Error::Error; };
struct NumericalBreakdown : Error { using Error::Error; };

// ---------------------------------------------------------------- types.hpp:9-33
struct Mat {  // column-major like Eigen::MatrixXd
    Index rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index r, Index c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), v) {}
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * rows)]; }
    double* col(Index j) { return a.data() + j * rows; }
    const double* col(Index j) const { return a.data() + j * rows; }
};
using Vec = std::vector<double>;

struct CostCounters {
    std::uint64_t sketch = 0, factor = 0, solve = 0, matvec = 0;
    std::uint64_t total() const { return sketch + factor + solve + matvec; }
};

// ---------------------------------------------------------------- rng.hpp:13-66
std::uint64_t splitmix64(std::uint64_t& state);                         // rng.hpp:13-18
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag);       // rng.hpp:23-28
std::mt19937_64 make_stream(std::uint64_t seed, std::uint64_t tag);     // rng.hpp:30-32
void fill_gaussian(double* M, Index rows, Index cols, std::mt19937_64& gen, double stddev = 1.0);  // :35-40
std::vector<double> rademacher(Index n, std::mt19937_64& gen);           // rng.hpp:48-52
std::vector<Index> sample_without_replacement(Index n, Index m, std::mt19937_64& gen);  // :56-66

// ---------------------------------------------------------------- sketch.hpp
enum class SketchKind { Gaussian = 0, SRHT = 1 };                        // sketch.hpp:16
Index next_pow2(Index n);                                                // sketch.hpp:26-28
void fwht_inplace(double* v, std::size_t n);                             // sketch.hpp:33-49
Mat gaussian_sketch(const Mat& A, Index m, std::uint64_t seed, CostCounters* c = nullptr);  // :58-69
Mat srht_sketch(const Mat& A, Index m, std::uint64_t seed, CostCounters* c = nullptr);      // :77-108
Mat apply_sketch(const Mat& A, SketchKind kind, Index m, std::uint64_t seed, CostCounters* c = nullptr);  // :110-117

// ---------------------------------------------------------------- problem.hpp
struct Problem {                                                         // problem.hpp:20-55
    Mat A;
    Vec b;
    double nu = 1.0;
    bool underdetermined = false;  // Orientation (problem.hpp:14)
    Problem(Mat A_, Vec b_, double nu_, bool underdetermined = false);
};
Vec gradient(const Problem& p, const Vec& x, CostCounters* c = nullptr); // problem.hpp:59-69
Vec direct_solve(const Problem& p);  // ridge normal equations (support.hpp:19-23), Cholesky
double prediction_error(const Problem& p, const Vec& x, const Vec& x_star);  // problem.hpp:104-109

// ---------------------------------------------------------------- sketched_system.hpp
enum class FactorKind { WoodburyInner = 0, DirectGram = 1 };             // sketched_system.hpp:12
class SketchedSystem {                                                   // :23-101
public:
    static SketchedSystem factorize(Mat SA, double nu, CostCounters* c = nullptr);
    Index m() const { return SA_.rows; }
    Index d() const { return SA_.cols; }
    FactorKind kind() const { return kind_; }
    const Mat& SA() const { return SA_; }
    Vec solve(const Vec& g, CostCounters* c = nullptr) const;
    std::uint64_t factor_flops() const;
    std::uint64_t flops_per_solve() const;
private:
    SketchedSystem(Mat SA, double nu);
    Mat SA_;
    double nu_;
    FactorKind kind_;
    Mat L_;  // lower Cholesky factor
};
double newton_decrement(const Vec& g, const Vec& gt);                    // :95-101

// ---------------------------------------------------------------- tuning.hpp:13-63
struct TuningParams { double lam = 1, Lam = 1, mu_gd = 1, c_gd = 0, mu_p = 1, beta_p = 0, c_p = 0; };
TuningParams rates_from_bounds(double lam, double Lam);
std::pair<double, double> gaussian_targets(double rho, double eta, bool enforce_validity = true);
std::pair<double, double> srht_targets(double rho);

// ---------------------------------------------------------------- solver.hpp
enum class SolveMode { PolyakThenGradient = 0, GradientOnly = 1 };       // :19-22
enum class StepKind { Polyak = 0, Gradient = 1, Resketch = 2 };          // :24
struct SolverConfig {                                                    // :28-57
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
    std::optional<Vec> warm_start;
    std::optional<TuningParams> tuning_override;
    std::function<Mat(const Mat&, Index, std::uint64_t)> sketch_override;
};
struct IterationRecord { Index t = 0, m = 0; double r = 0, r_prev = 0; StepKind branch = StepKind::Gradient; };
struct SolveReport {                                                     // :70-87
    Vec x;
    Index iterations = 1, rejections = 0, final_m = 0;
    double r1 = 0, r_final = 0;
    bool converged = false, sketch_exhausted = false;
    std::vector<IterationRecord> log;
    std::vector<Vec> iterates;
    CostCounters counters;
    double wall_seconds = 0;
    TuningParams tuning;
    bool recompute_r_after_resketch = true;
    Vec dual_final;  // underdetermined solves only (solver.hpp:82)
};
using GradFn = std::function<Vec(const Vec&, CostCounters*)>;
SolveReport adaptive_solve_core(const Mat& A, double nu, const GradFn& grad, const SolverConfig& cfg);  // :106-232
SolveReport adaptive_solve(const Problem& p, const SolverConfig& cfg);  // :242-250
SolveReport solve_underdetermined(const Problem& p, const SolverConfig& cfg);  // dual.hpp:13-33
enum class FixedMode { Gradient = 0, Polyak = 1 };
std::vector<Vec> fixed_sketch_ihs(const Problem& p, const SketchedSystem& sys, const TuningParams& tp,
                                  Index T, FixedMode mode, const Vec* x_start = nullptr);  // :258-276

// ---------------------------------------------------------------- baselines.hpp
struct CgResult {  // CgResult / PcgResult (baselines.hpp:16-36); the PCG fields stay 0 for plain CG
    Vec x;
    Index iterations = 0;
    std::vector<double> residuals;  // ||H x_k - A^T b|| per iteration, incl. the start
    bool converged = false;
    Index m = 0;
    bool m_capped = false;
    std::uint64_t setup_flops = 0;
    CostCounters counters;
};
CgResult cg_solve(const Problem& p, double tol, Index max_iters, const Vec* x0 = nullptr);  // :40-92
CgResult pcg_solve_with(const Problem& p, const Mat& SA, double tol, Index max_iters, CgResult res = {},
                        const Vec* x0 = nullptr);                                          // :98-165
std::pair<Index, bool> pcg_sketch_size(Index n, Index d, SketchKind kind, double rho);     // :170-187
CgResult pcg_solve(const Problem& p, SketchKind kind, std::uint64_t seed, double rho, double tol, Index max_iters,
                   const Vec* x0 = nullptr);                                               // :190-200

// ---------------------------------------------------------------- synthetic data
struct SynthSpec {
    Index n = 0, d = 0;
    int spectrum = 0;         // 0: decay^j, 1: 1/j  (j = 1..d, datasets.hpp:52-58 convention)
    double decay = 0.95, noise_std = 0.01, outlier_frac = 0.0, outlier_scale = 100.0;
    std::uint64_t data_seed = 0;
};
void synth_generate(const SynthSpec& s, Mat& A, Vec& b, Vec& x_true);

}  // namespace ihs_oracle
