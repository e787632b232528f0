"""Pin the CPU oracle to the reference itself.

oracle/_ref/libihs_ref.so is the reference's own headers (/root/reference/proj/include/ihs/{rng,sketch,problem,
sketched_system,tuning,solver,dual,baselines}.hpp), compiled unchanged by `make -C oracle ref` against the
Eigen-API subset in oracle/eigen_stub. Each test drives the oracle restatement (oracle/ihs_oracle.cpp) and the
reference code with identical inputs:

* bit-for-bit: seeds (rng.hpp:13-32), raw MT19937-64 draws, the Rademacher signs D (rng.hpp:48-52), the row
  sample P (rng.hpp:56-66), the Gaussian fill S (rng.hpp:35-40), the FWHT (sketch.hpp:33-49), the SRHT sketch SA
  (sketch.hpp:77-108), the Gaussian sketch (both sum S*A over n in ascending order), the synthetic data, the
  tuning scalars (tuning.hpp:25-63) and every cost counter;
* identical control flow: the adaptive solver's audit trail (t, m, branch) — i.e. the m-schedule and the
  Polyak/gradient/resketch decisions — iteration and rejection counts, convergence flags (solver.hpp:106-232);
* fp64 tolerance for values that pass through dense algebra (stated per test).
"""
import numpy as np
import pytest


def _abar_rel(A, nu, x, xr):
    num = np.linalg.norm(np.concatenate([A @ (x - xr), nu * (x - xr)]))
    den = np.linalg.norm(np.concatenate([A @ xr, nu * xr]))
    return num / den if den > 0 else num


def _counters(c):
    return (c.sketch, c.factor, c.solve, c.matvec)


def test_seeds_and_streams_bit_exact(O, R):
    for seed in (0, 1, 7, 12345, 2**63 + 11):
        for tag in (0, 1, 2, 3, 12, 13, 14, 1000, 2**40):
            assert O.derive_seed(seed, tag) == R.derive_seed(seed, tag)
    for s in (0, 5, O.derive_seed(3, 1)):
        assert np.array_equal(O.mt_raw(s, 20000), R.mt_raw(s, 20000))
        for n in (1, 2, 3, 1000, 4096, 1 << 17):
            assert np.array_equal(O.rademacher(s, n), R.rademacher(s, n))
        for n, m in ((1, 1), (7, 7), (4096, 1), (4096, 257), (1 << 20, 4096), (1 << 22, 4096), (1000, 1000)):
            assert np.array_equal(O.sample_without_replacement(s, n, m), R.sample_without_replacement(s, n, m))
        for rows, cols in ((1, 1), (1, 7), (37, 29), (1024, 3)):
            assert np.array_equal(O.fill_gaussian(s, rows, cols, 0.3), R.fill_gaussian(s, rows, cols, 0.3))


def test_fwht_bit_exact(O, R):
    rng = np.random.default_rng(0)
    for n in (1, 2, 4, 64, 1024, 1 << 16):
        v = rng.standard_normal(n)
        assert np.array_equal(O.fwht_inplace(v), R.fwht_inplace(v))
    for n in (0, 3, 12):
        with pytest.raises(Exception):
            O.fwht_inplace(np.ones(n))
        with pytest.raises(Exception):
            R.fwht_inplace(np.ones(n))


@pytest.mark.parametrize("n,d,outliers", [(3000, 12, 0.01), (4096, 48, 0.0), (70000, 3, 0.02)])
def test_synthetic_data_bit_exact(O, R, n, d, outliers):
    a = O.synth(n, d, decay=0.97, noise_std=0.1, outlier_frac=outliers, data_seed=4)
    b = R.synth(n, d, decay=0.97, noise_std=0.1, outlier_frac=outliers, data_seed=4)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    a = O.synth(n, d, spectrum=1, noise_std=0.01, data_seed=9)
    b = R.synth(n, d, spectrum=1, noise_std=0.01, data_seed=9)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("n,d", [(1, 1), (5, 3), (1000, 7), (4096, 16), (3001, 12), (70000, 4)])
def test_srht_sketch_bit_exact(O, R, n, d):
    A, _, _ = O.synth(n, d, decay=0.9, noise_std=0.0, data_seed=n)
    n_pad = O.next_pow2(n)
    assert n_pad == R.next_pow2(n)
    for m in sorted({1, min(2, n_pad), max(1, n_pad // 3), n_pad}):
        for seed in (0, 3):
            co, cr = O.abi.Counters(), O.abi.Counters()
            so = O.srht_sketch(A, m, seed, co)
            sr = R.srht_sketch(A, m, seed, cr)
            assert np.array_equal(so, sr), (n, d, m, seed)
            assert _counters(co) == _counters(cr)
    with pytest.raises(Exception):
        R.srht_sketch(A, n_pad + 1, 0)
    with pytest.raises(Exception):
        O.srht_sketch(A, n_pad + 1, 0)


@pytest.mark.parametrize("n,d,m", [(200, 5, 1), (1000, 7, 33), (4096, 16, 300)])
def test_gaussian_sketch_bit_exact(O, R, n, d, m):
    # both sum S*A over the n rows in ascending order, so even the product agrees to the bit
    A, _, _ = O.synth(n, d, decay=0.9, noise_std=0.0, data_seed=1)
    co, cr = O.abi.Counters(), O.abi.Counters()
    assert np.array_equal(O.gaussian_sketch(A, m, 5, co), R.gaussian_sketch(A, m, 5, cr))
    assert _counters(co) == _counters(cr)


def test_gradient_and_prediction_error(O, R):
    A, b, _ = O.synth(5000, 40, decay=0.95, noise_std=0.01, data_seed=2)
    x = np.random.default_rng(1).standard_normal(40)
    co, cr = O.abi.Counters(), O.abi.Counters()
    go, gr = O.gradient(A, b, 0.03, x, co), R.gradient(A, b, 0.03, x, cr)
    assert np.max(np.abs(go - gr)) <= 1e-12 * np.max(np.abs(gr))  # summation order differs (fp64 tolerance)
    assert _counters(co) == _counters(cr)
    xs = R.direct_solve(A, b, 0.03)
    assert _abar_rel(A, 0.03, O.direct_solve(A, b, 0.03), xs) <= 1e-12
    po, pr = O.prediction_error(A, b, 0.03, x, xs), R.prediction_error(A, b, 0.03, x, xs)
    assert abs(po - pr) <= 1e-12 * pr


@pytest.mark.parametrize("m,d", [(5, 20), (20, 20), (64, 20), (1, 1)])
def test_sketched_system(O, R, m, d):
    rng = np.random.default_rng(m)
    SA = rng.standard_normal((m, d))
    g = rng.standard_normal(d)
    co, cr = O.abi.Counters(), O.abi.Counters()
    zo, ko, fo, so = O.system_solve(SA, 0.3, g, co)
    zr, kr, fr, sr = R.system_solve(SA, 0.3, g, cr)
    assert (ko, fo, so) == (kr, fr, sr) and ko == (1 if m >= d else 0)  # branch rule m < d (:114)
    assert _counters(co) == _counters(cr)
    assert np.max(np.abs(zo - zr)) <= 1e-11 * np.max(np.abs(zr))
    assert abs(O.newton_decrement(g, zo) - R.newton_decrement(g, zr)) <= 1e-11 * R.newton_decrement(g, zr)


def test_tuning_bit_exact(O, R):
    for lam, Lam in [(0.5, 2.0), (1.0, 1.0), (0.2, 1.7), (1e-3, 3.9)]:
        a, b = O.rates_from_bounds(lam, Lam), R.rates_from_bounds(lam, Lam)
        assert [getattr(a, f) for f, _ in a._fields_] == [getattr(b, f) for f, _ in b._fields_]
    for rho in (0.01, 0.1, 0.18, 0.35, 0.55):
        assert O.srht_targets(rho) == R.srht_targets(rho)
        for eta in (0.001, 0.01):
            assert O.gaussian_targets(rho, eta, False) == R.gaussian_targets(rho, eta, False)
    for bad in [(0.5, 0.01, True), (0.1, 0.02, True)]:
        with pytest.raises(Exception):
            R.gaussian_targets(*bad)
        with pytest.raises(Exception):
            O.gaussian_targets(*bad)


SOLVE_CASES = [
    # (label, n, d, nu, decay, config overrides)
    ("gauss-default", 3000, 24, 0.05, 0.9, dict(sketch_kind=0)),
    ("srht-default", 3000, 24, 0.05, 0.9, dict(sketch_kind=1)),
    ("srht-gradonly", 4096, 32, 1e-2, 0.95, dict(sketch_kind=1, mode=1)),
    ("gauss-no-recompute", 3000, 24, 0.05, 0.9, dict(sketch_kind=0, recompute_r_after_resketch=0)),
    ("srht-no-recompute", 3000, 24, 0.05, 0.9, dict(sketch_kind=1, recompute_r_after_resketch=0)),
    ("gauss-eta", 3000, 24, 0.05, 0.9, dict(sketch_kind=0, rho=0.05, eta=0.001)),
    ("gauss-outside-validity", 3000, 24, 0.05, 0.9, dict(sketch_kind=0, rho=0.35, enforce_validity=0)),
    ("srht-minit-cap", 5000, 40, 1e-3, 0.97, dict(sketch_kind=1, m_initial=80, max_sketch=640, eps=1e-21)),
    ("srht-tight-eps", 8192, 64, 1e-3, 0.99, dict(sketch_kind=1, m_initial=128, eps=1e-21)),
    ("gauss-capped", 2000, 30, 1e-3, 0.97, dict(sketch_kind=0, max_sketch=64, max_iters=60)),
    ("srht-seed", 3000, 24, 0.05, 0.9, dict(sketch_kind=1, seed=77)),
]


@pytest.mark.parametrize("label,n,d,nu,decay,over", SOLVE_CASES, ids=[c[0] for c in SOLVE_CASES])
def test_adaptive_solve_pinned(O, R, label, n, d, nu, decay, over):
    A, b, _ = O.synth(n, d, decay=decay, noise_std=0.01, data_seed=11)
    cfg = O.default_config(**over)
    xo, ro, lo, _ = O.adaptive_solve(A, b, nu, cfg)
    xr, rr, lr, _ = R.adaptive_solve(A, b, nu, cfg)
    assert [(e[0], e[1], e[4]) for e in lo] == [(e[0], e[1], e[4]) for e in lr]  # m-schedule + branches
    assert (ro.iterations, ro.rejections, ro.final_m, ro.converged, ro.sketch_exhausted) == \
           (rr.iterations, rr.rejections, rr.final_m, rr.converged, rr.sketch_exhausted)
    assert _counters(ro.counters) == _counters(rr.counters)
    assert [getattr(ro.tuning, f) for f, _ in ro.tuning._fields_] == [getattr(rr.tuning, f) for f, _ in rr.tuning._fields_]
    for a, b_ in zip(lo, lr):  # decrements: fp64 tolerance (GEMV/Cholesky), floor 1e-20 r_1 near convergence
        assert abs(a[2] - b_[2]) <= 1e-8 * abs(b_[2]) + 1e-20 * rr.r1
    assert abs(ro.r1 - rr.r1) <= 1e-10 * rr.r1
    assert _abar_rel(A, nu, xo, xr) <= 1e-10


def test_warm_start_and_tuning_override_pinned(O, R):
    A, b, _ = O.synth(3000, 24, decay=0.9, noise_std=0.01, data_seed=12)
    x0 = np.random.default_rng(3).standard_normal(24)
    cfg = O.default_config(sketch_kind=1)
    cfg.warm_start = O._dp(np.ascontiguousarray(x0))
    cfg.has_tuning_override = 1
    t = R.rates_from_bounds(0.4, 1.6)
    cfg.tuning_override = t
    xo, ro, lo, _ = O.adaptive_solve(A, b, 0.05, cfg)
    xr, rr, lr, _ = R.adaptive_solve(A, b, 0.05, cfg)
    assert [(e[0], e[1], e[4]) for e in lo] == [(e[0], e[1], e[4]) for e in lr]
    assert _counters(ro.counters) == _counters(rr.counters)
    assert _abar_rel(A, 0.05, xo, xr) <= 1e-10


@pytest.mark.parametrize("kind", [0, 1])
def test_config_c1_full_size_pinned(O, R, kind):
    """BASELINE configs[0] (C1: n=8192, d=256, sigma_j=0.95^j, nu=1e-2, m from 1) at full size, both sketches."""
    A, b, _ = O.synth(8192, 256, decay=0.95, noise_std=0.01, data_seed=0)
    cfg = O.default_config(sketch_kind=kind, mode=1 if kind == 1 else 0)
    xo, ro, lo, _ = O.adaptive_solve(A, b, 1e-2, cfg)
    xr, rr, lr, _ = R.adaptive_solve(A, b, 1e-2, cfg)
    assert [(e[0], e[1], e[4]) for e in lo] == [(e[0], e[1], e[4]) for e in lr]
    assert _counters(ro.counters) == _counters(rr.counters)
    assert _abar_rel(A, 1e-2, xo, xr) <= 1e-10


def test_dual_and_fixed_sketch_pinned(O, R):
    Au, bu, _ = O.synth(300, 40, decay=0.95, noise_std=0.01, data_seed=8)
    Au = np.asfortranarray(Au.T)
    bu = bu[:40].copy()
    cfg = O.default_config(seed=5)
    xo, zo, ro, lo, _ = O.solve_underdetermined(Au, bu, 0.3, cfg)
    xr, zr, rr, lr, _ = R.solve_underdetermined(Au, bu, 0.3, cfg)
    assert [(e[0], e[1], e[4]) for e in lo] == [(e[0], e[1], e[4]) for e in lr]
    assert _counters(ro.counters) == _counters(rr.counters)
    assert np.max(np.abs(xo - xr)) <= 1e-9 * np.max(np.abs(xr))
    A, b, _ = O.synth(4096, 32, decay=0.95, data_seed=4)
    SA = R.gaussian_sketch(A, 128, 5)
    tp = R.rates_from_bounds(*R.gaussian_targets(0.3, 0.01, False))
    for mode in (0, 1):
        io = O.fixed_sketch_ihs(A, b, 0.05, SA, tp, 20, mode)
        ir = R.fixed_sketch_ihs(A, b, 0.05, SA, tp, 20, mode)
        assert np.array_equal(io[0], ir[0])
        for k in range(1, 21):
            assert _abar_rel(A, 0.05, io[k], ir[k]) <= 1e-10


def test_baselines_pinned(O, R):
    A, b, _ = O.synth(3000, 24, decay=0.9, noise_std=0.01, data_seed=7)
    # plain CG on this ill-conditioned instance is chaotic past ~15 iterations (residual traces of any two
    # summation orders separate there), so the trace is compared up to that horizon and the rest by its law
    xo, reso, ro = O.cg_solve(A, b, 0.05, 1e-8, 200)
    xr, resr, rr = R.cg_solve(A, b, 0.05, 1e-8, 200)
    assert ro.converged and rr.converged and abs(ro.iterations - rr.iterations) <= 2
    np.testing.assert_allclose(reso[:14], resr[:14], rtol=1e-12)
    n, d = A.shape
    for res, rep in ((reso, ro), (resr, rr)):  # baselines.hpp:51: one H apply per iteration plus the start
        assert rep.counters.matvec == (rep.iterations + 1) * (2 * n * d + 2 * d)
        assert len(res) == rep.iterations + 1
    for kind in (0, 1):
        assert O.pcg_sketch_size(3000, 24, kind, 0.1) == R.pcg_sketch_size(3000, 24, kind, 0.1)
        xo, reso, ro = O.pcg_solve(A, b, 0.05, kind, 4, 0.5, 1e-10, 100)
        xr, resr, rr = R.pcg_solve(A, b, 0.05, kind, 4, 0.5, 1e-10, 100)
        assert (ro.iterations, ro.m, ro.converged, ro.m_capped, ro.setup_flops) == \
               (rr.iterations, rr.m, rr.converged, rr.m_capped, rr.setup_flops)
        assert _counters(ro.counters) == _counters(rr.counters)
        assert _abar_rel(A, 0.05, xo, xr) <= 1e-10
