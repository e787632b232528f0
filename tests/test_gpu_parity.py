"""GPU parity: the CUDA path through the C-ABI against the CPU oracle.

Bit-exact for the integer/stream parts (mt19937_64 draws, Rademacher bits,
sample indices, SRHT SA values, FWHT); fp64 tolerance (stated per test) for
the Eigen-replaced linear algebra (Gaussian S*A, gradient, LLT solves).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng


def rand_mat(seed, n, d):
    return np.asfortranarray(RNG(seed).standard_normal((n, d)))


# ----------------------------------------------------------------- rng.hpp
def test_mt19937_64_known_answer(gpu):
    # C++ standard [rand.predef]: the 10000th draw of default mt19937_64 (seed 5489)
    raw = gpu.mt19937_64(5489, 10000)
    assert int(raw[-1]) == 9981545732273789042


@pytest.mark.parametrize("seed", [0, 1, 12345678901234567])
def test_mt19937_64_stream(gpu, O, seed):
    s = O.derive_seed(seed, 1)
    assert np.array_equal(gpu.mt19937_64(s, 5000), O.mt_raw(s, 5000))


@pytest.mark.parametrize("n", [1, 31, 32, 33, 311, 312, 313, 9984, 9985, 20000, 1 << 17])
def test_rademacher_bits(gpu, O, n):
    s = O.derive_seed(O.derive_seed(3, 5), 1)
    assert np.array_equal(gpu.rademacher(s, n), O.rademacher(s, n))


@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 7), (64, 33), (1000, 17)])
def test_fill_gaussian_small(gpu, O, rows, cols):
    s = O.derive_seed(11, 0)
    a = gpu.fill_gaussian(s, rows, cols, 0.25)
    b = O.fill_gaussian(s, rows, cols, 0.25)
    # acceptance is exact; values may differ from glibc's log by a last-ulp rounding
    np.testing.assert_allclose(a, b, rtol=1e-15, atol=0)


def test_fill_gaussian_jump_ahead(gpu, O):
    # long enough to use several jump-ahead substreams (stride 2^19 draws)
    s = O.derive_seed(2024, 0)
    rows, cols = 1024, 1200
    a = gpu.fill_gaussian(s, rows, cols, 1.0 / 32.0)
    b = O.fill_gaussian(s, rows, cols, 1.0 / 32.0)
    # positions are exact (acceptance uses no log); a last-ulp log difference from
    # glibc can move a value by <= 2 ulp through sqrt/div/mul
    np.testing.assert_allclose(a, b, rtol=1e-15, atol=0)
    assert np.mean(a == b) > 0.99  # measured: 99.88% bit-identical, the rest 1-2 ulp


# ----------------------------------------------------------------- sketch.hpp
@pytest.mark.parametrize("n", [1, 2, 4, 16, 64, 1024, 8192, 1 << 14, 1 << 16])
def test_fwht_bit_exact(gpu, O, n):
    v = RNG(n).standard_normal(n)
    a = gpu.fwht_inplace(v.copy())
    b = O.fwht_inplace(v)
    assert np.array_equal(a, b)


def test_fwht_known_answer(gpu):
    v = np.array([1.0, 0.0, 0.0, 0.0])
    gpu.fwht_inplace(v)
    assert np.all(v == 0.5)  # test_sketch.cpp:13-17


def test_fwht_rejects_non_pow2(gpu):
    with pytest.raises(gpu.InvalidInput):
        gpu.fwht_inplace(np.zeros(12))


@pytest.mark.parametrize("n,d,m,seed", [
    (12, 4, 8, 77), (1000, 2, 16, 0), (8192, 16, 100, 5), (8192, 8, 8192, 1), (5000, 7, 333, 2),
    (20000, 5, 1000, 3), (1 << 15, 4, 4096, 4), (100000, 3, 20000, 9), ((1 << 20) - 17, 2, 5000, 6),
    # n_pad = 2^20: compact T (one warp per distinct low index) from 1 to ~1000 distinct low indices
    ((1 << 19) + 3, 3, 1, 13), ((1 << 20) - 1, 2, 3, 14), (700000, 3, 100, 15), ((1 << 20), 2, 1024, 16),
    # n_pad = 2^21 / 2^22: one 11- / 12-bit pass of three-round 512-thread tiles
    ((1 << 20) + 5, 2, 3000, 8), ((1 << 21) + 1, 2, 40000, 10), ((1 << 22) - 3, 2, 777, 12)])
def test_srht_sketch_bit_exact(gpu, O, n, d, m, seed):
    A = rand_mat(n + d, n, d)
    c_gpu = gpu.CostCounters()
    SA = gpu.srht_sketch(A, m, seed, c_gpu)
    c_or = O.abi.Counters()
    SA_ref = O.srht_sketch(A, m, seed, c_or)
    assert np.array_equal(SA, SA_ref)
    assert c_gpu.sketch == c_or.sketch


@pytest.mark.parametrize("n,d,m,seed,shards", [
    (1000, 3, 64, 11, 2), (4096, 5, 4096, 2, 2), (3500, 4, 333, 5, 4), (100000, 3, 5000, 7, 8),
    ((1 << 20) - 5, 2, 20000, 1, 8), (1 << 16, 6, 1024, 3, 16), ((1 << 22) - 9, 2, 3000, 4, 2)])
def test_sharded_srht_kernels_bit_exact(gpu, O, n, d, m, seed, shards):
    """The row-sharded SRHT kernels (shard transform + all-gather layout + combine),
    run as P virtual shards on one device, equal the unsharded sketch bit for bit."""
    A = rand_mat(n * d, n, d)
    p = gpu.ProblemInstance(A, np.zeros(n), 1.0)
    SA = gpu.srht_sketch_sharded_emulated(p, m, seed, shards)
    assert np.array_equal(SA, O.srht_sketch(A, m, seed))


def test_srht_sketch_too_large(gpu):
    with pytest.raises(gpu.SketchTooLarge):
        gpu.srht_sketch(np.zeros((12, 2)), 17, 0)
    gpu.srht_sketch(np.zeros((12, 2)), 16, 0)


def test_srht_counter_formula(gpu):
    c16, c256 = gpu.CostCounters(), gpu.CostCounters()
    gpu.srht_sketch(np.zeros((1000, 2)), 16, 0, c16)
    gpu.srht_sketch(np.zeros((1000, 2)), 256, 0, c256)
    fw = 2 * 1024 * 10
    assert c16.sketch == fw + 2 * 1000 + 2 * 16  # test_sketch.cpp:119-126
    assert c256.sketch == fw + 2 * 1000 + 2 * 256


# the last two go through the 128x128 cp.async GEMM (split-K, ragged M/N/K edges)
@pytest.mark.parametrize("n,d,m,seed", [(10, 3, 4, 7), (12, 5, 6, 123), (500, 17, 33, 1), (4096, 64, 256, 2),
                                        (20000, 40, 130, 3), (8192, 130, 256, 4), (5003, 200, 300, 5)])
def test_gaussian_sketch(gpu, O, n, d, m, seed):
    A = rand_mat(seed, n, d)
    c = gpu.CostCounters()
    SA = gpu.gaussian_sketch(A, m, seed, c)
    SA_ref = O.gaussian_sketch(A, m, seed)
    # Eigen GEMM vs DMMA GEMM: different summation order (sketch.hpp:68)
    scale = np.abs(SA_ref).max() + 1e-300
    assert np.max(np.abs(SA - SA_ref)) <= 1e-13 * scale * np.sqrt(n)
    assert c.sketch == m * n * d


def test_gaussian_sketch_deterministic(gpu):
    A = rand_mat(4, 12, 5)
    s1 = gpu.gaussian_sketch(A, 6, 123)
    s2 = gpu.gaussian_sketch(A, 6, 123)
    assert np.array_equal(s1, s2)
    assert np.linalg.norm(s1 - gpu.gaussian_sketch(A, 6, 124)) > 0


# ----------------------------------------------------------------- problem / system
def test_gradient_known_answer(gpu):
    p = gpu.ProblemInstance(np.eye(2), [1.0, 2.0], 1.0)
    g = gpu.gradient(p, [1.0, 1.0])
    np.testing.assert_allclose(g, [1.0, 0.0], atol=1e-15)  # test_problem.cpp:61-65
    c = gpu.CostCounters()
    gpu.gradient(p, [0.0, 0.0], c)
    assert c.matvec == 2 * 2 * 2 + 2 + 2 * 2  # test_problem.cpp:74-78


# even d <= 4096: register-row kernel (1, 2, 4 or 8 column groups per row); odd d: panel kernels
@pytest.mark.parametrize("n,d", [(100, 3), (4096, 64), (65536 + 7, 130), (20000, 1000), (3000, 77), (70000, 512),
                                 (20000 + 3, 1024), (9000, 1538), (5000, 2048), (3001, 3000), (5000, 4096),
                                 (2000, 1001)])
def test_gradient_vs_oracle(gpu, O, n, d):
    A = rand_mat(n, n, d)
    b = RNG(1).standard_normal(n)
    x = RNG(2).standard_normal(d)
    p = gpu.ProblemInstance(A, b, 0.3)
    g = gpu.gradient(p, x)
    g_ref = O.gradient(A, b, 0.3, x)
    assert np.linalg.norm(g - g_ref) <= 1e-12 * (np.linalg.norm(g_ref) + np.linalg.norm(A) * np.linalg.norm(b))


@pytest.mark.parametrize("n,d", [(100, 3), (70000, 512), (5000, 130)])
def test_prediction_error_vs_oracle(gpu, O, n, d):
    A = rand_mat(n + 1, n, d)
    b = RNG(3).standard_normal(n)
    x, xs = RNG(4).standard_normal(d), RNG(5).standard_normal(d)
    p = gpu.ProblemInstance(A, b, 0.3)
    ref = O.prediction_error(A, b, 0.3, x, xs)
    assert abs(gpu.prediction_error(p, x, xs) - ref) <= 1e-12 * ref
    assert gpu.prediction_error(p, x, x) == 0.0
    with pytest.raises(gpu.InvalidInput):
        gpu.prediction_error(p, x[:-1], xs)


def test_system_known_answers(gpu):
    sys = gpu.SketchedSystem.factorize(np.zeros((3, 4)), 2.0)
    g = np.array([4.0, -8.0, 0.0, 2.0])
    np.testing.assert_allclose(sys.solve(g), g / 4.0, atol=1e-14)  # test_sketched_system.cpp:22-26
    SA = np.array([[1.0, 0.0, 0.0]])
    sys = gpu.SketchedSystem.factorize(SA, 1.0)
    assert sys.kind() == gpu.FactorKind.WoodburyInner
    np.testing.assert_allclose(sys.solve(np.ones(3)), [0.5, 1.0, 1.0], rtol=1e-14)


@pytest.mark.parametrize("m,d", [(4, 6), (9, 5), (6, 20), (20, 6), (8, 8), (300, 257), (100, 513), (2000, 700),
                                 # 128x128 DMMA kernels: Gram TN + W^T W (lower tiles, ragged edges), inner NT,
                                 # odd leading dimension (falls back to the 64x64 kernel)
                                 (4096, 512), (5000, 1300), (300, 2048), (1500, 1100), (4095, 300)])
def test_system_solve_vs_oracle(gpu, O, m, d):
    SA = rand_mat(m * d, m, d)
    g = RNG(m + d).standard_normal(d)
    nu = 0.7
    sys = gpu.SketchedSystem.factorize(SA, nu)
    assert sys.kind() == (gpu.FactorKind.WoodburyInner if m < d else gpu.FactorKind.DirectGram)
    z = sys.solve(g)
    H = SA.T @ SA + nu * nu * np.eye(d)
    assert np.linalg.norm(H @ z - g) <= 1e-9 * np.linalg.norm(g) * max(1.0, np.linalg.norm(H, 2) / 10)
    z_ref, kind, ff, fps = O.system_solve(SA, nu, g)
    assert kind == int(sys.kind())
    assert ff == sys.factor_flops() and fps == sys.flops_per_solve()
    assert np.linalg.norm(z - z_ref) <= 1e-10 * np.linalg.norm(z_ref) * max(1.0, np.linalg.cond(H) / 1e3)


def test_system_rejects(gpu):
    SA = np.zeros((2, 3))
    SA[1, 1] = np.inf
    with pytest.raises(gpu.InvalidInput):
        gpu.SketchedSystem.factorize(SA, 1.0)
    with pytest.raises(gpu.InvalidInput):
        gpu.SketchedSystem.factorize(np.zeros((2, 3)), 0.0)


def test_solve_counters(gpu):
    SA = rand_mat(23, 8, 32)
    c = gpu.CostCounters()
    sys = gpu.SketchedSystem.factorize(SA, 1.0, c)
    assert c.factor == 8 * 8 * 32 + 8 * 8 * 8 // 3  # test_sketched_system.cpp:142-150
    sys.solve(np.zeros(32), c)
    assert c.solve == 2 * 8 * 32 + 8 * 8 + 2 * 32


# ----------------------------------------------------------------- adaptive solve
def _cfg_pair(gpu, O, **kw):
    cfg = gpu.SolverConfig(**kw)
    c_or = O.default_config(rho=cfg.rho, eta=cfg.eta, sketch_kind=int(cfg.sketch_kind), mode=int(cfg.mode),
                            m_initial=cfg.m_initial, eps=cfg.eps, max_iters=cfg.max_iters,
                            max_sketch=cfg.max_sketch or 0, seed=cfg.seed,
                            enforce_validity=int(cfg.enforce_validity))
    return cfg, c_or


def _abar_rel(A, nu, x, x_ref):
    Ad = np.concatenate([A @ (x - x_ref), nu * (x - x_ref)])
    Ar = np.concatenate([A @ x_ref, nu * x_ref])
    return np.linalg.norm(Ad) / np.linalg.norm(Ar)


@pytest.mark.parametrize("kind,mode,seed", [("SRHT", "GradientOnly", 0), ("SRHT", "PolyakThenGradient", 1),
                                            ("Gaussian", "PolyakThenGradient", 2), ("Gaussian", "GradientOnly", 3)])
def test_adaptive_solve_matches_oracle(gpu, O, kind, mode, seed):
    A, b, _ = O.synth(2048, 64, decay=0.95, noise_std=0.01, data_seed=seed)
    nu = 1e-2
    cfg, c_or = _cfg_pair(gpu, O, sketch_kind=getattr(gpu.SketchKind, kind), mode=getattr(gpu.SolveMode, mode),
                          seed=seed)
    p = gpu.ProblemInstance(A, b, nu)
    rep = gpu.adaptive_solve(p, cfg)
    x_ref, rep_ref, log_ref, _ = O.adaptive_solve(A, b, nu, c_or)
    assert rep.converged and rep_ref.converged
    # identical m-schedule and branch sequence
    assert rep.rejections == rep_ref.rejections and rep.final_m == rep_ref.final_m
    assert rep.iterations == rep_ref.iterations
    assert [(e.t, e.m, int(e.branch)) for e in rep.log] == [(l[0], l[1], l[4]) for l in log_ref]
    # counters are closed forms of the same evaluations
    assert rep.counters.sketch == rep_ref.counters.sketch
    assert rep.counters.factor == rep_ref.counters.factor
    assert rep.counters.solve == rep_ref.counters.solve
    assert rep.counters.matvec == rep_ref.counters.matvec
    assert _abar_rel(A, nu, rep.x, x_ref) <= 1e-10


# ----------------------------------------------------------------- dual (dual.hpp:13-33)
@pytest.mark.parametrize("kind,rho,n,d,seed", [(0, 0.1, 16, 64, 62), (1, 0.25, 16, 64, 62), (1, 0.25, 12, 48, 63),
                                               (0, 0.15, 100, 700, 5), (1, 0.2, 300, 1000, 6)])
def test_solve_underdetermined_matches_oracle(gpu, O, kind, rho, n, d, seed):
    A, b = O.test_support_data(seed, n, d, n)
    nu = 0.8
    cfg, c_or = _cfg_pair(gpu, O, sketch_kind=gpu.SketchKind(kind), rho=rho, eps=1e-12)
    p = gpu.ProblemInstance(A, b, nu, gpu.Orientation.Underdetermined)
    rep = gpu.solve_underdetermined(p, cfg)
    x_ref, z_ref, rep_ref, log_ref, _ = O.solve_underdetermined(A, b, nu, c_or)
    assert rep.converged == bool(rep_ref.converged)
    assert rep.rejections == rep_ref.rejections and rep.final_m == rep_ref.final_m
    assert rep.iterations == rep_ref.iterations
    assert [(e.t, e.m, int(e.branch)) for e in rep.log] == [(l[0], l[1], l[4]) for l in log_ref]
    assert rep.counters.sketch == rep_ref.counters.sketch and rep.counters.matvec == rep_ref.counters.matvec
    assert rep.counters.factor == rep_ref.counters.factor and rep.counters.solve == rep_ref.counters.solve
    assert rep.dual_final.shape == (n,) and rep.x.shape == (d,)
    np.testing.assert_allclose(rep.x, A.T @ rep.dual_final, rtol=1e-11, atol=1e-11 * np.abs(rep.x).max())
    assert np.linalg.norm(rep.x - x_ref) <= 1e-8 * (1.0 + np.linalg.norm(x_ref))


def test_solve_underdetermined_reference_cases(gpu, O):
    # test_dual.cpp:10-31, 81-87
    p = gpu.ProblemInstance(np.array([[1.0, 1.0]]), [2.0], 1.0, gpu.Orientation.Underdetermined)
    rep = gpu.solve_underdetermined(p, gpu.SolverConfig(eps=1e-14))
    assert rep.converged and np.allclose(rep.x, [2 / 3, 2 / 3], rtol=1e-8) and np.allclose(rep.dual_final, [2 / 3])
    A, _ = O.test_support_data(61, 4, 12)
    p = gpu.ProblemInstance(A, np.zeros(4), 0.5, gpu.Orientation.Underdetermined)
    rep = gpu.solve_underdetermined(p, gpu.SolverConfig())
    assert rep.converged and np.linalg.norm(rep.x) == 0.0
    A, b = O.test_support_data(64, 8, 3, 8)
    with pytest.raises(gpu.InvalidInput):
        gpu.solve_underdetermined(gpu.ProblemInstance(A, b, 1.0), gpu.SolverConfig())
    with pytest.raises(gpu.InvalidInput):
        gpu.adaptive_solve(gpu.ProblemInstance(np.array([[1.0, 1.0]]), [2.0], 1.0, gpu.Orientation.Underdetermined),
                           gpu.SolverConfig())


@pytest.mark.parametrize("n,d,kind,decay,nu", [(8192, 1024, "SRHT", 0.997, 0.5), (3000, 2050, "Gaussian", 0.99, 5.0),
                                               (600000, 8, "SRHT", 0.9, 0.5)])
def test_adaptive_solve_wide_rows_matches_oracle(gpu, O, n, d, kind, decay, nu):
    # d > 512: the register-row gradient with 2 / 8 column groups per row, candidates formed in-kernel
    A, b, _ = O.synth(n, d, decay=decay, noise_std=0.05, data_seed=4)
    cfg, c_or = _cfg_pair(gpu, O, sketch_kind=getattr(gpu.SketchKind, kind), seed=3, rho=0.25,
                          enforce_validity=False)
    rep = gpu.adaptive_solve(gpu.ProblemInstance(A, b, nu), cfg)
    x_ref, rep_ref, log_ref, _ = O.adaptive_solve(A, b, nu, c_or)
    assert rep.converged and rep_ref.converged
    assert (rep.rejections, rep.final_m, rep.iterations) == (rep_ref.rejections, rep_ref.final_m, rep_ref.iterations)
    assert [(e.t, e.m, int(e.branch)) for e in rep.log] == [(l[0], l[1], l[4]) for l in log_ref]
    assert _abar_rel(A, nu, rep.x, x_ref) <= 1e-10


def test_adaptive_solve_deterministic(gpu, O):
    A, b, _ = O.synth(1024, 32, decay=0.95, data_seed=9)
    p = gpu.ProblemInstance(A, b, 0.2)
    cfg = gpu.SolverConfig(rho=0.15, seed=7)
    a = gpu.adaptive_solve(p, cfg)
    c = gpu.adaptive_solve(p, cfg)
    assert a.iterations == c.iterations and a.rejections == c.rejections
    assert np.array_equal(a.x, c.x)
    assert [e.r for e in a.log] == [e.r for e in c.log]


def test_adaptive_solve_zero_rhs(gpu):
    A = rand_mat(52, 10, 3)
    p = gpu.ProblemInstance(A, np.zeros(10), 1.0)
    rep = gpu.adaptive_solve(p, gpu.SolverConfig(sketch_kind=gpu.SketchKind.Gaussian, rho=0.1))
    assert rep.converged and rep.iterations == 1 and rep.r1 == 0.0 and np.linalg.norm(rep.x) == 0.0


def test_adaptive_solve_validates(gpu):
    A = rand_mat(53, 6, 3)
    p = gpu.ProblemInstance(A, RNG(1).standard_normal(6), 1.0)
    with pytest.raises(gpu.InvalidInput):
        gpu.adaptive_solve(p, gpu.SolverConfig(eps=0.0))
    with pytest.raises(gpu.OutOfValidityRange):
        gpu.adaptive_solve(p, gpu.SolverConfig(rho=0.5))
    gpu.adaptive_solve(p, gpu.SolverConfig(rho=0.5, enforce_validity=False))


def test_sketch_exhaustion_flagged(gpu, O):
    A = rand_mat(54, 4, 2)
    b = RNG(54).standard_normal(4)
    p = gpu.ProblemInstance(A, b, 0.5)
    cfg = gpu.SolverConfig(tuning_override=gpu.rates_from_bounds(1.0, 1.0), eps=1e-12, max_iters=40)
    rep = gpu.adaptive_solve(p, cfg)
    assert rep.sketch_exhausted and rep.final_m <= 4


def test_fixed_sketch_ihs_matches_oracle(gpu, O):
    A, b, _ = O.synth(4096, 32, decay=0.95, data_seed=4)
    nu = 0.05
    SA = O.gaussian_sketch(A, 128, 5)
    tp = gpu.rates_from_bounds(*gpu.gaussian_targets(0.3, 0.01, False))
    p = gpu.ProblemInstance(A, b, nu)
    sys = gpu.SketchedSystem.factorize(SA, nu)
    its = gpu.fixed_sketch_ihs(p, sys, tp, 25, gpu.FixedMode.Polyak)
    ref = O.fixed_sketch_ihs(A, b, nu, SA, O.abi.Tuning(**tp.__dict__), 25, 1)
    # x_0 = 0 on both sides exactly; every later iterate within 1e-9 in the Abar norm
    assert np.array_equal(its[0], np.zeros(32)) and np.array_equal(ref[0], np.zeros(32))
    for k in range(1, 26):
        assert _abar_rel(A, nu, its[k], ref[k]) <= 1e-9


# ----------------------------------------------------------------- NCCL plumbing
@pytest.mark.gpu
def test_nccl_single_rank_communicator(gpu):
    """libnccl is loaded at run time and a communicator initialises (1 rank on cuda:0): the
    plumbing of the row-sharded path; the multi-rank exchange itself is covered by the
    emulated-shard tests above and by tests/test_multirank_gloo.py."""
    uid = gpu.nccl_unique_id()
    assert len(uid) == 128
    comm = gpu.NcclComm(uid, 1, 0, 0)
    assert comm.handle
    del comm


# n_pad = 2^18 .. 2^22 (8 .. 12 high bits): ragged n (partial and virtual chunks), d above the L2-resident
# launch's ring depth, sparse and dense tile occupancy
@pytest.mark.parametrize("n,d,m,seed", [((1 << 18) + 7, 9, 5000, 21), ((1 << 19) - 1, 6, 300, 22),
                                        ((1 << 20) - 3, 11, 30000, 23), ((1 << 21) + 3, 5, 70000, 24),
                                        ((1 << 22) - 3, 4, 131072, 25), ((1 << 22), 3, 9, 26)])
def test_srht_l2_resident_bit_exact(gpu, O, n, d, m, seed):
    A = rand_mat(seed, n, d)
    assert np.array_equal(gpu.srht_sketch(A, m, seed), O.srht_sketch(A, m, seed))


def test_srht_l2_ring_depths_and_two_kernel_path_agree(gpu):
    """The L2-resident launch (default for 10..12 high bits; IHS_SRHT_L2=1 also takes 9) at ring depths 2 and 3
    (every slot reused), with sparse tiles at n_pad = 2^20 (compact T disabled), at 2^19, 2^21 and 2^22 rows, and
    the two-kernel path (IHS_SRHT_L2=0) all give the oracle's bytes."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "from oracle import oracle as O\n"
            "rng = np.random.default_rng(10)\n"
            "A = np.asfortranarray(rng.standard_normal(((1 << 20) - 77, 7)))\n"
            "for m in (5, 900, 40000):\n"
            "    assert np.array_equal(ihs.srht_sketch(A, m, 3 + m), O.srht_sketch(A, m, 3 + m)), m\n"
            "B = np.asfortranarray(rng.standard_normal(((1 << 22) - 3, 3)))\n"
            "for m in (9, 131072):\n"
            "    assert np.array_equal(ihs.srht_sketch(B, m, 4 + m), O.srht_sketch(B, m, 4 + m)), m\n"
            "C = np.asfortranarray(rng.standard_normal(((1 << 19) - 5, 5)))\n"
            "D = np.asfortranarray(rng.standard_normal(((1 << 21) + 9, 3)))\n"
            "for X, m in ((C, 300), (C, 60000), (D, 70000)):\n"
            "    assert np.array_equal(ihs.srht_sketch(X, m, 5 + m), O.srht_sketch(X, m, 5 + m)), m\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    for extra in ({"IHS_SRHT_L2": "1", "IHS_SRHT_L2_NS": "2"},
                  {"IHS_SRHT_L2": "1", "IHS_SRHT_L2_NS": "3", "IHS_SRHT_NO_COMPACT": "1"}, {"IHS_SRHT_L2": "0"}, {}):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, (extra, r.stderr[-2000:])


def test_srht_l2_concurrent_problems(gpu, O):
    """Two problems sketching at once from two host threads (two streams): the L2-resident launches, whose CTAs
    wait on each other, are chained on the device and never share it — no hang, both bit-exact."""
    import threading
    rng = np.random.default_rng(12)
    mats = [np.asfortranarray(rng.standard_normal(((1 << 20) - 3, 6))) for _ in range(2)]
    probs = [gpu.ProblemInstance(M, np.zeros(M.shape[0]), 1e-2) for M in mats]
    out, err = [None, None], []

    def work(i):
        try:
            out[i] = [gpu.srht_sketch(probs[i], 30000 + 7 * k, 40 + k) for k in range(4)]
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th) and not err, err
    for i in range(2):
        for k in range(4):
            assert np.array_equal(out[i][k], O.srht_sketch(mats[i], 30000 + 7 * k, 40 + k))


def test_srht_column_batches_bit_exact(gpu):
    """Sketches whose phase-1 scratch exceeds the cap run over column batches (C4 at 2^22 rows): with a
    1 MiB cap a 2^15-row problem runs 4 columns per batch and must stay bit-exact."""
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "from oracle import oracle as O\n"
            "rng = np.random.default_rng(7)\n"
            "A = np.asfortranarray(rng.standard_normal(((1 << 15) - 5, 10)))\n"
            "for m in (3, 700):\n"
            "    assert np.array_equal(ihs.srht_sketch(A, m, 11 + m), O.srht_sketch(A, m, 11 + m)), m\n"
            "print('ok')\n")
    import os
    env = dict(os.environ, IHS_SRHT_SCRATCH_CAP_MB="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_srht_compact_modes_bit_exact(gpu):
    """Compact T (n_pad = 2^20, few distinct low indices) is forced for every sample size, and also combined
    with column batches (8 MiB cap = one column per batch): the sketches stay bit-exact."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "from oracle import oracle as O\n"
            "rng = np.random.default_rng(8)\n"
            "A = np.asfortranarray(rng.standard_normal(((1 << 20) - 9, 3)))\n"
            "for m in (2, 300, 2500):\n"
            "    assert np.array_equal(ihs.srht_sketch(A, m, 5 + m), O.srht_sketch(A, m, 5 + m)), m\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    for extra in ({}, {"IHS_SRHT_SCRATCH_CAP_MB": "8"}):
        env = dict(os.environ, IHS_SRHT_COMPACT_MAX="1024", **extra)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_srht_three_round_pass_column_batches_bit_exact(gpu):
    """n_pad = 2^22 (one 12-bit emitting pass of three-round tiles) over column batches (40 MiB cap = one
    32 MiB column per batch), as C4 runs it: bit-exact."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "from oracle import oracle as O\n"
            "rng = np.random.default_rng(9)\n"
            "A = np.asfortranarray(rng.standard_normal(((1 << 22) - 3, 3)))\n"
            "for m in (7, 500):\n"
            "    assert np.array_equal(ihs.srht_sketch(A, m, 2 + m), O.srht_sketch(A, m, 2 + m)), m\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    env = dict(os.environ, IHS_SRHT_SCRATCH_CAP_MB="40")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_gaussian_streamed_sketch_matches(gpu):
    """The streamed Gaussian sketch (S generated in chunks of jump-ahead substreams with a carried
    acceptance count, consumed in column blocks by an accumulating GEMM; forced here with one 2^22-draw
    substream per chunk and 64-column blocks) equals the oracle's materialised sketch to fp64 tolerance,
    and an adaptive solve through it takes the same m-schedule."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "from oracle import oracle as O\n"
            "rng = np.random.default_rng(10)\n"
            "A = np.asfortranarray(rng.standard_normal((40000, 6)))\n"
            "for m in (1, 300):\n"
            "    SA, ref = ihs.gaussian_sketch(A, m, 3 + m), O.gaussian_sketch(A, m, 3 + m)\n"
            "    assert np.max(np.abs(SA - ref)) <= 1e-12 * np.abs(ref).max(), m\n"
            "A, b, _ = O.synth(30000, 24, decay=0.9, noise_std=0.05, data_seed=3)\n"
            "cfg = ihs.SolverConfig(seed=4)\n"
            "r = ihs.adaptive_solve(ihs.ProblemInstance(A, b, 0.2), cfg)\n"
            "x, rep, log, _ = O.adaptive_solve(A, b, 0.2, O.default_config(seed=4))\n"
            "assert (r.iterations, r.rejections, r.final_m) == (rep.iterations, rep.rejections, rep.final_m)\n"
            "assert np.linalg.norm(r.x - x) <= 1e-9 * (1 + np.linalg.norm(x))\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    for extra in ({}, {"IHS_GAUSS_MAX_JUMP_SUBS": "3"}):
        env = dict(os.environ, IHS_GAUSS_STREAM="1", IHS_GAUSS_STREAM_COLS="64", **extra)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env,
                           cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, (extra, r.stderr[-3000:])


@pytest.mark.parametrize("streamed", [False, True])
def test_fill_gaussian_window(gpu, streamed):
    """A row shard's window of the normal stream (sharded Gaussian sketch: normals [row0 m, (row0 + n_loc) m)),
    emitted at once or in blocks (the streamed sketch's scheme), equals the slice of the full stream."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "full = ihs.fill_gaussian(12345, 7000000, 1, 0.5).reshape(-1)\n"
            f"streamed = {streamed}\n"
            "for first, count in ((0, 1000), (1, 999), (3000001, 2500000), (6999990, 10), (0, 1), (4321, 1),\n"
            "                     (6999999, 1)):\n"
            "    w = ihs.fill_gaussian_window(12345, first, count, 0.5, streamed, 4097)\n"
            "    assert np.array_equal(w, full[first:first + count]), (first, count)\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    # default plan (emitting substreams = jump substreams) and a forced two-level plan (4 jump substreams, each
    # dumping the windows of its emitting substreams), the one long streams take
    for extra in ({}, {"IHS_GAUSS_MAX_JUMP_SUBS": "4"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root,
                           env=dict(os.environ, **extra))
        assert r.returncode == 0 and "ok" in r.stdout, (extra, r.stderr[-3000:])
