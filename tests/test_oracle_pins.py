"""Pin the CPU oracle against every known answer the reference's own tests hold
for the hot path (proj/tests/test_sketch.cpp, test_sketched_system.cpp,
test_problem.cpp, test_tuning.cpp, test_solver.cpp) plus the C++ standard's
mt19937_64 known answer, and against the committed golden fixtures.
CPU only."""
import numpy as np
import pytest

RNG = np.random.default_rng


# ------------------------------------------------------------ rng.hpp
def test_mt19937_64_standard_known_answer(O):
    # [rand.predef]: 10000th invocation of a default-constructed mt19937_64
    assert int(O.mt_raw(5489, 10000)[-1]) == 9981545732273789042


def test_derive_seed_is_two_splitmix_steps(O):
    def splitmix(s):
        s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return s, z ^ (z >> 31)

    for seed, tag in [(0, 0), (1, 2), (2**63, 7), (12345, 1000)]:
        s = (seed + 0x632BE59BD9B4E019 * (tag + 1)) & (2**64 - 1)
        s, a = splitmix(s)
        s, b = splitmix(s)
        assert O.derive_seed(seed, tag) == a ^ ((b << 1) & (2**64 - 1))


def test_sampling_without_replacement(O):
    # test_sketch.cpp:129-138
    for rep in range(5):
        idx = np.sort(O.sample_without_replacement(O.derive_seed(7, rep), 128, 100))
        assert np.all(np.diff(idx) > 0) and idx[0] >= 0 and idx[-1] < 128


# ------------------------------------------------------------ sketch.hpp
def test_fwht_known_answers(O):
    v = O.fwht_inplace(np.array([1.0, 0.0, 0.0, 0.0]))
    assert np.all(v == 0.5)  # test_sketch.cpp:13-17
    x = RNG(2).standard_normal(64)
    w = O.fwht_inplace(x)
    assert abs(np.linalg.norm(w) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert np.max(np.abs(O.fwht_inplace(w) - x)) <= 1e-12  # involution :18-26
    with pytest.raises(O.OracleError):
        O.fwht_inplace(np.zeros(12))  # :27-32


def test_next_pow2(O):
    assert [O.next_pow2(k) for k in (1, 2, 3, 1000, 1024)] == [1, 2, 4, 1024, 1024]


def test_gaussian_sketch_properties(O):
    assert np.linalg.norm(O.gaussian_sketch(np.zeros((10, 3)), 4, 7)) == 0.0
    A = np.asfortranarray(RNG(4).standard_normal((12, 5)))
    assert np.array_equal(O.gaussian_sketch(A, 6, 123), O.gaussian_sketch(A, 6, 123))
    assert np.linalg.norm(O.gaussian_sketch(A, 6, 123) - O.gaussian_sketch(A, 6, 124)) > 0
    # S*A equals the materialized S times A (test_sketch.cpp:47-53)
    S = O.gaussian_sketch(np.eye(10), 3, 55)
    A = np.asfortranarray(RNG(9).standard_normal((10, 4)))
    assert np.max(np.abs(S @ A - O.gaussian_sketch(A, 3, 55))) <= 1e-14
    # S is make_stream(seed, 0) filled column-major with stddev 1/sqrt(m)
    S_direct = O.fill_gaussian(O.derive_seed(55, 0), 3, 10, 1.0 / np.sqrt(3.0))
    assert np.array_equal(S, S_direct)
    c = O.abi.Counters()
    O.gaussian_sketch(np.zeros((10, 3)), 4, 7, c)
    assert c.sketch == 4 * 10 * 3  # :74-78


def test_srht_sketch_properties(O):
    assert np.linalg.norm(O.srht_sketch(np.zeros((10, 3)), 4, 7)) == 0.0
    S = O.srht_sketch(np.eye(16), 16, 3)
    assert np.linalg.norm(S.T @ S - np.eye(16), 2) <= 1e-10  # :85-89
    A = np.asfortranarray(RNG(17).standard_normal((12, 4)))
    SA = O.srht_sketch(A, 8, 77)
    S = O.srht_sketch(np.eye(12), 8, 77)
    assert np.max(np.abs(S @ A - SA)) <= 1e-12  # :102-108
    with pytest.raises(O.OracleError) as e:
        O.srht_sketch(np.zeros((12, 2)), 17, 0)
    assert e.value.status == O.abi.IHS_SKETCH_TOO_LARGE
    O.srht_sketch(np.zeros((12, 2)), 16, 0)
    A = np.asfortranarray(RNG(6).standard_normal((20, 3)))
    assert np.array_equal(O.srht_sketch(A, 8, 42), O.srht_sketch(A, 8, 42))
    assert np.linalg.norm(O.srht_sketch(A, 8, 42) - O.srht_sketch(A, 8, 43)) > 0
    c16, c256 = O.abi.Counters(), O.abi.Counters()
    O.srht_sketch(np.zeros((1000, 2)), 16, 0, c16)
    O.srht_sketch(np.zeros((1000, 2)), 256, 0, c256)
    assert c16.sketch == 2 * 1024 * 10 + 2 * 1000 + 2 * 16  # :119-126
    assert c256.sketch == 2 * 1024 * 10 + 2 * 1000 + 2 * 256


def test_srht_definition_from_streams(O):
    """SA = sqrt(n_pad/m) * R H D A spelled out with numpy from the oracle's D and P."""
    n, d, m, seed = 100, 3, 20, 5
    A = np.asfortranarray(RNG(1).standard_normal((n, d)))
    SA = O.srht_sketch(A, m, seed)
    n_pad = 128
    eps = O.rademacher(O.derive_seed(seed, 1), n_pad)
    rows = O.sample_without_replacement(O.derive_seed(seed, 2), n_pad, m)
    B = np.zeros((n_pad, d))
    B[:n] = eps[:n, None] * A
    for j in range(d):
        B[:, j] = O.fwht_inplace(B[:, j].copy())
    ref = np.sqrt(n_pad / m) * B[rows]
    assert np.array_equal(SA, ref)


# ------------------------------------------------------------ problem / system / tuning
def test_gradient_known_answers(O):
    A = np.eye(2)
    b = np.array([1.0, 2.0])
    np.testing.assert_allclose(O.gradient(A, b, 1.0, [1.0, 1.0]), [1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(O.gradient(A, b, 1.0, [0.0, 0.0]), -b, atol=1e-15)
    c = O.abi.Counters()
    O.gradient(A, b, 1.0, [0.0, 0.0], c)
    assert c.matvec == 2 * 2 * 2 + 2 + 2 * 2


def test_direct_solve_known_answer(O):
    np.testing.assert_allclose(O.direct_solve(np.eye(2), [1.0, 2.0], 1.0), [0.5, 1.0], rtol=1e-12)


def test_system_known_answers(O):
    g = np.array([4.0, -8.0, 0.0, 2.0])
    z, kind, _, _ = O.system_solve(np.zeros((3, 4)), 2.0, g)
    np.testing.assert_allclose(z, g / 4.0, atol=1e-14)
    z, kind, _, _ = O.system_solve(np.array([[1.0, 0.0, 0.0]]), 1.0, np.ones(3))
    assert kind == O.abi.FACTOR_WOODBURY_INNER
    np.testing.assert_allclose(z, [0.5, 1.0, 1.0], rtol=1e-14)
    _, kind, _, _ = O.system_solve(RNG(0).standard_normal((5, 5)), 1.0)
    assert kind == O.abi.FACTOR_DIRECT_GRAM
    _, kind, _, _ = O.system_solve(RNG(0).standard_normal((4, 5)), 1.0)
    assert kind == O.abi.FACTOR_WOODBURY_INNER
    c = O.abi.Counters()
    O.system_solve(RNG(23).standard_normal((8, 32)), 1.0, np.zeros(32), c)
    assert c.factor == 8 * 8 * 32 + 8 * 8 * 8 // 3 and c.solve == 2 * 8 * 32 + 8 * 8 + 2 * 32
    with pytest.raises(O.OracleError):
        O.newton_decrement(np.ones(3), -np.ones(3))


@pytest.mark.parametrize("m,d", [(6, 20), (20, 6), (8, 8)])
def test_system_residual(O, m, d):
    SA = RNG(16).standard_normal((m, d))
    g = RNG(17).standard_normal(d)
    z, _, _, _ = O.system_solve(SA, 0.3, g)
    H = SA.T @ SA + 0.09 * np.eye(d)
    assert np.linalg.norm(H @ z - g) <= 1e-8 * np.linalg.norm(g)


def test_tuning_known_answers(O):
    t = O.rates_from_bounds(0.5, 2.0)
    assert abs(t.mu_gd - 0.8) <= 1e-14 and abs(t.c_gd - 0.36) <= 1e-14  # test_tuning.cpp:18-22
    lam, Lam = O.gaussian_targets(0.1, 0.01)
    assert abs(lam - 0.34681) <= 1e-4 * 0.34681 and abs(Lam - 1.99119) <= 1e-4 * 1.99119
    lam, Lam = O.srht_targets(0.04)
    assert abs(lam - 0.8) <= 1e-14 and abs(Lam - 1.2) <= 1e-14
    for rho in np.arange(0.01, 1.0, 0.01):
        l, L = O.srht_targets(rho)
        assert abs(O.rates_from_bounds(l, L).c_gd - rho) <= 1e-14
    with pytest.raises(O.OracleError) as e:
        O.gaussian_targets(0.19, 0.01)
    assert e.value.status == O.abi.IHS_OUT_OF_VALIDITY_RANGE


# ------------------------------------------------------------ solver.hpp
def test_adaptive_zero_rhs(O):
    A = np.asfortranarray(RNG(52).standard_normal((10, 3)))
    x, rep, log, _ = O.adaptive_solve(A, np.zeros(10), 1.0, O.default_config())
    assert rep.converged and rep.iterations == 1 and rep.r1 == 0.0 and np.linalg.norm(x) == 0.0


def test_adaptive_audit_trail(O):
    A, b, _ = O.synth(512, 16, decay=0.95, data_seed=4)
    for seed in range(5):
        x, rep, log, _ = O.adaptive_solve(A, b, 0.1, O.default_config(seed=seed))
        assert rep.converged
        acc = sum(1 for l in log if l[4] != O.abi.STEP_RESKETCH)
        res = sum(1 for l in log if l[4] == O.abi.STEP_RESKETCH)
        assert acc == rep.iterations - 1 and res == rep.rejections
        assert rep.final_m == 1 << rep.rejections
        assert rep.r_final <= 1e-10 * rep.r1
        ms = [l[1] for l in log]
        assert ms == sorted(ms)


def test_adaptive_error_transfer(O):
    # r_T <= eps * r_1 is the reference's stopping rule (solver.hpp:154,177); r_1 is
    # measured under the m = 1 sketch, so it bounds delta only through the final
    # sketch's spectrum: delta_T <= gamma_1(C_S) r_T (test_solver.cpp:240-276).
    A, b, _ = O.synth(2048, 32, decay=0.95, data_seed=8)
    nu = 0.05
    x_star = O.direct_solve(A, b, nu)
    for kind in (O.abi.SKETCH_GAUSSIAN, O.abi.SKETCH_SRHT):
        x, rep, _, _ = O.adaptive_solve(A, b, nu, O.default_config(sketch_kind=kind))
        assert rep.converged and rep.r_final <= 1e-10 * rep.r1
        assert O.prediction_error(A, b, nu, x, x_star) <= 2.0 * rep.r_final


def test_synth_spectrum(O):
    A, b, xt = O.synth(4096, 8, decay=0.5, noise_std=0.0, data_seed=1)
    col = np.linalg.norm(A, axis=0) / np.sqrt(4096)
    np.testing.assert_allclose(col, 0.5 ** np.arange(1, 9), rtol=0.05)
    np.testing.assert_array_equal(b, np.array([sum(A[i, j] * xt[j] for j in range(8)) for i in range(4096)]))


# ------------------------------------------------------------ dual.hpp (test_dual.cpp, with the reference tests'
# own data: support.hpp's random_matrix / random_vector replayed by O.test_support_data)
def _ridge_kernel_form(A, b, nu):
    return A.T @ np.linalg.solve(A @ A.T + nu * nu * np.eye(A.shape[0]), b)


def test_dual_hand_example(O):  # test_dual.cpp:10-22
    x, z, rep, log, _ = O.solve_underdetermined(np.array([[1.0, 1.0]]), np.array([2.0]), 1.0,
                                                O.default_config(eps=1e-14))
    assert rep.converged
    assert abs(x[0] - 2 / 3) <= 1e-8 * 2 / 3 and abs(x[1] - 2 / 3) <= 1e-8 * 2 / 3
    assert z.shape == (1,) and abs(z[0] - 2 / 3) <= 1e-8 * 2 / 3


def test_dual_zero_observations(O):  # test_dual.cpp:24-31
    A, _ = O.test_support_data(61, 4, 12)
    x, z, rep, log, _ = O.solve_underdetermined(A, np.zeros(4), 0.5, O.default_config())
    assert rep.converged and np.linalg.norm(x) == 0.0


@pytest.mark.parametrize("kind,rho", [(0, 0.1), (1, 0.25)])
def test_dual_matches_kernel_form(O, kind, rho):  # test_dual.cpp:33-56
    A, b = O.test_support_data(62, 16, 64, 16)
    x_ref = _ridge_kernel_form(A, b, 0.8)
    x, z, rep, log, _ = O.solve_underdetermined(A, b, 0.8, O.default_config(eps=1e-18, sketch_kind=kind, rho=rho))
    assert rep.converged and rep.final_m <= 64
    assert np.linalg.norm(x - x_ref) <= 1e-8 * (1.0 + np.linalg.norm(x_ref))
    # counters: the dual gradient's 2nd + d + 2n per evaluation (dual.hpp:23-27)
    evals = rep.iterations + sum(1 for l in log if l[4] == O.abi.STEP_RESKETCH)
    assert rep.counters.matvec % (2 * 16 * 64 + 64 + 2 * 16) == 0


def test_dual_transfer_bound(O):  # test_dual.cpp:58-79
    A, b = O.test_support_data(63, 12, 48, 12)
    nu = 0.9
    x_ref = _ridge_kernel_form(A, b, nu)
    x, z, rep, log, _ = O.solve_underdetermined(A, b, nu, O.default_config(eps=1e-12, sketch_kind=1, rho=0.25))
    assert rep.converged
    sigma1 = np.linalg.svd(A, compute_uv=False)[0]
    f_star = 0.5 * np.linalg.norm(A @ x_ref - b) ** 2 + 0.5 * nu * nu * np.linalg.norm(x_ref) ** 2
    bound = 10.0 * np.sqrt(2.0 * 1e-12 * f_star) * sigma1 / (nu * nu)
    assert np.linalg.norm(x - x_ref) / (1.0 + np.linalg.norm(x_ref)) <= bound


def test_dual_rejects_overdetermined(O):  # test_dual.cpp:81-87
    A, b = O.test_support_data(64, 8, 3, 8)
    with pytest.raises(O.OracleError) as e:
        O.solve_underdetermined(A, b, 1.0, O.default_config())
    assert e.value.status == O.abi.IHS_INVALID_INPUT
