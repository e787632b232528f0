"""GPU parity of the CG / sketch-preconditioned CG baselines (baselines.hpp:40-200)
against the CPU oracle, through the C-ABI (ihs_gpu_cg_solve / ihs_gpu_pcg_solve_with /
ihs_gpu_pcg_solve). The reference's own cases (test_baselines.cpp) run on the device,
and every run is compared with the oracle on the same inputs: identical iteration
counts, counters, sketch sizes and convergence flags; iterates and residual traces
within fp64 tolerance (the reductions' summation order differs from the oracle's).
"""
import math

import numpy as np
import pytest

from test_oracle_baselines import exp_instance, orthogonal_sketch

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng


def counters_eq(a, b):
    return (a.sketch, a.factor, a.solve, a.matvec) == (int(b.sketch), int(b.factor), int(b.solve), int(b.matvec))


def np_trace(A, b, nu, tol, max_iters, SA=None, x0=None):
    """An independent fp64 restatement of baselines.hpp's CG / PCG loop on numpy BLAS (different
    summation order from the oracle), used only to measure how far the instance's residual trace
    is reproducible across implementations."""
    import scipy.linalg as sl

    d = A.shape[1]
    H = lambda v: A.T @ (A @ v) + nu * nu * v  # noqa: E731
    if SA is not None:
        L = np.linalg.cholesky(SA.T @ SA + nu * nu * np.eye(d))
        Minv = lambda v: sl.solve_triangular(L.T, sl.solve_triangular(L, v, lower=True), lower=False)  # noqa: E731
    atb = A.T @ b
    target = tol * np.linalg.norm(atb)
    x = np.zeros(d) if x0 is None else np.array(x0, dtype=float)
    r = atb - H(x)
    res = [np.linalg.norm(r)]
    if res[0] <= target:
        return np.array(res)
    z = Minv(r) if SA is not None else r
    p, rz = z.copy(), r @ z
    for _ in range(max_iters):
        hp = H(p)
        alpha = rz / (p @ hp)
        x, r = x + alpha * p, r - alpha * hp
        res.append(np.linalg.norm(r))
        if res[-1] <= target:
            break
        z = Minv(r) if SA is not None else r
        rz_new = r @ z
        p, rz = z + (rz_new / rz) * p, rz_new
    return np.array(res)


def check_vs_oracle(r, xo, reso, repo, inst, xtol=1e-9, rtol=1e-6):
    """Parity with the oracle on the same inputs. CG's recurrence amplifies rounding differences, so
    two correct fp64 implementations (the oracle, numpy's BLAS, the reference's Eigen build) share
    their residual trace only up to an instance-dependent horizon: it is measured here against
    np_trace (first iteration where numpy and the oracle differ by more than 1e-8 relative). The
    device trace must match the oracle's within rtol up to that horizon; when the horizon covers the
    whole trace the iteration count and counters must be identical, otherwise the stopping iteration
    may differ by up to 2 (the counters then follow the reference's formulas for the iterations
    taken). The final iterate must agree within xtol either way."""
    A, b, nu, tol, max_iters = inst[:5]
    SA = inst[5] if len(inst) > 5 else None
    x0 = inst[6] if len(inst) > 6 else None
    resn = np_trace(A, b, nu, tol, max_iters, SA, x0)
    k = min(len(resn), len(reso))
    bad = np.nonzero(np.abs(resn[:k] - reso[:k]) > 1e-8 * reso[:k])[0]
    horizon = int(bad[0]) if bad.size else k
    exact = horizon == len(reso) == len(resn)
    assert r.converged == bool(repo.converged)
    assert abs(r.iterations - repo.iterations) <= (0 if exact else 2)
    assert len(r.residuals) == r.iterations + 1 and len(reso) == repo.iterations + 1
    h = min(horizon, len(r.residuals))
    np.testing.assert_allclose(r.residuals[:h], reso[:h], rtol=rtol)
    assert (r.counters.sketch, r.counters.factor) == (int(repo.counters.sketch), int(repo.counters.factor))
    if r.iterations == repo.iterations:
        assert counters_eq(r.counters, repo.counters)
    else:
        per_hv = int(repo.counters.matvec) // (repo.iterations + 1)
        assert r.counters.matvec == per_hv * (r.iterations + 1)
    assert np.linalg.norm(r.x - xo) <= xtol * (1 + np.linalg.norm(xo))
    return horizon


# ---------------------------------------------------------------- cg_solve
def test_cg_identity_instance(gpu, O):  # test_baselines.cpp:11-19
    p = gpu.ProblemInstance(np.eye(2), np.array([1.0, 2.0]), 1.0)
    r = gpu.cg_solve(p, 1e-12, 10)
    assert r.converged and r.iterations <= 2
    assert r.x == pytest.approx([0.5, 1.0], rel=1e-10)
    check_vs_oracle(r, *O.cg_solve(np.eye(2), np.array([1.0, 2.0]), 1.0, 1e-12, 10),
                    (np.eye(2), np.array([1.0, 2.0]), 1.0, 1e-12, 10))
    assert r.kernel_launches > 0 and r.device_ms > 0


def test_cg_start_at_solution(gpu, O):  # :20-28
    A, b = O.test_support_data(71, 12, 4, 12)
    xs = O.direct_solve(A, b, 0.6)
    r = gpu.cg_solve(gpu.ProblemInstance(A, b, 0.6), 1e-10, 50, x0=xs)
    assert r.converged and r.iterations == 0 and len(r.residuals) == 1
    assert r.counters.matvec == 2 * 12 * 4 + 2 * 4


def test_cg_matches_direct(gpu, O):  # :29-37
    A, b = O.test_support_data(72, 30, 6, 30)
    r = gpu.cg_solve(gpu.ProblemInstance(A, b, 1.0), 1e-12, 200)
    assert r.converged
    assert np.linalg.norm(r.x - O.direct_solve(A, b, 1.0)) <= 1e-10 * (1 + np.linalg.norm(r.x))
    check_vs_oracle(r, *O.cg_solve(A, b, 1.0, 1e-12, 200), (A, b, 1.0, 1e-12, 200))


def test_cg_energy_error_non_increasing(gpu, O):  # :38-49
    A, b = exp_instance(48, 10, 5)
    xs = O.direct_solve(A, b, 0.2)
    p = gpu.ProblemInstance(A, b, 0.2)
    prev = math.inf
    for k in range(13):
        r = gpu.cg_solve(p, 0.0, k)
        assert r.iterations == k and not r.converged
        delta = gpu.prediction_error(p, r.x, xs)
        assert delta <= prev * (1 + 1e-10)
        prev = delta
        check_vs_oracle(r, *O.cg_solve(A, b, 0.2, 0.0, k), (A, b, 0.2, 0.0, k), xtol=1e-8)


def test_cg_not_converged_flag(gpu, O):  # :50-56
    A, b = O.test_support_data(73, 40, 20, 40)
    r = gpu.cg_solve(gpu.ProblemInstance(A, b, 1e-3), 1e-14, 1)
    assert not r.converged and r.iterations == 1
    check_vs_oracle(r, *O.cg_solve(A, b, 1e-3, 1e-14, 1), (A, b, 1e-3, 1e-14, 1))


@pytest.mark.parametrize("max_iters", [0, 1, 15, 16, 17, 33, 100])
def test_cg_batch_boundaries(gpu, O, max_iters):
    # iterations are enqueued in batches of up to 16 between state read-backs: runs that stop at, just
    # before and just after a batch boundary, and one that converges inside a batch (iteration 56),
    # keep the reference's iteration count, trace and counters (well conditioned, cond(H) ~ 36, and
    # converging long before d = 160; numpy and the oracle agree to 1e-8 over the first 48 residuals)
    A = np.asfortranarray(RNG(80).standard_normal((1200, 160)) * (0.99 ** np.arange(160)))
    b = RNG(81).standard_normal(1200)
    r = gpu.cg_solve(gpu.ProblemInstance(A, b, 1.0), 1e-9, max_iters)
    xo, reso, repo = O.cg_solve(A, b, 1.0, 1e-9, max_iters)
    assert max_iters < 56 or (repo.converged and repo.iterations == 56)
    h = check_vs_oracle(r, xo, reso, repo, (A, b, 1.0, 1e-9, max_iters))
    assert h >= min(len(reso), 40)  # most of the trace is reproducible on this instance


def test_cg_warm_start(gpu, O):
    A, b = O.test_support_data(79, 200, 16, 200)
    x0 = RNG(3).standard_normal(16)
    r = gpu.cg_solve(gpu.ProblemInstance(A, b, 0.3), 1e-11, 100, x0=x0)
    check_vs_oracle(r, *O.cg_solve(A, b, 0.3, 1e-11, 100, x0=x0), (A, b, 0.3, 1e-11, 100, None, x0))


def test_cg_errors(gpu, O):
    A, b = O.test_support_data(77, 3, 5, 3)
    p = gpu.ProblemInstance(A, b, 0.5, orientation=gpu.Orientation.Underdetermined)
    with pytest.raises(gpu.InvalidInput, match="overdetermined"):
        gpu.cg_solve(p, 1e-8, 5)
    with pytest.raises(gpu.InvalidInput, match="overdetermined"):
        gpu.pcg_solve(p, gpu.SketchKind.Gaussian, 1, 0.5, 1e-8, 5)
    q = gpu.ProblemInstance(*O.test_support_data(78, 8, 3, 8), 0.5)
    with pytest.raises(gpu.InvalidInput):
        gpu.cg_solve(q, 1e-8, 5, x0=np.zeros(2))
    with pytest.raises(gpu.InvalidInput, match="rho"):
        gpu.pcg_solve(q, gpu.SketchKind.Gaussian, 1, 1.0, 1e-8, 5)


# ---------------------------------------------------------------- pcg_solve
def test_pcg_exact_preconditioner_one_iteration(gpu, O):  # :60-70
    A, b = O.test_support_data(74, 16, 5, 16)
    SA = orthogonal_sketch(A, 4)
    r = gpu.pcg_solve_with(gpu.ProblemInstance(A, b, 0.7), SA, 1e-10, 20)
    assert r.converged and r.iterations == 1 and r.m == 16
    assert np.linalg.norm(r.x - O.direct_solve(A, b, 0.7)) <= 1e-8 * (1 + np.linalg.norm(r.x))
    xo, reso, repo = O.pcg_solve_with(A, b, 0.7, SA, 1e-10, 20)
    assert r.setup_flops == repo.setup_flops
    check_vs_oracle(r, xo, reso, repo, (A, b, 0.7, 1e-10, 20, SA), rtol=1e-5)


def test_pcg_prescribed_sketch_sizes(gpu, O):  # :71-81
    assert gpu.pcg_sketch_size(4096, 32, gpu.SketchKind.Gaussian, 0.25) == (128, False)
    assert gpu.pcg_sketch_size(4096, 32, gpu.SketchKind.SRHT, 0.25) == (math.ceil(32 * math.log(32) / 0.25), False)
    assert gpu.pcg_sketch_size(64, 32, gpu.SketchKind.SRHT, 0.25) == (64, True)
    for n, d, rho in [(1000, 7, 0.1), (1 << 20, 1024, 0.35), (5, 5, 0.9), (100, 1, 0.5)]:
        for kind in (0, 1):
            assert gpu.pcg_sketch_size(n, d, kind, rho) == O.pcg_sketch_size(n, d, kind, rho)
    with pytest.raises(gpu.InvalidInput):
        gpu.pcg_sketch_size(64, 32, gpu.SketchKind.Gaussian, 0.0)


@pytest.mark.parametrize("kind", [0, 1])
def test_pcg_agrees_with_direct(gpu, O, kind):  # :82-88
    A, b = exp_instance(128, 16, 6)
    r = gpu.pcg_solve(gpu.ProblemInstance(A, b, 0.1), kind, 17, 0.25, 1e-11, 100)
    assert r.converged
    assert np.linalg.norm(r.x - O.direct_solve(A, b, 0.1)) <= 1e-7 * (1 + np.linalg.norm(r.x))
    xo, reso, repo = O.pcg_solve(A, b, 0.1, kind, 17, 0.25, 1e-11, 100)
    assert (r.m, r.m_capped, r.setup_flops) == (repo.m, bool(repo.m_capped), repo.setup_flops)
    m, _ = O.pcg_sketch_size(128, 16, kind, 0.25)
    check_vs_oracle(r, xo, reso, repo, (A, b, 0.1, 1e-11, 100, O.sketch(A, kind, m, 17)), rtol=1e-5)


def test_pcg_setup_counter(gpu, O):  # :89-99
    A, b = O.test_support_data(75, 64, 8, 64)
    r = gpu.pcg_solve(gpu.ProblemInstance(A, b, 0.5), gpu.SketchKind.Gaussian, 1, 0.25, 1e-8, 50)
    assert r.setup_flops == r.m * 64 * 8 + 8 * 8 * r.m + 8 * 8 * 8 // 3
    check_vs_oracle(r, *O.pcg_solve(A, b, 0.5, 0, 1, 0.25, 1e-8, 50),
                    (A, b, 0.5, 1e-8, 50, O.sketch(A, 0, r.m, 1)), rtol=1e-5)


def test_pcg_srht_capped_and_small_m(gpu, O):
    # m < d: the preconditioner is still the d x d Gram form (baselines.hpp:111-114)
    A, b = O.test_support_data(78, 40, 12, 40)
    r = gpu.pcg_solve(gpu.ProblemInstance(A, b, 0.3), gpu.SketchKind.SRHT, 3, 0.25, 1e-10, 100)
    assert r.m_capped and r.m == 64 and r.converged
    check_vs_oracle(r, *O.pcg_solve(A, b, 0.3, 1, 3, 0.25, 1e-10, 100),
                    (A, b, 0.3, 1e-10, 100, O.sketch(A, 1, 64, 3)), rtol=1e-5)
    SA = RNG(5).standard_normal((6, 12))
    r = gpu.pcg_solve_with(gpu.ProblemInstance(A, b, 0.3), SA, 1e-10, 200)
    check_vs_oracle(r, *O.pcg_solve_with(A, b, 0.3, SA, 1e-10, 200), (A, b, 0.3, 1e-10, 200, SA), xtol=1e-7)


@pytest.mark.parametrize("kind", [0, 1])
def test_pcg_synthetic_larger(gpu, O, kind):
    # a SURVEY §8(d) instance (A = G diag(0.99^j)), tall enough for the gradient kernels' large-n paths
    A, b, _ = O.synth(16384, 96, decay=0.97, noise_std=0.1)
    p = gpu.ProblemInstance(A, b, 1e-3)
    r = gpu.pcg_solve(p, kind, 5, 0.5, 1e-10, 200)
    xo, reso, repo = O.pcg_solve(A, b, 1e-3, kind, 5, 0.5, 1e-10, 200)
    assert r.converged and (r.m, r.setup_flops) == (repo.m, repo.setup_flops)
    check_vs_oracle(r, xo, reso, repo, (A, b, 1e-3, 1e-10, 200, O.sketch(A, kind, r.m, 5)), xtol=1e-8)
    c = gpu.cg_solve(p, 1e-6, 300)
    check_vs_oracle(c, *O.cg_solve(A, b, 1e-3, 1e-6, 300), (A, b, 1e-3, 1e-6, 300), xtol=1e-5)
