"""Pin the oracle's restatement of the CG / sketch-preconditioned CG baselines
(proj/include/ihs/baselines.hpp) against every case of the reference's own
proj/tests/test_baselines.cpp. CPU only.

The reference's generate_synthetic(Exp, n, d, seed) (datasets.hpp:63-80) draws
U, V from Householder QR of seeded Gaussians; `exp_instance` keeps its spectrum
0.95^j and planted model but takes U, V from numpy's QR (the properties the
tests check do not depend on the particular orthonormal factors).
"""
import math

import numpy as np
import pytest

from paper_2006_05874_b200 import _abi as abi


def exp_instance(n, d, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, d)))
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    sigma = 0.95 ** np.arange(1, d + 1)
    A = np.asfortranarray(U @ np.diag(sigma) @ V.T)
    b = A @ (rng.standard_normal(d) / math.sqrt(d)) + rng.standard_normal(n) / math.sqrt(n)
    return A, b


def orthogonal_sketch(A, seed):
    """sketch.hpp:121-128: Q^T A for an orthogonal n x n Q, so (QA)^T QA = A^T A."""
    n = A.shape[0]
    Q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return np.asfortranarray(Q.T @ A)


# ------------------------------------------------------------ cg_solve (test_baselines.cpp:10-57)
def test_cg_identity_instance(O):  # :11-19
    x, res, rep = O.cg_solve(np.eye(2), np.array([1.0, 2.0]), 1.0, 1e-12, 10)
    assert rep.converged and rep.iterations <= 2
    assert x == pytest.approx([0.5, 1.0], rel=1e-10)
    assert len(res) == rep.iterations + 1


def test_cg_start_at_solution(O):  # :20-28
    A, b = O.test_support_data(71, 12, 4, 12)
    xs = O.direct_solve(A, b, 0.6)
    x, res, rep = O.cg_solve(A, b, 0.6, 1e-10, 50, x0=xs)
    assert rep.converged and rep.iterations == 0 and len(res) == 1
    assert rep.counters.matvec == 2 * 12 * 4 + 2 * 4  # the starting residual's H x


def test_cg_matches_direct(O):  # :29-37
    A, b = O.test_support_data(72, 30, 6, 30)
    x, _, rep = O.cg_solve(A, b, 1.0, 1e-12, 200)
    assert rep.converged
    assert np.linalg.norm(x - O.direct_solve(A, b, 1.0)) <= 1e-10 * (1 + np.linalg.norm(x))


def test_cg_energy_error_non_increasing(O):  # :38-49
    A, b = exp_instance(48, 10, 5)
    xs = O.direct_solve(A, b, 0.2)
    prev = math.inf
    for k in range(13):
        x, _, rep = O.cg_solve(A, b, 0.2, 0.0, k)  # exactly k iterations
        assert rep.iterations == k
        delta = O.prediction_error(A, b, 0.2, x, xs)
        assert delta <= prev * (1 + 1e-10)
        prev = delta


def test_cg_not_converged_flag(O):  # :50-56
    A, b = O.test_support_data(73, 40, 20, 40)
    _, _, rep = O.cg_solve(A, b, 1e-3, 1e-14, 1)
    assert not rep.converged and rep.iterations == 1


def test_cg_counters(O):
    A, b = O.test_support_data(76, 20, 5, 20)
    _, _, rep = O.cg_solve(A, b, 0.5, 0.0, 3)
    assert rep.counters.matvec == 4 * (2 * 20 * 5 + 2 * 5)  # start + 3 iterations (baselines.hpp:51)
    assert rep.counters.sketch == rep.counters.factor == rep.counters.solve == 0


def test_cg_rejects_underdetermined_dimension(O):
    A, b = O.test_support_data(77, 3, 5, 3)
    with pytest.raises(Exception):
        O.cg_solve(A, b, 0.5, 1e-8, 5)


# ------------------------------------------------------------ pcg_solve (test_baselines.cpp:59-100)
def test_pcg_exact_preconditioner_one_iteration(O):  # :60-70
    A, b = O.test_support_data(74, 16, 5, 16)
    x, _, rep = O.pcg_solve_with(A, b, 0.7, orthogonal_sketch(A, 4), 1e-10, 20)
    assert rep.converged and rep.iterations == 1
    assert np.linalg.norm(x - O.direct_solve(A, b, 0.7)) <= 1e-8 * (1 + np.linalg.norm(x))
    assert rep.m == 16


def test_pcg_prescribed_sketch_sizes(O):  # :71-81
    assert O.pcg_sketch_size(4096, 32, abi.SKETCH_GAUSSIAN, 0.25) == (128, False)
    assert O.pcg_sketch_size(4096, 32, abi.SKETCH_SRHT, 0.25) == (math.ceil(32 * math.log(32) / 0.25), False)
    assert O.pcg_sketch_size(64, 32, abi.SKETCH_SRHT, 0.25) == (64, True)
    for bad in (0.0, 1.0, -0.5, float("nan")):
        with pytest.raises(Exception):
            O.pcg_sketch_size(64, 32, abi.SKETCH_GAUSSIAN, bad)


@pytest.mark.parametrize("kind", [abi.SKETCH_GAUSSIAN, abi.SKETCH_SRHT])
def test_pcg_agrees_with_direct(O, kind):  # :82-88 (Gaussian there; SRHT added)
    A, b = exp_instance(128, 16, 6)
    x, _, rep = O.pcg_solve(A, b, 0.1, kind, 17, 0.25, 1e-11, 100)
    assert rep.converged
    assert np.linalg.norm(x - O.direct_solve(A, b, 0.1)) <= 1e-7 * (1 + np.linalg.norm(x))


def test_pcg_setup_counter(O):  # :89-99
    A, b = O.test_support_data(75, 64, 8, 64)
    _, _, rep = O.pcg_solve(A, b, 0.5, abi.SKETCH_GAUSSIAN, 1, 0.25, 1e-8, 50)
    m = rep.m
    assert rep.setup_flops == m * 64 * 8 + 8 * 8 * m + 8 * 8 * 8 // 3
    # one M^{-1} apply for the start and after every non-final iteration (baselines.hpp:119-123)
    assert rep.converged and rep.counters.solve == 2 * 8 * 8 * rep.iterations


def test_pcg_srht_capped(O):
    A, b = O.test_support_data(78, 40, 12, 40)
    x, _, rep = O.pcg_solve(A, b, 0.3, abi.SKETCH_SRHT, 3, 0.25, 1e-10, 100)
    assert rep.m_capped and rep.m == 64 and rep.converged
