"""Committed golden fixtures (tests/golden/golden.npz, made by make_golden.py
from the reference's own headers compiled in oracle/_ref): CPU checks keep the
oracle restatement and the product's host logic on the fixtures; GPU checks
hold the CUDA path to the same bytes (bit-exact where the reference's result
involves no floating-point reduction, fp64 tolerance otherwise)."""
import pathlib

import numpy as np
import pytest

G = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "golden.npz")


def test_oracle_reproduces_golden(O):
    for i in range(3):
        seed, K, sub = (int(v) for v in G[f"derive_{i}"])
        assert O.derive_seed(seed, K) == sub
        assert np.array_equal(O.mt_raw(O.derive_seed(sub, 1), 1024), G[f"mt_raw_{i}"])
        assert np.array_equal(O.rademacher(O.derive_seed(sub, 1), 4096).astype(np.int8), G[f"signs_{i}"])
        assert np.array_equal(O.sample_without_replacement(O.derive_seed(sub, 2), 4096, 257), G[f"rows_{i}"])
        assert np.array_equal(O.fill_gaussian(O.derive_seed(sub, 0), 37, 29, 1.0 / np.sqrt(37.0)), G[f"normals_{i}"])
    A, b, _ = O.synth(3000, 12, decay=0.9, noise_std=0.01, outlier_frac=0.01, data_seed=7)
    assert np.array_equal(A, G["A"]) and np.array_equal(b, G["b"])
    assert np.array_equal(O.srht_sketch(A, 64, 3), G["srht_m64_s3"])


def test_host_logic_matches_golden(ihs):
    for i in range(3):
        seed, K, sub = (int(v) for v in G[f"derive_{i}"])
        assert ihs.derive_seed(seed, K) == sub
        assert np.array_equal(ihs.sample_without_replacement(ihs.derive_seed(sub, 2), 4096, 257), G[f"rows_{i}"])
    A, b, _ = ihs.synth_generate(3000, 12, decay=0.9, noise_std=0.01, outlier_frac=0.01, data_seed=7)
    assert np.array_equal(A, G["A"]) and np.array_equal(b, G["b"])


@pytest.mark.gpu
def test_gpu_streams_match_golden(gpu):
    for i in range(3):
        sub = int(G[f"derive_{i}"][2])
        assert np.array_equal(gpu.mt19937_64(gpu.derive_seed(sub, 1), 1024), G[f"mt_raw_{i}"])
        assert np.array_equal(gpu.rademacher(gpu.derive_seed(sub, 1), 4096).astype(np.int8), G[f"signs_{i}"])
        z = gpu.fill_gaussian(gpu.derive_seed(sub, 0), 37, 29, 1.0 / np.sqrt(37.0))
        np.testing.assert_allclose(z, G[f"normals_{i}"], rtol=1e-15, atol=0)


@pytest.mark.gpu
def test_gpu_sketches_match_golden(gpu):
    A = G["A"]
    for m, seed in [(1, 0), (64, 3), (4096, 9)]:
        assert np.array_equal(gpu.srht_sketch(A, m, seed), G[f"srht_m{m}_s{seed}"])
    SA = gpu.gaussian_sketch(A, 40, 2)
    ref = G["gauss_m40_s2"]
    assert np.max(np.abs(SA - ref)) <= 1e-13 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,name", [(0, "gauss"), (1, "srht")])
def test_gpu_solves_match_golden(gpu, kind, name):
    A, b = G["A"], G["b"]
    p = gpu.ProblemInstance(A, b, 0.05)
    rep = gpu.adaptive_solve(p, gpu.SolverConfig(sketch_kind=gpu.SketchKind(kind), seed=3))
    log = np.array([[e.t, e.m, int(e.branch)] for e in rep.log], dtype=np.int64)
    assert np.array_equal(log, G[f"solve_{name}_log"])
    assert [rep.iterations, rep.rejections, rep.final_m, int(rep.converged)] == list(G[f"solve_{name}_summary"])
    c = rep.counters
    assert [c.sketch, c.factor, c.solve, c.matvec] == [int(v) for v in G[f"solve_{name}_counters"]]
    x_ref = G[f"solve_{name}_x"]
    num = np.linalg.norm(np.concatenate([A @ (rep.x - x_ref), 0.05 * (rep.x - x_ref)]))
    den = np.linalg.norm(np.concatenate([A @ x_ref, 0.05 * x_ref]))
    assert num <= 1e-10 * den


def test_reference_reproduces_golden(R):
    """The fixtures are the reference code's output (provenance check; needs oracle/_ref)."""
    A, b = G["A"], G["b"]
    assert np.array_equal(R.synth(3000, 12, decay=0.9, noise_std=0.01, outlier_frac=0.01, data_seed=7)[0], A)
    for m, seed in [(1, 0), (64, 3), (4096, 9)]:
        assert np.array_equal(R.srht_sketch(A, m, seed), G[f"srht_m{m}_s{seed}"])
    assert np.array_equal(R.gaussian_sketch(A, 40, 2), G["gauss_m40_s2"])
    x, rep, log, _ = R.adaptive_solve(A, b, 0.05, R.default_config(sketch_kind=1, seed=3))
    assert np.array_equal(x, G["solve_srht_x"])
    assert np.array_equal(R.direct_solve(A, b, 0.05), G["direct_x"])


def test_oracle_reproduces_golden_solves(O):
    """Oracle restatement vs the reference's fixtures: audit trail, counters and summaries exact; iterates within
    1e-12 in the Abar norm (its dense algebra sums in another order)."""
    A, b = G["A"], G["b"]
    assert np.array_equal(O.gaussian_sketch(A, 40, 2), G["gauss_m40_s2"])
    for kind, name in [(0, "gauss"), (1, "srht")]:
        x, rep, log, _ = O.adaptive_solve(A, b, 0.05, O.default_config(sketch_kind=kind, seed=3))
        assert np.array_equal(np.array([[l[0], l[1], l[4]] for l in log], dtype=np.int64), G[f"solve_{name}_log"])
        assert [rep.iterations, rep.rejections, rep.final_m, rep.converged] == list(G[f"solve_{name}_summary"])
        c = rep.counters
        assert [c.sketch, c.factor, c.solve, c.matvec] == [int(v) for v in G[f"solve_{name}_counters"]]
        x_ref = G[f"solve_{name}_x"]
        num = np.linalg.norm(np.concatenate([A @ (x - x_ref), 0.05 * (x - x_ref)]))
        den = np.linalg.norm(np.concatenate([A @ x_ref, 0.05 * x_ref]))
        assert num <= 1e-12 * den


def test_oracle_reproduces_golden_baselines_and_dual(O):
    A, b = G["A"], G["b"]
    for kind, name in [(0, "gauss"), (1, "srht")]:
        x, res, rep = O.pcg_solve(A, b, 0.05, kind, 4, 0.5, 1e-10, 100)
        it, m, conv, setup = (int(v) for v in G[f"pcg_{name}_summary"])
        assert (rep.iterations, rep.m, int(rep.converged), rep.setup_flops) == (it, m, conv, setup)
        assert _rel(x, G[f"pcg_{name}_x"]) <= 1e-11
        np.testing.assert_allclose(res[:8], G[f"pcg_{name}_res"][:8], rtol=1e-10)  # before the chaotic tail
    x, res, rep = O.cg_solve(A, b, 0.05, 1e-8, 200)
    assert rep.converged and rep.iterations == int(G["cg_summary"][0]) and _rel(x, G["cg_x"]) <= 1e-8
    np.testing.assert_allclose(res[:8], G["cg_res"][:8], rtol=1e-10)
    assert _rel(O.direct_solve(A, b, 0.05), G["direct_x"]) <= 1e-13
    x, z, rep, _, _ = O.solve_underdetermined(G["Au"], G["bu"], 0.3, O.default_config(seed=5))
    assert [rep.iterations, rep.rejections, rep.final_m, int(rep.converged)] == list(G["dual_summary"])
    assert _rel(x, G["dual_x"]) <= 1e-13 and _rel(z, G["dual_z"]) <= 1e-13


def _rel(x, ref):
    return np.linalg.norm(x - ref) / (1 + np.linalg.norm(ref))


@pytest.mark.gpu
def test_gpu_baselines_and_dual_match_golden(gpu):
    A, b = G["A"], G["b"]
    p = gpu.ProblemInstance(A, b, 0.05)
    for kind, name in [(0, "gauss"), (1, "srht")]:
        r = gpu.pcg_solve(p, gpu.SketchKind(kind), 4, 0.5, 1e-10, 100)
        it, m, conv, setup = (int(v) for v in G[f"pcg_{name}_summary"])
        assert (r.m, int(r.converged), r.setup_flops) == (m, conv, setup) and abs(r.iterations - it) <= 1
        assert _rel(r.x, G[f"pcg_{name}_x"]) <= 1e-9
    r = gpu.cg_solve(p, 1e-8, 200)
    assert r.converged and abs(r.iterations - int(G["cg_summary"][0])) <= 1 and _rel(r.x, G["cg_x"]) <= 1e-7
    assert _rel(gpu.direct_solve(p), G["direct_x"]) <= 1e-11
    q = gpu.ProblemInstance(G["Au"], G["bu"], 0.3, orientation=gpu.Orientation.Underdetermined)
    rep = gpu.solve_underdetermined(q, gpu.SolverConfig(seed=5))
    assert [rep.iterations, rep.rejections, rep.final_m, int(rep.converged)] == list(G["dual_summary"])
    assert _rel(rep.x, G["dual_x"]) <= 1e-9 and _rel(rep.dual_final, G["dual_z"]) <= 1e-9
