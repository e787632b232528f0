"""Regularization-path driver (bench.hpp) on the device: the reference's own cases
(proj/tests/test_bench.cpp) plus parity of every path entry with the same path
composed from oracle solves (same sub-seeds derive_seed(seed, j), same warm
starts), and the device direct_solve / set_nu used by the path."""
import io
import math

import numpy as np
import pytest

from test_oracle_baselines import exp_instance

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng


@pytest.fixture(scope="module")
def P():
    from paper_2006_05874_b200 import path

    return path


# ---------------------------------------------------------------- direct_solve / set_nu
@pytest.mark.parametrize("n,d,nu", [(96, 12, 0.5), (4096, 200, 1e-2), (20000, 64, 1e-3)])
def test_direct_solve_vs_oracle(gpu, O, n, d, nu):
    A, b = exp_instance(n, d, 3) if n < 1000 else O.synth(n, d, decay=0.98, noise_std=0.1)[:2]
    x = gpu.direct_solve(gpu.ProblemInstance(A, b, nu))
    xo = O.direct_solve(A, b, nu)
    assert np.linalg.norm(x - xo) <= 1e-10 * (1 + np.linalg.norm(xo))


def test_direct_solve_underdetermined_kernel_form(gpu, O):
    A, b = O.test_support_data(62, 16, 64, 16)
    x = gpu.direct_solve(gpu.ProblemInstance(A, b, 0.4, orientation=gpu.Orientation.Underdetermined))
    ref = A.T @ np.linalg.solve(A @ A.T + 0.16 * np.eye(16), b)  # support.hpp:26-30
    assert np.linalg.norm(x - ref) <= 1e-10 * (1 + np.linalg.norm(ref))


def test_set_nu_matches_fresh_instance(gpu, O):
    A, b = O.test_support_data(40, 300, 24, 300)
    x = RNG(1).standard_normal(24)
    p = gpu.ProblemInstance(A, b, 1.0)
    p.set_nu(0.3)
    assert p.nu() == 0.3
    assert np.array_equal(gpu.gradient(p, x), gpu.gradient(gpu.ProblemInstance(A, b, 0.3), x))
    with pytest.raises(gpu.InvalidInput):
        p.set_nu(0.0)
    with pytest.raises(gpu.InvalidInput):
        p.set_nu(float("inf"))
    # re-upload of A refreshes the dual problem's transposed copy
    Au, bu = O.test_support_data(63, 12, 48, 12)
    q = gpu.ProblemInstance(Au, bu, 0.5, orientation=gpu.Orientation.Underdetermined)
    x1 = gpu.direct_solve(q)
    q.upload(2.0 * Au, bu)
    x2 = gpu.direct_solve(q)
    ref = 2.0 * Au.T @ np.linalg.solve(4.0 * Au @ Au.T + 0.25 * np.eye(12), bu)
    assert np.linalg.norm(x2 - ref) <= 1e-10 * (1 + np.linalg.norm(ref))
    assert not np.allclose(x1, x2)


# ---------------------------------------------------------------- run_path (test_bench.cpp:11-98)
def test_single_nu_path(gpu, P):  # :14-20
    A, b = exp_instance(96, 12, 30)
    pr = P.run_path(P.Dataset(A, b), [0.5], P.SolverSpec(), 1e-10, 1)
    assert len(pr.entries) == 1 and pr.entries[0].ok and pr.entries[0].converged


def test_oracle_mode_prediction_errors(gpu, P):  # :25-37
    A, b = exp_instance(96, 12, 30)
    pr = P.run_path(P.Dataset(A, b), [1.0, 0.1, 0.01], P.SolverSpec(rho=0.1), 1e-10, 2, True)
    assert len(pr.entries) == 3
    for e in pr.entries:
        assert e.ok and e.converged and math.isfinite(e.delta) and e.delta <= 1e-6
    assert len(pr.cumulative_seconds) == 3 and pr.cumulative_seconds[2] >= pr.cumulative_seconds[0]


def test_warm_starts_do_not_cost_iterations(gpu, P):  # :38-50
    A, b = exp_instance(512, 64, 77)
    ds = P.Dataset(A, b)
    warm_le = 0
    for seed in range(30):
        spec = P.SolverSpec(rho=0.1)
        pr = P.run_path(ds, [1.0, 0.1], spec, 1e-10, seed)
        cold = P.run_one(ds, 0.1, spec, 1e-10, gpu.derive_seed(seed, 1), None)
        warm_le += pr.entries[1].iterations <= cold.iterations
    assert warm_le >= 24


def test_adaptive_sketch_below_prescription(gpu, P):  # :51-70 (the unconditional part)
    A, b = exp_instance(512, 64, 78)
    p = gpu.ProblemInstance(A, b, 0.1)
    m_pcg, _ = gpu.pcg_sketch_size(512, 64, gpu.SketchKind.Gaussian, 0.1)
    for seed in range(5):
        rep = gpu.adaptive_solve(p, gpu.SolverConfig(rho=0.1, eps=1e-10, seed=seed))
        assert rep.final_m < m_pcg


def test_underdetermined_path_through_dual(gpu, O, P):  # :71-83
    A, _ = exp_instance(96, 12, 30)
    At = np.asfortranarray(A.T)
    ub = O.test_support_data(99, 0, 0, 12)[1]
    pr = P.run_path(P.Dataset(At, ub), [1.0, 0.5], P.SolverSpec(), 1e-12, 3)
    for e in pr.entries:
        assert e.ok
        ref = At.T @ np.linalg.solve(At @ At.T + e.nu ** 2 * np.eye(12), ub)
        assert np.linalg.norm(e.x - ref) <= 1e-6 * (1 + np.linalg.norm(ref))


def test_path_errors_recorded_per_nu(gpu, P):
    A, b = exp_instance(96, 12, 30)
    spec = P.SolverSpec(id=P.SolverId.PCG, rho=1.5)  # pcg_sketch_size rejects rho >= 1
    pr = P.run_path(P.Dataset(A, b), [0.5, 0.1], spec, 1e-10, 1)
    assert [e.ok for e in pr.entries] == [False, False] and "rho" in pr.entries[0].error


# ---------------------------------------------------------------- compare_solvers (test_bench.cpp:100-135)
def test_compare_single_solver(gpu, P):
    A, b = exp_instance(96, 12, 31)
    rep = P.compare_solvers(P.Dataset(A, b), [0.5], [P.SolverSpec()], 1e-10, 2, 5)
    assert len(rep.aggregates) == 1 and rep.aggregates[0].all_converged


def test_compare_multiple_solvers_and_csv(gpu, P):
    A, b = exp_instance(96, 12, 31)
    specs = [P.SolverSpec(id=P.SolverId.AdaptivePolyak), P.SolverSpec(id=P.SolverId.AdaptiveGradient),
             P.SolverSpec(id=P.SolverId.CG), P.SolverSpec(id=P.SolverId.PCG, sketch=1, rho=0.5)]
    rep = P.compare_solvers(P.Dataset(A, b), [1.0, 0.1], specs, 1e-10, 2, 6)
    assert len(rep.aggregates) == 4 and all(a.all_converged for a in rep.aggregates)
    f = io.StringIO()
    P.write_plot_csv(f, rep)
    lines = f.getvalue().splitlines()
    assert lines[0] == "nu,adaptive,adaptive-gd,cg,pcg"
    assert len([ln for ln in lines[1:] if ln]) == 2 and lines[1].startswith("1,") and lines[2].startswith("0.1,")


# ---------------------------------------------------------------- parity with an oracle-composed path
def oracle_path(O, A, b, nus, spec, eps, seed):
    """bench.hpp:131-171 composed from oracle solves: sub-seed derive_seed(seed, j), warm start at the
    previous entry's x."""
    from paper_2006_05874_b200 import _abi as abi

    out, warm = [], None
    for j, nu in enumerate(nus):
        sub = O.derive_seed(seed, j)
        if spec.id in (0, 1):
            cfg = O.default_config(rho=spec.rho, eta=spec.eta, sketch_kind=int(spec.sketch),
                                   m_initial=spec.m_initial, eps=eps, max_iters=spec.max_iters, seed=sub,
                                   mode=abi.MODE_POLYAK_THEN_GRADIENT if spec.id == 0 else abi.MODE_GRADIENT_ONLY,
                                   enforce_validity=int(spec.enforce_validity))
            keep = None
            if warm is not None:
                keep = np.ascontiguousarray(warm)
                cfg.warm_start = keep.ctypes.data_as(abi.C.POINTER(abi.C.c_double))
            x, rep, _, _ = O.adaptive_solve(A, b, nu, cfg)
            out.append((x, int(rep.iterations), int(rep.final_m), bool(rep.converged)))
        elif spec.id == 2:
            x, _, rep = O.cg_solve(A, b, nu, eps, spec.max_iters, x0=warm)
            out.append((x, int(rep.iterations), 0, bool(rep.converged)))
        else:
            x, _, rep = O.pcg_solve(A, b, nu, int(spec.sketch), sub, spec.rho, eps, spec.max_iters, x0=warm)
            out.append((x, int(rep.iterations), int(rep.m), bool(rep.converged)))
        warm = x
    return out


@pytest.mark.parametrize("sid,sketch", [(0, 0), (0, 1), (1, 1), (2, 0), (3, 0), (3, 1)])
def test_path_entries_match_oracle_path(gpu, O, P, sid, sketch):
    A, b, _ = O.synth(4096, 48, decay=0.95, noise_std=0.05)
    spec = P.SolverSpec(id=P.SolverId(sid), sketch=gpu.SketchKind(sketch), rho=0.25 if sid == 3 else 0.1)
    nus = [1.0, 0.3, 0.1]
    pr = P.run_path(P.Dataset(A, b), nus, spec, 1e-10, 7)
    ref = oracle_path(O, A, b, nus, spec, 1e-10, 7)
    for e, (xo, it, m, conv) in zip(pr.entries, ref):
        assert e.ok and e.converged == conv
        if sid in (0, 1):
            # adaptive IHS: identical m-schedule and iteration count (decisions are exact on the host)
            assert (e.iterations, e.final_m) == (it, m)
        else:
            assert e.final_m == m and abs(e.iterations - it) <= 2
        assert np.linalg.norm(e.x - xo) <= 1e-8 * (1 + np.linalg.norm(xo))


def test_upload_async_matches_sync(gpu, O):
    """ihs_gpu_problem_upload_async: the next solve / gradient / sketch / CG orders its first A-reading kernel
    after the side-stream copy; results equal those after a synchronous upload."""
    A, b, _ = O.synth(20000, 64, decay=0.97, noise_std=0.05)
    A2 = np.asfortranarray(A * 1.5)
    b2 = np.ascontiguousarray(b * 0.5)
    ref = gpu.ProblemInstance(A2, b2, 0.1)
    for kind in (0, 1):
        p = gpu.ProblemInstance(A, b, 0.1)
        p.upload_async(A2, b2)
        cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind(kind), seed=2)
        r1 = gpu.adaptive_solve(p, cfg)
        r0 = gpu.adaptive_solve(ref, cfg)
        assert np.array_equal(r1.x, r0.x) and r1.iterations == r0.iterations
    p = gpu.ProblemInstance(A, b, 0.1)
    x = RNG(4).standard_normal(64)
    p.upload_async(A2, b2)
    assert np.array_equal(gpu.gradient(p, x), gpu.gradient(ref, x))
    p.upload_async(A, b)
    assert np.array_equal(gpu.pcg_solve(p, gpu.SketchKind.SRHT, 1, 0.5, 1e-10, 50).x,
                          gpu.pcg_solve(gpu.ProblemInstance(A, b, 0.1), gpu.SketchKind.SRHT, 1, 0.5, 1e-10, 50).x)
    with pytest.raises(gpu.InvalidInput):
        p.upload_async(np.ascontiguousarray(A), b)  # C-ordered: would need a copy that dies before the transfer


def test_upload_async_chunked_matches_sync(gpu):
    """A large A (>= 256 MB, IHS_UPLOAD_CHUNK_MB) re-uploaded asynchronously goes in column chunks whose row-major
    copies are built as they land, and the next solve's first SRHT runs chunk by chunk behind the copies: the solve
    and a gradient must equal those after a synchronous upload bit for bit."""
    n, d = (1 << 19) + 5, 72  # 302 MB
    A, b, _ = gpu.synth_generate(n, d, decay=0.97, noise_std=0.05, data_seed=11)
    A2 = np.asfortranarray(A * 0.75)
    b2 = np.ascontiguousarray(b * 1.25)
    ref = gpu.ProblemInstance(A2, b2, 0.05)
    p = gpu.ProblemInstance(A, b, 0.05)
    cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind.SRHT, seed=3, m_initial=2 * d, eps=1e-21)
    p.upload_async(A2, b2)
    r1 = gpu.adaptive_solve(p, cfg)
    r0 = gpu.adaptive_solve(ref, cfg)
    assert np.array_equal(r1.x, r0.x) and r1.iterations == r0.iterations and r1.final_m == r0.final_m
    x = RNG(9).standard_normal(d)
    p.upload_async(A, b)
    assert np.array_equal(gpu.gradient(p, x), gpu.gradient(gpu.ProblemInstance(A, b, 0.05), x))


@pytest.mark.parametrize("m_initial,eps", [(144, 1e-21), (8, 1e-21), (4096, 1e-12)])
def test_doublings_sketched_behind_chunked_upload(gpu, m_initial, eps):
    """An adaptive SRHT solve started while a chunked upload is in flight prepares the first sketch and the next
    doublings (IHS_UPLOAD_SPEC_DEPTH, default 5) up front and runs them chunk by chunk behind the copies, their
    factorizations on side streams; doublings beyond them are sketched in place, unused ones are only waited for.
    The solve must equal the one on a resident A bit for bit: x, the m-schedule, iterations and cost counters
    (few doublings, more doublings than the depth, and none needed)."""
    n, d = (1 << 19) + 5, 72  # 302 MB: copied in chunks
    A, b, _ = gpu.synth_generate(n, d, decay=0.97, noise_std=0.05, data_seed=11)
    A2 = np.asfortranarray(A * 0.75)
    b2 = np.ascontiguousarray(b * 1.25)
    ref = gpu.ProblemInstance(A2, b2, 0.05)
    p = gpu.ProblemInstance(A, b, 0.05)
    cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind.SRHT, seed=3, m_initial=m_initial, eps=eps)
    r0 = gpu.adaptive_solve(ref, cfg)
    before = gpu.thread_upload_doublings()
    for _ in range(2):  # the second round reuses the pooled systems and sketch contexts
        p.upload_async(A2, b2)
        r1 = gpu.adaptive_solve(p, cfg)
        assert np.array_equal(r1.x, r0.x)
        assert (r1.iterations, r1.rejections, r1.final_m) == (r0.iterations, r0.rejections, r0.final_m)
        assert [(e.t, e.m, e.r, e.branch) for e in r1.log] == [(e.t, e.m, e.r, e.branch) for e in r0.log]
        assert r1.counters == r0.counters
    assert gpu.thread_upload_doublings() - before == 2 * 5
    # and a solve of the now resident problem takes the plain path with the same result
    r2 = gpu.adaptive_solve(p, cfg)
    assert np.array_equal(r2.x, r0.x) and r2.counters == r0.counters
    assert gpu.thread_upload_doublings() - before == 2 * 5


@pytest.mark.parametrize("d", [512, 300])
def test_gram_accumulated_behind_chunked_upload(gpu, d):
    """With d >= 256 the sketched Gram SA^T SA of each doubling prepared behind the upload is launched block row by
    block row (128 rows) as the columns are sketched, on the same tiles and K partition as the single product, and
    the factorization only reduces it: the solve must still equal the resident one bit for bit. (m = 1024..4096
    fall back to the whole product - too few tiles for the 128 x 128 kernel - the larger doublings take the pieces.)"""
    n = 1 << 19  # d = 512: 2 GiB in 8 chunks of 64 columns; d = 300: chunks of 38 columns, a ragged last block row
    A, b, _ = gpu.synth_generate(n, d, decay=0.99, noise_std=0.05, data_seed=5)
    p = gpu.ProblemInstance(A, b, 0.02)
    cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind.SRHT, seed=7, m_initial=1024, eps=1e-21)
    r0 = gpu.adaptive_solve(p, cfg)
    rows0, dbl0 = gpu.thread_upload_gram_rows(), gpu.thread_upload_doublings()
    for _ in range(2):
        p.upload_async(A, b)
        r1 = gpu.adaptive_solve(p, cfg)
        assert np.array_equal(r1.x, r0.x)
        assert (r1.iterations, r1.rejections, r1.final_m) == (r0.iterations, r0.rejections, r0.final_m)
        assert [(e.t, e.m, e.r, e.branch) for e in r1.log] == [(e.t, e.m, e.r, e.branch) for e in r0.log]
        assert r1.counters == r0.counters
    assert gpu.thread_upload_doublings() - dbl0 == 10
    rows = gpu.thread_upload_gram_rows() - rows0
    assert rows > 0 and rows % (2 * d) == 0  # whole Gram matrices of some doublings, both rounds


@pytest.mark.parametrize("d", [640, 200])
def test_gaussian_product_behind_chunked_upload(gpu, d):
    """A Gaussian-sketch solve started behind a chunked upload launches S*A in block-column pieces (128 columns,
    the tiles and K partition of the single call) as A's chunks land and reduces them at the end: bit-identical to
    the solve on a resident A (d = 640: pieces every 128 columns over chunks of 80; d = 200: chunks of 25)."""
    n = (1 << 16) + 3 if d == 640 else (1 << 18) + 1  # 335 MB / 419 MB
    A, b, _ = gpu.synth_generate(n, d, decay=0.98, noise_std=0.01, data_seed=2)
    p = gpu.ProblemInstance(A, b, 1e-3)
    cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind.Gaussian, seed=1, rho=0.35, m_initial=1024, max_sketch=1024,
                           enforce_validity=False, eps=1e-18)
    r0 = gpu.adaptive_solve(p, cfg)
    for _ in range(2):
        p.upload_async(A, b)
        r1 = gpu.adaptive_solve(p, cfg)
        assert np.array_equal(r1.x, r0.x)
        assert (r1.iterations, r1.rejections, r1.final_m) == (r0.iterations, r0.rejections, r0.final_m)
        assert r1.counters == r0.counters
