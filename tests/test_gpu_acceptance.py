"""The reference's acceptance audit (proj/tests/acceptance.cpp), hot-path criteria, run against the B200 path.

* criterion 1 (:67-80): the SRHT targets compose to c_gd = rho (host tuning scalars of the C-ABI; CPU test);
* criteria 7-9 (:295-392): 200 adaptive solves — n = 1024, d = 128, generate_synthetic(Exp, seed 2024), nu = 0.1,
  rho = 0.1, eta = 0.01, m from 1, eps = 1e-10, max_iters = 200, Gaussian and SRHT, seeds 0..99 — on the device:
  7: m / K within the closed-form bounds in >= 95/100 runs per kind;
  8: anchor decay r_t <= r_1 c_gd^(t-1) on every accepted step, and the SRHT relative-error envelope
     delta_T / delta_1 <= 2 (1 + sigma_1^2 / nu^2) 0.1^(T-1);
  9: every SRHT run converges within predicted_iterations(0.1, 1e-10, sigma_1, nu) + K iterations;
  and every one of the 200 runs reproduces the CPU oracle's audit trail (m-schedule, branches, counters) with
  x within 1e-10 in the Abar norm;
* criterion 12 (:508-544): the analytic cost counters of the device path follow the claimed growth laws.
The SVD quantities (d_e, sigma_1, x*) come from numpy, as the reference's SpectralOracle computes them.
"""
import math

import numpy as np
import pytest


def _linear_r2(x, y):  # acceptance.cpp:33-48
    x, y = np.asarray(x, float), np.asarray(y, float)
    mx, my = x.mean(), y.mean()
    sxy = ((x - mx) * (y - my)).sum()
    return sxy * sxy / (((x - mx) ** 2).sum() * ((y - my) ** 2).sum())


def _predicted_iterations(rho, eps, sigma1, nu):  # tuning.hpp:103-110
    num = math.log(2.0) + math.log1p(sigma1 * sigma1 / (nu * nu)) + math.log(1.0 / eps)
    v = num / math.log(1.0 / rho)
    return max(1, int(math.ceil(v * (1.0 - 1e-13))))


def test_criterion_1_srht_rate_identity(ihs):
    for k in range(1, 100):
        rho = k / 100.0
        lam, Lam = ihs.srht_targets(rho)
        assert abs(ihs.rates_from_bounds(lam, Lam).c_gd - rho) <= 1e-14


@pytest.fixture(scope="module")
def suite(gpu, O):
    from paper_2006_05874_b200 import datasets

    ds = datasets.generate_synthetic(datasets.SyntheticKind.Exp, 1024, 128, 2024)
    A, b, nu = np.asfortranarray(ds.A), ds.b, 0.1
    sigma = np.linalg.svd(A, compute_uv=False)
    r = sigma**2 / (sigma**2 + nu * nu)
    d_e = r.sum() / r.max()  # problem.hpp:87-101
    Abar = np.vstack([A, nu * np.eye(128)])
    x_star = np.linalg.lstsq(Abar, np.concatenate([b, np.zeros(128)]), rcond=None)[0]

    def pe(x):  # problem.hpp:104-109
        dx = x - x_star
        return 0.5 * np.sum((A @ dx) ** 2) + 0.5 * nu * nu * np.sum(dx * dx)

    p = gpu.ProblemInstance(A, b, nu)
    runs = {0: [], 1: []}
    for kind in (0, 1):
        for seed in range(100):
            cfg = gpu.SolverConfig(sketch_kind=gpu.SketchKind(kind), rho=0.1, eta=0.01, m_initial=1, eps=1e-10,
                                   max_iters=200, seed=seed)
            rep = gpu.adaptive_solve(p, cfg)
            ocfg = O.default_config(sketch_kind=kind, rho=0.1, eta=0.01, m_initial=1, eps=1e-10, max_iters=200,
                                    seed=seed)
            x_o, rep_o, log_o, _ = O.adaptive_solve(A, b, nu, ocfg)
            runs[kind].append((rep, rep_o, log_o, x_o))
    return dict(A=A, b=b, nu=nu, d_e=d_e, sigma1=sigma[0], x_star=x_star, delta1=pe(np.zeros(128)), pe=pe, runs=runs)


@pytest.mark.gpu
def test_audit_runs_match_oracle(suite):
    A, nu = suite["A"], suite["nu"]
    for kind in (0, 1):
        for rep, rep_o, log_o, x_o in suite["runs"][kind]:
            assert [(e.t, e.m, int(e.branch)) for e in rep.log] == [(e[0], e[1], e[4]) for e in log_o]
            assert (rep.iterations, rep.rejections, rep.final_m, rep.converged) == \
                   (rep_o.iterations, rep_o.rejections, rep_o.final_m, bool(rep_o.converged))
            c, co = rep.counters, rep_o.counters
            assert (c.sketch, c.factor, c.solve, c.matvec) == (co.sketch, co.factor, co.solve, co.matvec)
            num = np.linalg.norm(np.concatenate([A @ (rep.x - x_o), nu * (rep.x - x_o)]))
            den = np.linalg.norm(np.concatenate([A @ x_o, nu * x_o]))
            assert num <= 1e-10 * den


@pytest.mark.gpu
def test_criterion_7_sketch_size_bounds(suite):
    d_e = suite["d_e"]
    m_bound_g, k_bound_g = 10.0 * d_e / 0.1, math.log2(5.0 * d_e / 0.1) + 1.0
    ok_g = sum(rep.converged and rep.final_m <= m_bound_g and rep.rejections <= k_bound_g
               for rep, *_ in suite["runs"][0])
    a_rho = (1 + math.sqrt(0.1)) / (1 - math.sqrt(0.1))                 # tuning.hpp:86-90
    C = 16.0 / 3.0 * (1.0 + math.sqrt(8.0 * math.log(d_e * 1024.0) / d_e)) ** 2  # tuning.hpp:66-70
    m_bound_s = 2.0 * a_rho * C * d_e * math.log(d_e) / 0.1
    k_bound_s = math.log2(m_bound_s / 2.0) + 1.0
    ok_s = sum(rep.converged and rep.final_m <= m_bound_s and rep.rejections <= k_bound_s
               for rep, *_ in suite["runs"][1])
    assert ok_g >= 95, f"gaussian bounds held in {ok_g}/100"
    assert ok_s >= 95, f"srht bounds held in {ok_s}/100"


@pytest.mark.gpu
def test_criterion_8_anchor_decay_and_envelope(suite):
    anchor_viol = 0
    for kind in (0, 1):
        for rep, *_ in suite["runs"][kind]:
            for e in rep.log:
                if int(e.branch) == 2:
                    continue
                if e.r > rep.r1 * rep.tuning.c_gd ** (e.t - 1) * (1.0 + 1e-9):
                    anchor_viol += 1
    assert anchor_viol == 0
    factor = 2.0 * (1.0 + suite["sigma1"] ** 2 / suite["nu"] ** 2)
    for rep, *_ in suite["runs"][1]:
        assert suite["pe"](rep.x) / suite["delta1"] <= factor * 0.1 ** (rep.iterations - 1)


@pytest.mark.gpu
def test_criterion_9_iteration_budget(suite):
    pred = _predicted_iterations(0.1, 1e-10, suite["sigma1"], suite["nu"])
    for rep, *_ in suite["runs"][1]:
        assert rep.converged and rep.iterations <= pred + rep.rejections


@pytest.mark.gpu
def test_criterion_12_cost_counter_laws(gpu):
    ms, cost = [], []
    for m in (16, 32, 64, 128, 256, 512):
        sys = gpu.SketchedSystem.factorize(np.zeros((m, 1024)), 1.0)
        assert sys.kind() == gpu.FactorKind.WoodburyInner
        ms.append(m)
        cost.append(sys.flops_per_solve())
    assert _linear_r2(ms, cost) >= 0.99
    nlogn, scost, ratio_m = [], [], 0.0
    for n in (256, 512, 1024, 2048, 4096, 8192):
        c16, c256 = gpu.CostCounters(), gpu.CostCounters()
        gpu.srht_sketch(np.zeros((n, 4)), 16, 0, c16)
        gpu.srht_sketch(np.zeros((n, 4)), 256, 0, c256)
        npad = gpu.next_pow2(n)
        nlogn.append(npad * math.log2(npad))
        scost.append(c16.sketch)
        if n == 4096:
            ratio_m = c256.sketch / c16.sketch
    assert _linear_r2(nlogn, scost) >= 0.999
    assert ratio_m <= 1.01
    g16, g256 = gpu.CostCounters(), gpu.CostCounters()
    gpu.gaussian_sketch(np.zeros((4096, 4)), 16, 0, g16)
    gpu.gaussian_sketch(np.zeros((4096, 4)), 256, 0, g256)
    assert g256.sketch == 16 * g16.sketch
