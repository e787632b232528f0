"""Adaptive-solve parity at the BASELINE configs.

* C1 (n=8192, d=256) and C2 (n=65536, d=512, Gaussian m=1024) at full size against a live CPU oracle solve, with
  the bench's knobs (bench.CONFIGS) and with the reference defaults;
* C3, C4 (SRHT and Gaussian) and C5 down-scaled to n/16 — same seeded generator, d, nu, sigma — against the
  committed oracle solves in tests/golden/configs_n16.npz (tests/golden/make_config_golden.py; a single-thread
  oracle solve of the C4/C5 shapes takes minutes to tens of minutes);
* the convention knobs the defaults never exercise: recompute_r_after_resketch = false and non-default eta.

Each case requires the identical audit trail (t, m, branch) — the m-schedule and every Polyak / gradient /
resketch decision — identical iteration count, rejections, final m and cost counters, and the final iterate within
1e-10 of the oracle's in the Abar norm ||Abar (x - x_ref)|| / ||Abar x_ref||, Abar = [A; nu I].
"""
import pathlib

import numpy as np
import pytest

import bench

G16 = pathlib.Path(__file__).resolve().parent / "golden" / "configs_n16.npz"


def _abar_rel(A, nu, x, xr):
    num = np.linalg.norm(np.concatenate([A @ (x - xr), nu * (x - xr)]))
    den = np.linalg.norm(np.concatenate([A @ xr, nu * xr]))
    return num / den


def _gpu_cfg(gpu, c, **over):
    kw = dict(rho=c["rho"], sketch_kind=getattr(gpu.SketchKind, c["sketch"]), mode=getattr(gpu.SolveMode, c["mode"]),
              m_initial=c["m_initial"], max_sketch=c["max_sketch"], eps=c["eps"], seed=0,
              enforce_validity=c["enforce_validity"])
    kw.update(over)
    return gpu.SolverConfig(**kw)


def _oracle_cfg(O, c, **over):
    kw = dict(rho=c["rho"], sketch_kind=1 if c["sketch"] == "SRHT" else 0,
              mode=1 if c["mode"] == "GradientOnly" else 0, m_initial=c["m_initial"],
              max_sketch=c["max_sketch"] or 0, eps=c["eps"], seed=0, enforce_validity=int(c["enforce_validity"]))
    kw.update({k: (int(v) if isinstance(v, bool) else (v or 0) if k == "max_sketch" else v) for k, v in over.items()})
    return O.default_config(**kw)


def _check(rep, log_ref, summary_ref, counters_ref, A, nu, x_ref):
    assert [(e.t, e.m, int(e.branch)) for e in rep.log] == [tuple(map(int, r)) for r in log_ref]
    assert [rep.iterations, rep.rejections, rep.final_m, int(rep.converged)] == [int(v) for v in summary_ref[:4]]
    c = rep.counters
    assert [c.sketch, c.factor, c.solve, c.matvec] == [int(v) for v in counters_ref]
    assert _abar_rel(A, nu, rep.x, x_ref) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name,over", [("c1", {}), ("c1", dict(eps=1e-10)), ("c2", {}),
                                       ("c2", dict(eps=1e-10))], ids=["c1-bench", "c1-default", "c2-bench", "c2-eps"])
def test_full_size_config_matches_oracle(gpu, O, name, over):
    c = bench.CONFIGS[name]
    A, b, _ = gpu.synth_generate(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                                 outlier_frac=c["outliers"], data_seed=0)
    p = gpu.ProblemInstance(A, b, c["nu"])
    rep = gpu.adaptive_solve(p, _gpu_cfg(gpu, c, **over))
    x_o, rep_o, log_o, _ = O.adaptive_solve(A, b, c["nu"], _oracle_cfg(O, c, **over))
    co = rep_o.counters
    _check(rep, [(e[0], e[1], e[4]) for e in log_o],
           [rep_o.iterations, rep_o.rejections, rep_o.final_m, rep_o.converged],
           [co.sketch, co.factor, co.solve, co.matvec], A, c["nu"], x_o)


def _n16_cases():
    if not G16.exists():
        return []
    z = np.load(G16)
    return sorted({k[: -len("_spec")] for k in z.files if k.endswith("_spec")})


@pytest.mark.gpu
@pytest.mark.parametrize("case", _n16_cases())
def test_downscaled_config_matches_oracle(gpu, case):
    z = np.load(G16)
    name = case.split("_")[0]
    c = bench.CONFIGS[name]
    n, d = (int(v) for v in z[f"{case}_spec"])
    m_init, max_sketch, recompute = (int(v) for v in z[f"{case}_knobs"])
    eps = float(z[f"{case}_eps"][0])
    A, b, _ = gpu.synth_generate(n, d, spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                                 outlier_frac=c["outliers"], data_seed=0)
    p = gpu.ProblemInstance(A, b, c["nu"])
    rep = gpu.adaptive_solve(p, _gpu_cfg(gpu, c, m_initial=m_init, max_sketch=max_sketch or None, eps=eps,
                                         recompute_r_after_resketch=bool(recompute)))
    _check(rep, z[f"{case}_log"], z[f"{case}_summary"], z[f"{case}_counters"], A, c["nu"], z[f"{case}_x"])
    assert rep.sketch_exhausted == bool(z[f"{case}_summary"][4])
    # the recorded decrements follow the oracle's to fp64 tolerance (floor: 1e-20 r_1 near convergence)
    r_ref = z[f"{case}_r"]
    r1 = float(z[f"{case}_r1"][0])
    for e, (r, r_prev) in zip(rep.log, r_ref):
        assert abs(e.r - r) <= 1e-7 * abs(r) + 1e-20 * r1


CONVENTION_CASES = [
    # (label, n, d, nu, decay, sketch, overrides)
    ("srht-no-recompute", 8192, 128, 1e-3, 0.97, "SRHT", dict(recompute_r_after_resketch=False, m_initial=256,
                                                                 eps=1e-21)),
    ("gauss-no-recompute", 8192, 64, 1e-2, 0.95, "Gaussian", dict(recompute_r_after_resketch=False)),
    ("gauss-eta-0.001", 8192, 64, 1e-2, 0.95, "Gaussian", dict(eta=0.001, rho=0.05)),
    ("gauss-eta-0.005-permissive", 8192, 64, 1e-2, 0.95, "Gaussian", dict(eta=0.005, rho=0.3,
                                                                         enforce_validity=False)),
    ("srht-gradonly-no-recompute", 8192, 128, 1e-2, 0.95, "SRHT", dict(mode="GradientOnly",
                                                                        recompute_r_after_resketch=False)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("label,n,d,nu,decay,sketch,over", CONVENTION_CASES, ids=[c[0] for c in CONVENTION_CASES])
def test_convention_knobs_match_oracle(gpu, O, label, n, d, nu, decay, sketch, over):
    A, b, _ = gpu.synth_generate(n, d, decay=decay, noise_std=0.01, data_seed=3)
    over = dict(over)
    mode = over.pop("mode", "PolyakThenGradient")
    gkw = dict(sketch_kind=getattr(gpu.SketchKind, sketch), mode=getattr(gpu.SolveMode, mode), seed=1, **over)
    okw = dict(sketch_kind=1 if sketch == "SRHT" else 0, mode=1 if mode == "GradientOnly" else 0, seed=1,
               **{k: (int(v) if isinstance(v, bool) else v) for k, v in over.items()})
    p = gpu.ProblemInstance(A, b, nu)
    rep = gpu.adaptive_solve(p, gpu.SolverConfig(**gkw))
    x_o, rep_o, log_o, _ = O.adaptive_solve(A, b, nu, O.default_config(**okw))
    co = rep_o.counters
    _check(rep, [(e[0], e[1], e[4]) for e in log_o],
           [rep_o.iterations, rep_o.rejections, rep_o.final_m, rep_o.converged],
           [co.sketch, co.factor, co.solve, co.matvec], A, nu, x_o)
    assert rep.recompute_r_after_resketch == bool(over.get("recompute_r_after_resketch", True))
