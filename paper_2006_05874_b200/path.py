"""Regularization-path driver and solver comparison (proj/include/ihs/bench.hpp:17-239).

Same API and semantics as the reference: `run_one` solves one (dataset, nu)
with any of the four solvers, `run_path` sweeps a strictly decreasing nu
sequence warm-starting each solve at the previous solution with sub-seed
derive_seed(seed, j), `compare_solvers` repeats paths over seeds
derive_seed(base_seed, 97 si + r) and aggregates, `write_plot_csv` writes the
time-vs-regularizer series.

B200 difference: the reference rebuilds a ProblemInstance (a copy of A) for
every nu (bench.hpp:71,151); here a path uploads A to the device once and only
changes nu between solves (ProblemInstance.set_nu), so the sweep pays the
host->device copy of A once. The oracle-mode reference solution is computed on
the device too (ihs.direct_solve: DMMA Gram + Cholesky + iterative refinement).
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import ihs
from .datasets import Dataset


class SolverId(enum.IntEnum):  # bench.hpp:17
    AdaptivePolyak = 0
    AdaptiveGradient = 1
    CG = 2
    PCG = 3


def solver_name(sid: SolverId) -> str:  # bench.hpp:19-27
    return {SolverId.AdaptivePolyak: "adaptive", SolverId.AdaptiveGradient: "adaptive-gd", SolverId.CG: "cg",
            SolverId.PCG: "pcg"}.get(SolverId(sid), "?")


@dataclass
class SolverSpec:  # bench.hpp:29-41
    id: SolverId = SolverId.AdaptivePolyak
    sketch: ihs.SketchKind = ihs.SketchKind.Gaussian
    rho: float = 0.1
    eta: float = 0.01
    m_initial: int = 1
    max_iters: int = 2000
    enforce_validity: bool = True
    label: str = ""

    def name(self) -> str:
        return self.label if self.label else solver_name(self.id)


@dataclass
class RunSummary:  # bench.hpp:44-59
    solver: str = ""
    nu: float = 0.0
    x: np.ndarray = field(default_factory=lambda: np.empty(0))
    dual_final: np.ndarray = field(default_factory=lambda: np.empty(0))
    ok: bool = False
    converged: bool = False
    iterations: int = 0
    final_m: int = 0
    rejections: int = 0
    wall_seconds: float = 0.0
    flops: int = 0
    error: str = ""
    delta: float = math.nan  # oracle mode only
    device_ms: float = 0.0   # device time of the solve (CUDA events on the library stream)


@dataclass
class PathResult:  # bench.hpp:61-65
    nus: List[float] = field(default_factory=list)
    entries: List[RunSummary] = field(default_factory=list)
    cumulative_seconds: List[float] = field(default_factory=list)


@dataclass
class SolverAggregate:  # bench.hpp:173-182
    label: str = ""
    mean_seconds: float = 0.0
    std_seconds: float = 0.0
    mean_iterations: float = 0.0
    mean_final_m: float = 0.0
    max_final_m: int = 0
    all_converged: bool = True
    mean_cumulative: List[float] = field(default_factory=list)


@dataclass
class ComparisonReport:  # bench.hpp:184-190
    nus: List[float] = field(default_factory=list)
    repeats: int = 0
    eps: float = 0.0
    aggregates: List[SolverAggregate] = field(default_factory=list)
    runs: List[List[PathResult]] = field(default_factory=list)


def _instance(dataset: Dataset, nu: float, problem: Optional[ihs.ProblemInstance]) -> ihs.ProblemInstance:
    if problem is None:
        return ihs.ProblemInstance.make(dataset.A, dataset.b, nu)
    problem.set_nu(nu)
    return problem


def run_one(dataset: Dataset, nu: float, spec: SolverSpec, eps: float, seed: int,
            warm: Optional[RunSummary] = None, problem: Optional[ihs.ProblemInstance] = None) -> RunSummary:
    """One solve of `dataset` at `nu`, optionally warm-started (bench.hpp:66-127). `problem`: a
    device-resident instance of the same dataset to reuse (its nu is set here)."""
    out = RunSummary(solver=spec.name(), nu=nu)
    try:
        p = _instance(dataset, nu, problem)
        under = p.orientation() == ihs.Orientation.Underdetermined and p.rows() != p.cols()
        if spec.id in (SolverId.AdaptivePolyak, SolverId.AdaptiveGradient):
            cfg = ihs.SolverConfig(rho=spec.rho, eta=spec.eta, sketch_kind=spec.sketch, m_initial=spec.m_initial,
                                   eps=eps, max_iters=spec.max_iters, seed=seed,
                                   mode=ihs.SolveMode.PolyakThenGradient if spec.id == SolverId.AdaptivePolyak
                                   else ihs.SolveMode.GradientOnly,
                                   enforce_validity=spec.enforce_validity)
            if warm is not None and warm.ok:
                if under and warm.dual_final.size == p.rows():
                    cfg.warm_start = warm.dual_final
                elif not under and warm.x.size == p.cols():
                    cfg.warm_start = warm.x
            rep = ihs.solve_underdetermined(p, cfg) if under else ihs.adaptive_solve(p, cfg)
            out.x = rep.x
            out.dual_final = rep.dual_final if rep.dual_final is not None else np.empty(0)
            out.converged, out.iterations = rep.converged, rep.iterations
            out.final_m, out.rejections = rep.final_m, rep.rejections
            out.wall_seconds, out.flops = rep.wall_seconds, rep.counters.total()
            out.device_ms = rep.device_times.get("total_ms", 0.0)
        else:
            x0 = warm.x if warm is not None and warm.ok and warm.x.size == p.cols() else None
            if spec.id == SolverId.CG:
                r = ihs.cg_solve(p, eps, spec.max_iters, x0)
            else:
                r = ihs.pcg_solve(p, spec.sketch, seed, spec.rho, eps, spec.max_iters, x0)
                out.final_m = r.m
            out.x, out.converged, out.iterations = r.x, r.converged, r.iterations
            out.wall_seconds, out.flops, out.device_ms = r.wall_seconds, r.counters.total(), r.device_ms
        out.ok = True
    except ihs.Error as e:
        out.error = str(e)
    return out


def run_path(dataset: Dataset, nus: Sequence[float], spec: SolverSpec, eps: float, seed: int,
             oracle_mode: bool = False) -> PathResult:
    """Regularization path (bench.hpp:131-171): strictly decreasing nus, each solve warm-started at the
    previous solution with seed derive_seed(seed, j); failures are recorded per nu and the path goes
    on. oracle_mode records the prediction error against the exact minimizer."""
    nus = [float(v) for v in nus]
    if not nus:
        raise ihs.InvalidInput("run_path: empty regularization path")
    for i in range(1, len(nus)):
        if not nus[i] < nus[i - 1]:
            raise ihs.InvalidInput("run_path: nu values must be strictly decreasing")
    path = PathResult(nus=list(nus))
    problem = None
    try:
        problem = ihs.ProblemInstance.make(dataset.A, dataset.b, nus[0])  # A resident for the whole path
    except ihs.Error:
        problem = None  # run_one reports the construction error per nu, as the reference does
    cum = 0.0
    warm = None
    for j, nu in enumerate(nus):
        s = run_one(dataset, nu, spec, eps, ihs.derive_seed(seed, j), warm, problem)
        if oracle_mode and s.ok:
            p = _instance(dataset, nu, problem)
            x_star = ihs.direct_solve(p)
            s.delta = ihs.prediction_error(p, s.x, x_star)
        cum += s.wall_seconds
        path.cumulative_seconds.append(cum)
        path.entries.append(s)
        warm = s
    return path


def compare_solvers(dataset: Dataset, nus: Sequence[float], specs: Sequence[SolverSpec], eps: float, repeats: int,
                    base_seed: int, oracle_mode: bool = False) -> ComparisonReport:
    """Every solver `repeats` times with seeds derive_seed(base_seed, 97 si + r) over the same path,
    aggregated (bench.hpp:194-239)."""
    if repeats < 1:
        raise ihs.InvalidInput("compare_solvers: repeats must be >= 1")
    if not specs:
        raise ihs.InvalidInput("compare_solvers: no solvers given")
    rep = ComparisonReport(nus=[float(v) for v in nus], repeats=repeats, eps=eps)
    for si, spec in enumerate(specs):
        per_repeat = [run_path(dataset, nus, spec, eps, ihs.derive_seed(base_seed, 97 * si + r), oracle_mode)
                      for r in range(repeats)]
        agg = SolverAggregate(label=spec.name(), mean_cumulative=[0.0] * len(nus))
        totals, iter_sum, m_sum, count = [], 0.0, 0.0, 0
        for pr in per_repeat:
            totals.append(pr.cumulative_seconds[-1])
            for j in range(len(nus)):
                s = pr.entries[j]
                agg.mean_cumulative[j] += pr.cumulative_seconds[j] / repeats
                iter_sum += s.iterations
                m_sum += s.final_m
                agg.max_final_m = max(agg.max_final_m, s.final_m)
                agg.all_converged = agg.all_converged and s.ok and s.converged
                count += 1
        agg.mean_seconds = sum(totals) / repeats
        var = sum((t - agg.mean_seconds) ** 2 for t in totals)
        agg.std_seconds = math.sqrt(var / (repeats - 1)) if repeats > 1 else 0.0
        agg.mean_iterations = iter_sum / count
        agg.mean_final_m = m_sum / count
        rep.aggregates.append(agg)
        rep.runs.append(per_repeat)
    return rep


def _fmt(v: float) -> str:
    # std::ostream's default double formatting (6 significant digits, %g)
    return f"{v:g}"


def write_plot_csv(f, rep: ComparisonReport):
    """Header row then one row per nu: mean cumulative seconds per solver (bench.hpp:244-254)."""
    f.write("nu" + "".join("," + a.label for a in rep.aggregates) + "\n")
    for j, nu in enumerate(rep.nus):
        f.write(_fmt(nu) + "".join("," + _fmt(a.mean_cumulative[j]) for a in rep.aggregates) + "\n")
