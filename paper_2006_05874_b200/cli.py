"""`ihs` command-line driver (proj/tools/ihs_cli.cpp) over the device solvers.

    python -m paper_2006_05874_b200.cli solve   (--csv F | --libsvm F | --synthetic exp|poly [--n --d --data-seed])
                                                --nu NU [solver options] [--out R.json] [--oracle]
    python -m paper_2006_05874_b200.cli path    ... [--nus 1,0.1,...] [--solver adaptive|adaptive-gd|cg|pcg]
    python -m paper_2006_05874_b200.cli compare ... [--nus ...] [--solvers adaptive,adaptive-gd,cg,pcg]
                                                [--repeats R] [--out plot.csv | report.json]
    python -m paper_2006_05874_b200.cli synth   --synthetic exp|poly [--n --d --data-seed] [--out F.csv]

Solver options: --sketch gaussian|srht, --rho, --eta, --eps, --seed, --m-initial,
--mode polyak|gradient-only, --max-iters, --force-params. Reports are the
reference's JSON layout (serialize.hpp:33-117); exit status 0 when every solve
converged, 1 otherwise, 2 on an error (ihs_cli.cpp:340-350). The reference's
`concentration` subcommand (Monte Carlo eigenvalue experiments,
concentration.hpp) is outside this build's scope.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

import numpy as np

from . import ihs
from . import path as P
from .datasets import DatasetSource, SyntheticKind, generate_synthetic, load_csv, load_libsvm

_STEP_NAMES = {0: "polyak", 1: "gradient", 2: "resketch"}  # serialize.hpp:15-22


# ------------------------------------------------------------------ serialize.hpp
def counters_json(c: ihs.CostCounters) -> dict:
    return {"sketch": c.sketch, "factor": c.factor, "solve": c.solve, "matvec": c.matvec, "total": c.total()}


def report_json(rep: ihs.SolveReport) -> dict:  # serialize.hpp:33-57
    t = rep.tuning
    return {"iterations": rep.iterations, "rejected": rep.rejections, "final_m": rep.final_m, "r1": rep.r1,
            "r_final": rep.r_final, "converged": rep.converged, "sketch_exhausted": rep.sketch_exhausted,
            "wall_seconds": rep.wall_seconds, "recompute_r_after_resketch": rep.recompute_r_after_resketch,
            "tuning": {"lam": t.lam, "Lam": t.Lam, "mu_gd": t.mu_gd, "c_gd": t.c_gd, "mu_p": t.mu_p,
                       "beta_p": t.beta_p, "c_p": t.c_p},
            "counters": counters_json(rep.counters),
            "log": [{"t": e.t, "m": e.m, "r": e.r, "r_prev": e.r_prev, "branch": _STEP_NAMES[int(e.branch)]}
                    for e in rep.log],
            "x": [float(v) for v in rep.x]}


def summary_json(s: P.RunSummary) -> dict:  # serialize.hpp:84-95
    j = {"solver": s.solver, "nu": s.nu, "ok": s.ok, "converged": s.converged, "iterations": s.iterations,
         "final_m": s.final_m, "rejected": s.rejections, "wall_seconds": s.wall_seconds, "flops": s.flops}
    if s.error:
        j["error"] = s.error
    if math.isfinite(s.delta):
        j["delta"] = s.delta
    j["x"] = [float(v) for v in s.x]
    return j


def path_json(pr: P.PathResult) -> dict:  # serialize.hpp:97-103
    return {"nus": pr.nus, "cumulative_seconds": pr.cumulative_seconds,
            "entries": [summary_json(e) for e in pr.entries]}


def comparison_json(rep: P.ComparisonReport) -> dict:  # serialize.hpp:105-117
    return {"nus": rep.nus, "repeats": rep.repeats, "eps": rep.eps,
            "solvers": [{"solver": a.label, "mean_seconds": a.mean_seconds, "std_seconds": a.std_seconds,
                         "mean_iterations": a.mean_iterations, "mean_final_m": a.mean_final_m,
                         "max_final_m": a.max_final_m, "all_converged": a.all_converged,
                         "mean_cumulative_seconds": a.mean_cumulative} for a in rep.aggregates]}


# ------------------------------------------------------------------ options (ihs_cli.cpp:19-100)
def _add_data(p):
    g = p.add_mutually_exclusive_group()
    g.add_argument("--csv", default="", help="CSV dataset (last column is b)")
    g.add_argument("--libsvm", default="", help="libsvm/svmlight dataset")
    g.add_argument("--synthetic", default="", choices=["exp", "poly"], help="synthetic spectrum: exp or poly")
    p.add_argument("--n", type=int, default=1024, help="synthetic rows")
    p.add_argument("--d", type=int, default=128, help="synthetic columns")
    p.add_argument("--data-seed", type=int, default=0, help="synthetic dataset seed")


def _add_solver(p):
    p.add_argument("--sketch", default="gaussian", choices=["gaussian", "srht"], help="embedding")
    p.add_argument("--rho", type=float, default=0.1, help="target aspect ratio")
    p.add_argument("--eta", type=float, default=0.01, help="Gaussian tail parameter")
    p.add_argument("--eps", type=float, default=1e-10, help="relative decrement target")
    p.add_argument("--seed", type=int, default=0, help="solver seed")
    p.add_argument("--m-initial", type=int, default=1, help="initial sketch size")
    p.add_argument("--mode", default="polyak", choices=["polyak", "gradient-only"])
    p.add_argument("--max-iters", type=int, default=2000, help="iteration cap")
    p.add_argument("--force-params", action="store_true", help="accept (rho, eta) outside the proven region")


def load_data(a):
    if a.csv:
        return load_csv(a.csv)
    if a.libsvm:
        return load_libsvm(a.libsvm)
    if a.synthetic:
        return generate_synthetic(SyntheticKind.Exp if a.synthetic == "exp" else SyntheticKind.Poly, a.n, a.d,
                                  a.data_seed)
    raise ihs.InvalidInput("no dataset given: use --csv, --libsvm or --synthetic")


def _kind(a):
    return ihs.SketchKind.SRHT if a.sketch == "srht" else ihs.SketchKind.Gaussian


def to_config(a) -> ihs.SolverConfig:
    return ihs.SolverConfig(sketch_kind=_kind(a), rho=a.rho, eta=a.eta, eps=a.eps, seed=a.seed,
                            m_initial=a.m_initial,
                            mode=ihs.SolveMode.PolyakThenGradient if a.mode == "polyak" else ihs.SolveMode.GradientOnly,
                            max_iters=a.max_iters, enforce_validity=not a.force_params)


def _spec(a, sid: P.SolverId) -> P.SolverSpec:
    return P.SolverSpec(id=sid, sketch=_kind(a), rho=a.rho, eta=a.eta, m_initial=a.m_initial,
                        max_iters=a.max_iters, enforce_validity=not a.force_params)


def parse_nus(text: str, ds) -> list:
    """ihs_cli.cpp:102-117: 10^4..10^-2 for real data, 10^0..10^-4 for synthetic spectra by default."""
    if not text:
        synthetic = ds.source in (DatasetSource.SyntheticExp, DatasetSource.SyntheticPoly)
        hi, lo = (0, -4) if synthetic else (4, -2)
        return [10.0 ** j for j in range(hi, lo - 1, -1)]
    return [float(t) for t in text.split(",")]


def _write(path: str, content: str):
    try:
        with open(path, "w") as f:
            f.write(content)
    except OSError:
        raise ihs.InvalidInput(f"cannot open output file '{path}'") from None


_SOLVER_IDS = {"adaptive": P.SolverId.AdaptivePolyak, "adaptive-gd": P.SolverId.AdaptiveGradient,
               "cg": P.SolverId.CG, "pcg": P.SolverId.PCG}


# ------------------------------------------------------------------ subcommands (ihs_cli.cpp:119-290)
def cmd_solve(a) -> int:
    ds = load_data(a)
    p = ihs.ProblemInstance.make(ds.A, ds.b, a.nu)
    cfg = to_config(a)
    over = p.orientation() == ihs.Orientation.Overdetermined
    rep = ihs.adaptive_solve(p, cfg) if over else ihs.solve_underdetermined(p, cfg)
    j = report_json(rep)
    j["nu"] = a.nu
    j["dataset"] = ds.provenance
    if a.oracle:
        x_star = ihs.direct_solve(p)
        j["delta"] = ihs.prediction_error(p, rep.x, x_star)
        j["rel_error"] = float(np.linalg.norm(rep.x - x_star) / (1.0 + np.linalg.norm(x_star)))
    if a.out:
        _write(a.out, json.dumps(j, indent=2) + "\n")
    print(f"solver: {'adaptive' if cfg.mode == ihs.SolveMode.PolyakThenGradient else 'adaptive-gd'} ({a.sketch})")
    print(f"converged: {'yes' if rep.converged else 'no'}")
    print(f"iterations: {rep.iterations}  rejected: {rep.rejections}  final m: {rep.final_m}")
    print(f"r_final/r_1: {rep.r_final / rep.r1 if rep.r1 > 0 else 0.0:g}")
    print(f"wall seconds: {rep.wall_seconds:g}")
    if a.oracle:
        print(f"delta (oracle): {j['delta']:g}")
    return 0 if rep.converged else 1


def cmd_path(a) -> int:
    ds = load_data(a)
    nus = parse_nus(a.nus, ds)
    pr = P.run_path(ds, nus, _spec(a, _SOLVER_IDS[a.solver]), a.eps, a.seed, a.oracle)
    j = path_json(pr)
    j["dataset"] = ds.provenance
    if a.out:
        _write(a.out, json.dumps(j, indent=2) + "\n")
    ok = True
    print("nu          iters  final_m  cum_seconds  converged")
    for e, cum in zip(pr.entries, pr.cumulative_seconds):
        status = ("yes" if e.converged else "NO") if e.ok else e.error
        print(f"{e.nu:<11.3g} {e.iterations:<6d} {e.final_m:<8d} {cum:<12.4f} {status}")
        ok = ok and e.ok and e.converged
    return 0 if ok else 1


def cmd_compare(a) -> int:
    ds = load_data(a)
    nus = parse_nus(a.nus, ds)
    specs = []
    for name in [s for s in a.solvers.split(",") if s != ""]:
        if name not in _SOLVER_IDS:
            raise ihs.InvalidInput(f"unknown solver '{name}'")
        specs.append(_spec(a, _SOLVER_IDS[name]))
    if not specs:
        raise ihs.InvalidInput("no solvers given")
    rep = P.compare_solvers(ds, nus, specs, a.eps, a.repeats, a.seed, a.oracle)
    if a.out:
        if len(a.out) > 4 and a.out.endswith(".csv"):
            import io

            f = io.StringIO()
            P.write_plot_csv(f, rep)
            _write(a.out, f.getvalue())
        else:
            _write(a.out, json.dumps(comparison_json(rep), indent=2) + "\n")
    ok = True
    print("solver       mean_s     std_s      mean_iters  mean_m   converged")
    for g in rep.aggregates:
        print(f"{g.label:<12s} {g.mean_seconds:<10.4f} {g.std_seconds:<10.4f} {g.mean_iterations:<11.1f} "
              f"{g.mean_final_m:<8.1f} {'yes' if g.all_converged else 'NO'}")
        ok = ok and g.all_converged
    return 0 if ok else 1


def cmd_synth(a) -> int:
    if not a.synthetic:
        raise ihs.InvalidInput("synth requires --synthetic {exp,poly}")
    ds = load_data(a)
    rows = "".join(",".join(repr(float(v)) for v in ds.A[i]) + "," + repr(float(ds.b[i])) + "\n"
                   for i in range(ds.n()))
    if a.out:
        _write(a.out, rows)
    else:
        sys.stdout.write(rows)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ihs", description="adaptive sketch-size solver for L2-regularized least "
                                                         "squares (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve one instance adaptively")
    _add_data(s)
    _add_solver(s)
    s.add_argument("--nu", type=float, required=True, help="regularization scale")
    s.add_argument("--out", default="", help="write a JSON report")
    s.add_argument("--oracle", action="store_true", help="also report the direct-solve prediction error")
    pth = sub.add_parser("path", help="solve a decreasing regularization path with warm starts")
    _add_data(pth)
    _add_solver(pth)
    pth.add_argument("--nus", default="", help="comma-separated decreasing nu values")
    pth.add_argument("--solver", default="adaptive", choices=sorted(_SOLVER_IDS))
    pth.add_argument("--out", default="", help="write a JSON report")
    pth.add_argument("--oracle", action="store_true", help="record prediction errors against direct solves")
    cmp_ = sub.add_parser("compare", help="run several solvers over the same path")
    _add_data(cmp_)
    _add_solver(cmp_)
    cmp_.add_argument("--nus", default="", help="comma-separated decreasing nu values")
    cmp_.add_argument("--solvers", default="adaptive,adaptive-gd,cg,pcg", help="comma-separated solver list")
    cmp_.add_argument("--repeats", type=int, default=5, help="independent trials per solver")
    cmp_.add_argument("--out", default="", help="plot-data CSV (.csv) or JSON report")
    cmp_.add_argument("--oracle", action="store_true", help="record prediction errors against direct solves")
    syn = sub.add_parser("synth", help="emit a synthetic dataset as CSV")
    _add_data(syn)
    syn.add_argument("--out", default="", help="output CSV path (stdout if omitted)")
    a = ap.parse_args(argv)
    try:
        return {"solve": cmd_solve, "path": cmd_path, "compare": cmd_compare, "synth": cmd_synth}[a.cmd](a)
    except (ihs.Error, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
