#!/usr/bin/env python3
"""Benchmark: adaptive-IHS time-to-1e-10 on the BASELINE configs (B200).

Default workload = BASELINE.json configs[1] ("C2"): Gaussian-sketch
Polyak-IHS, fp64, n=65536, d=512, fixed m=1024, nu=1e-3, sigma_j=0.98^j,
b = A x_true + N(0, 0.01^2). A "step" is one complete adaptive_solve
(solver.hpp:242) to r_t/r_1 <= 1e-10 with A resident in HBM; `value` is the
device-timed seconds per solve (lower is better). `e2e` repeats the step
through the public API with the H2D upload of A and b from pinned host
memory and the D2H of x inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                  [--impl b200|reference] [--no-cpu-baseline] [--solver ihs|pcg|cg]

--solver pcg|cg times the paper's comparators on the same data instead
(baselines.hpp: sketch-preconditioned CG with the prescribed sketch size
m = d/rho or d ln d/rho at bench.hpp's default rho = 0.1, and plain CG), to
tol 1e-10 on ||H x - A^T b|| <= tol ||A^T b||, max 2000 iterations.

Multi-GPU (torchrun, one rank per GPU): A is row-sharded over the ranks
(strong scaling of the same problem; --replicas for independent copies),
value = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# --------------------------------------------------------------------- configs
CONFIGS = {
    "c1": dict(desc="C1 SRHT adaptive gradient-IHS n=8192 d=256", n=8192, d=256, spectrum=0, decay=0.95,
               noise=0.01, nu=1e-2, outliers=0.0, sketch="SRHT", mode="GradientOnly", rho=0.1,
               m_initial=1, max_sketch=None, enforce_validity=True),
    "c2": dict(desc="C2 Gaussian Polyak-IHS n=65536 d=512 fixed m=1024", n=65536, d=512, spectrum=0, decay=0.98,
               noise=0.01, nu=1e-3, outliers=0.0, sketch="Gaussian", mode="PolyakThenGradient", rho=0.35,
               m_initial=1024, max_sketch=1024, enforce_validity=False),
    "c3": dict(desc="C3 SRHT adaptive Polyak-IHS n=2^20 d=1024", n=1 << 20, d=1024, spectrum=0, decay=0.99,
               noise=0.1, nu=1e-3, outliers=0.0, sketch="SRHT", mode="PolyakThenGradient", rho=0.1,
               m_initial=1, max_sketch=None, enforce_validity=True),
    "c4": dict(desc="C4 SRHT adaptive Polyak-IHS n=2^22 d=2048 sigma=1/j", n=1 << 22, d=2048, spectrum=1,
               decay=0.0, noise=0.01, nu=1e-4, outliers=0.0, sketch="SRHT", mode="PolyakThenGradient", rho=0.1,
               m_initial=1, max_sketch=None, enforce_validity=True),
    "c4g": dict(desc="C4 Gaussian adaptive Polyak-IHS n=2^22 d=2048 sigma=1/j (streamed S)", n=1 << 22, d=2048,
                spectrum=1, decay=0.0, noise=0.01, nu=1e-4, outliers=0.0, sketch="Gaussian", mode="PolyakThenGradient",
                rho=0.1, m_initial=1, max_sketch=None, enforce_validity=True),
    "c5": dict(desc="C5 SRHT adaptive Polyak-IHS n=10^6 (pad 2^20) d=4096 +1% x100 outliers", n=10**6, d=4096,
               spectrum=0, decay=0.999, noise=0.01, nu=1e-5, outliers=0.01, sketch="SRHT",
               mode="PolyakThenGradient", rho=0.1, m_initial=1, max_sketch=None, enforce_validity=True),
}
METRIC = "adaptive-IHS time-to-1e-10 error (r_t/r_1 <= 1e-10)"
METRICS = {"ihs": METRIC,
           "pcg": "PCG time-to-1e-10 (||H x - A^T b|| <= 1e-10 ||A^T b||, sketch-preconditioned, baselines.hpp)",
           "cg": "CG time-to-1e-10 (||H x - A^T b|| <= 1e-10 ||A^T b||, baselines.hpp)"}
PCG_RHO, CG_TOL, CG_MAX_ITERS = 0.1, 1e-10, 2000  # bench.hpp:32-36 SolverSpec defaults
L2_BYTES = 126 * 2**20


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def read_stream_peak():
    """Measured read-only HBM stream (the gradient's and SRHT phase 1's access pattern): tools/hbm_read_bw.cu ->
    profiles/hbm_read_bw.json. A kernel that only reads A can exceed the copy figure of MEASURED_PEAKS.json."""
    try:
        return float(json.loads((ROOT / "profiles" / "hbm_read_bw.json").read_text())["read_gbs"])
    except Exception:  # noqa: BLE001
        return None


def fp64_peak():
    """Measured fp64 tensor (DMMA) peak: tools/fp64_peak.cu -> profiles/fp64_peak.json."""
    try:
        j = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())
        return float(j["fp64_dmma_tflops"]), "measured (tools/fp64_peak.cu, mma.sync m8n8k4 f64 loop)"
    except Exception:  # noqa: BLE001
        return 37.0, "fallback (B200 fp64 tensor nominal)"


def ncu_traffic(cfg, which):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant kernel from the
    committed `ncu --set full` summary profiles/traffic.json (written by tools/ncu_traffic.py), or None."""
    try:
        j = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return j[cfg][which]
    except Exception:  # noqa: BLE001
        return None


def solver_config(ihs, c, seed=0):
    return ihs.SolverConfig(rho=c["rho"], sketch_kind=getattr(ihs.SketchKind, c["sketch"]),
                            mode=getattr(ihs.SolveMode, c["mode"]), m_initial=c["m_initial"],
                            max_sketch=c["max_sketch"], eps=1e-10, seed=seed,
                            enforce_validity=c["enforce_validity"])


def oracle_config(O, c, seed=0):
    from paper_2006_05874_b200 import _abi as abi
    return O.default_config(rho=c["rho"], sketch_kind=abi.SKETCH_SRHT if c["sketch"] == "SRHT" else abi.SKETCH_GAUSSIAN,
                            mode=abi.MODE_GRADIENT_ONLY if c["mode"] == "GradientOnly" else abi.MODE_POLYAK_THEN_GRADIENT,
                            m_initial=c["m_initial"], max_sketch=c["max_sketch"] or 0, eps=1e-10, seed=seed,
                            enforce_validity=int(c["enforce_validity"]))


# --------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device: int, path: pathlib.Path):
        self.path = path
        self.proc = None
        self.device = device

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi takes a few hundred ms to start: wait for its first row so the samples cover the
            # timed region from its start (a short region still yields only a few rows at 100 ms)
            t_end = time.time() + 3.0
            while time.time() < t_end and self.proc.poll() is None and self.path.stat().st_size == 0:
                time.sleep(0.01)
        except Exception:  # noqa: BLE001
            self.proc = None
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.window_ms = 1e3 * (time.time() - self.t0)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in self.path.read_text().strip().splitlines()]
            rows = [[x.strip() for x in r] for r in rows if len(r) >= 9]
        except Exception:  # noqa: BLE001
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [s for s in sm if s > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "interval_ms": 100,
                "window_ms": round(getattr(self, "window_ms", 0.0), 1)}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# --------------------------------------------------------------------- reference arm
def run_reference(args, c, rank, world):
    from oracle import oracle as O
    if rank != 0:
        return 0
    A, b, _ = O.synth(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                      outlier_frac=c["outliers"], data_seed=0)
    cfg = oracle_config(O, c)
    times = []
    for i in range(args.warmup_ref + args.steps):
        t0 = time.perf_counter()
        if args.solver == "ihs":
            x, rep, log, _ = O.adaptive_solve(A, b, c["nu"], cfg)
            wall = rep.wall_seconds
        else:
            kind = 1 if c["sketch"] == "SRHT" else 0
            x, _, rep = (O.pcg_solve(A, b, c["nu"], kind, 0, PCG_RHO, CG_TOL, CG_MAX_ITERS) if args.solver == "pcg"
                         else O.cg_solve(A, b, c["nu"], CG_TOL, CG_MAX_ITERS))
            wall = time.perf_counter() - t0
        if i >= args.warmup_ref:
            times.append(wall)
    v = float(np.mean(times))
    extra = ({"rejections": int(rep.rejections), "final_m": int(rep.final_m)} if args.solver == "ihs"
             else {"m": int(rep.m), "converged": bool(rep.converged)})
    line = {"impl": "reference", "metric": METRICS[args.solver], "value": v, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d) generator)",
            "config": {"workload": c["desc"], **{k: c[k] for k in ("n", "d", "nu", "sketch", "mode", "rho")}},
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "port",
                             "sample": f"full {args.solver} solve of {args.config.upper()} per step (oracle C++ "
                                       "restatement, single thread like the reference)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "iterations": int(rep.iterations), **extra}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- b200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="do not sample nvidia-smi during the timed steps")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of row sharding")
    ap.add_argument("--solver", default="ihs", choices=["ihs", "pcg", "cg"],
                    help="ihs: adaptive Polyak-IHS (the headline); pcg / cg: the baselines.hpp comparators")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.warmup_ref = 0  # the CPU reference has nothing to warm up; W is reported as given
    c = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        if args.impl == "b200":
            torch.cuda.set_device(local)
        tdist.init_process_group("nccl" if args.impl == "b200" else "gloo")
        dist = tdist
    if args.impl == "reference":
        rc = run_reference(args, c, rank, world)
        if dist:
            dist.destroy_process_group()
        return rc

    import torch
    from paper_2006_05874_b200 import ihs

    torch.cuda.set_device(local)
    n, d, nu = c["n"], c["d"], c["nu"]
    # N > 1: A is row-sharded: rank r holds rows [r n_pad/N, (r+1) n_pad/N) of the padded index
    # space, the sketch partials and gradient partials are combined over NCCL inside the library, and every
    # rank runs the same replicated small solve. --replicas runs N independent copies instead.
    sharded = world > 1 and not args.replicas
    parallelism = "single GPU"
    row0, rows = 0, n
    comm = None
    if sharded:
        row0, rows = ihs.shard_rows(n, world, rank)
        uid = [ihs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ihs.NcclComm(uid[0], world, rank, local)
        parallelism = f"row-sharded x{world} (NCCL all-gather/all-reduce of sketch and gradient partials)"
    elif world > 1:
        parallelism = f"replicas x{world}"
    # inputs in pinned host memory (torch is plumbing only)
    A_t = torch.empty((d, rows), dtype=torch.float64, pin_memory=True)  # column-major rows x d
    b_t = torch.empty((rows,), dtype=torch.float64, pin_memory=True)
    A = A_t.numpy().T
    b = b_t.numpy()
    t0 = time.perf_counter()
    ihs.synth_generate(n, d, spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                       outlier_frac=c["outliers"], data_seed=0 if sharded else rank, row0=row0, rows=rows,
                       A_out=A, b_out=b)
    gen_s = time.perf_counter() - t0
    assert A.flags.f_contiguous

    if sharded:
        p = ihs.ProblemInstance(A, b, nu, device=local, world_size=world, rank=rank, comm=comm, n_global=n)
    else:
        p = ihs.ProblemInstance(A, b, nu, device=local)
    cfg = solver_config(ihs, c)
    kind = getattr(ihs.SketchKind, c["sketch"])
    if args.solver == "ihs":
        solve = lambda: ihs.adaptive_solve(p, cfg)  # noqa: E731
    elif args.solver == "pcg":
        solve = lambda: ihs.pcg_solve(p, kind, 0, PCG_RHO, CG_TOL, CG_MAX_ITERS)  # noqa: E731
    else:
        solve = lambda: ihs.cg_solve(p, CG_TOL, CG_MAX_ITERS)  # noqa: E731
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        rep = solve()
    # per-phase CUDA events cost host time on the solve's critical path (~15% of a C2 step): the timed
    # steps run without them; the roofline comes from one instrumented solve right after (see below)
    p.set_phase_timing(False)
    barrier()
    launches0 = ihs.kernel_launch_count()
    step_ms, lib_ms, reps = [], [], []
    clk = ClockSampler(local, ROOT / "gpurun_out" / f"clocks_rank{rank}.csv") if (ROOT / "gpurun_out").exists() \
        else ClockSampler(local, pathlib.Path(f"/tmp/clocks_rank{rank}.csv"))
    if args.no_clocks:
        clk.__enter__ = lambda: clk  # noqa: E731
    with (clk if not args.no_clocks else _Null()):
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the timed bracket)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rep = solve()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            lib_ms.append(rep.device_times["total_ms"])
            reps.append(rep)
    barrier()
    launches = ihs.kernel_launch_count() - launches0
    ms = float(np.mean(step_ms))
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = clk.summary()

    # ---- e2e through the public API: H2D(A, b) + solve + D2H(x) every step
    e2e = None
    if not args.no_e2e:
        e2e_ms = []
        for i in range(args.steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p.upload_async(A, b)  # H2D on the side stream; the sketch RNG overlaps it
            rep_e = solve()
            torch.cuda.synchronize()
            if i > 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        v = float(np.mean(e2e_ms)) / 1e3
        if dist:
            t = torch.tensor([v], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            v = float(t.item())
        e2e = {"value": v, "unit": "s", "h2d_bytes_per_step": 8 * rows * d + 8 * rows, "d2h_bytes_per_step": 8 * d,
               "timer": "host wall clock around upload_async+solve (includes the H2D copies; A-independent sketch "
                        "work overlaps them)"}

    # ---- roofline of the dominant kernel (live, from CUDA-event phase timers on the library's stream: the
    # sketch kernels (SRHT transform / S*A GEMM) and the fused gradient kernels are bracketed by events) of an
    # instrumented solve of the same problem run right after the timed steps
    p.set_phase_timing(True)
    flush.zero_()
    torch.cuda.synchronize()
    inst = solve()
    last = reps[-1]
    t = inst.device_times
    hbm, peak_kind = peaks()
    fp64, fp64_kind = fp64_peak()
    rd_peak = read_stream_peak()
    phases = {"gradient": t["gradient_ms"], "sketch": t["sketch_ms"], "factor": t["factor_ms"], "solve": t["solve_ms"]}
    kern = {}
    if t["n_gradient_kernel"] > 0 and t["gradient_kernel_ms"] > 0:
        # gradient_bytes counts every pass the solve made (speculative ones included), as do the timers
        per_pass = t["gradient_bytes"] / max(1, t["n_gradient"])
        ach = per_pass * t["n_gradient_kernel"] / (t["gradient_kernel_ms"] * 1e-3) / 1e9
        kern["gradient"] = {"kernel": "grad_rr/grad_rm kernel (+grad_reduce) — fused A^T(Ax-b)+nu^2 x, 1-2 RHS, "
                                      "one pass over A" + (" (b = 0: the CG product H p)" if args.solver != "ihs"
                                                           else ""),
                            "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                            "per_launch_ms": t["gradient_kernel_ms"] / t["n_gradient_kernel"],
                            "algorithmic_bytes_per_launch": per_pass,
                            "launches": t["n_gradient_kernel"], "total_ms": t["gradient_kernel_ms"],
                            "peak_source": peak_kind + " copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                            "read_stream_peak": rd_peak, "frac_read_stream": ach / rd_peak if rd_peak else None}
    if t["n_sketch_kernel"] > 0 and t["sketch_kernel_ms"] > 0:
        sk_ms = t["sketch_kernel_ms"]
        if c["sketch"] == "SRHT":
            ach = t["sketch_bytes"] / (sk_ms * 1e-3) / 1e9
            kern["sketch"] = {"kernel": "srht_phase1_tma_kernel + srht_phase2_kernel (FWHT, sign, sample gather)",
                              "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                              "algorithmic_bytes_per_launch": t["sketch_bytes"] / t["n_sketch_kernel"],
                              "peak_source": peak_kind}
        else:
            ach = t["sketch_flops"] / (sk_ms * 1e-3) / 1e12
            kern["sketch"] = {"kernel": "dgemm_kernel<0,0> S*A (mma.sync m8n8k4 f64 = DMMA)", "bound": "tensor",
                              "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64 if fp64 else None,
                              "algorithmic_flops_per_launch": t["sketch_flops"] / t["n_sketch_kernel"],
                              "peak_source": fp64_kind}
        kern["sketch"].update({"per_launch_ms": sk_ms / t["n_sketch_kernel"], "launches": t["n_sketch_kernel"],
                               "total_ms": sk_ms})
    dom = max(kern, key=lambda k: kern[k]["total_ms"]) if kern else None
    roof = dict(kern[dom]) if dom else {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None}
    roof["traffic"] = ncu_traffic(args.config, dom)
    roof["dominant"] = dom
    roof["other_kernels"] = {k: {kk: v[kk] for kk in ("kernel", "achieved", "unit", "frac", "per_launch_ms")}
                             for k, v in kern.items() if k != dom}
    roof["phase_ms"] = phases
    roof["timing"] = ("CUDA events around the kernels on the library stream, in one instrumented solve after the "
                      "timed steps (the timed steps run with phase events off)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and n * d > (1 << 26):
        cpu = {"value": None, "unit": "s", "cores": 1, "kind": "port",
               "sample": "not run: a single-thread oracle solve of this config exceeds the few-minute bench budget "
                         "(the default config C2 carries the CPU baseline)"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline and args.solver == "pcg" and \
            kind == ihs.SketchKind.Gaussian and last.m * n * d > (1 << 34):
        cpu = {"value": None, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"not run: the oracle's single-thread Gaussian sketch (m={last.m}) of this config exceeds "
                         "the few-minute bench budget"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline and args.solver != "ihs":
        from oracle import oracle as O
        t0 = time.perf_counter()
        x_ref, _, orep = (O.pcg_solve(A, b, nu, int(kind), 0, PCG_RHO, CG_TOL, CG_MAX_ITERS) if args.solver == "pcg"
                          else O.cg_solve(A, b, nu, CG_TOL, CG_MAX_ITERS))
        cpu = {"value": time.perf_counter() - t0, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"one full {args.solver} solve of {args.config.upper()} (oracle C++ restatement, 1 thread)",
               "iterations": int(orep.iterations), "same_iterations": int(orep.iterations) == last.iterations}
        Ad = np.concatenate([A @ (last.x - x_ref), nu * (last.x - x_ref)])
        Ar = np.concatenate([A @ x_ref, nu * x_ref])
        cpu["abar_rel_err_vs_oracle"] = float(np.linalg.norm(Ad) / np.linalg.norm(Ar))
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        ocfg = oracle_config(O, c)
        x_ref, orep, olog, _ = O.adaptive_solve(A, b, nu, ocfg)
        cpu = {"value": float(orep.wall_seconds), "unit": "s", "cores": 1, "kind": "port",
               "sample": f"one full adaptive_solve of {args.config.upper()} (oracle C++ restatement, 1 thread)",
               "same_m_schedule": bool(orep.rejections == last.rejections and orep.final_m == last.final_m
                                      and orep.iterations == last.iterations)}
        Ad = np.concatenate([A @ (last.x - x_ref), nu * (last.x - x_ref)])
        Ar = np.concatenate([A @ x_ref, nu * x_ref])
        cpu["abar_rel_err_vs_oracle"] = float(np.linalg.norm(Ad) / np.linalg.norm(Ar))

    if rank == 0:
        if args.solver == "ihs":
            summary = {"iterations": last.iterations, "rejections": last.rejections, "final_m": last.final_m,
                       "converged": last.converged, "m_schedule": [e.m for e in last.log if int(e.branch) == 2]}
            cfg_extra = {"rho": c["rho"], "m_initial": c["m_initial"], "max_sketch": c["max_sketch"],
                         "enforce_validity": c["enforce_validity"], "eps": 1e-10}
        else:
            summary = {"iterations": last.iterations, "converged": last.converged, "m": last.m,
                       "m_capped": last.m_capped, "residual_ratio": last.residuals[-1] / last.residuals[0]}
            cfg_extra = {"solver": args.solver, "tol": CG_TOL, "max_iters": CG_MAX_ITERS,
                         **({"rho": PCG_RHO} if args.solver == "pcg" else {})}
        summary.update({"lib_total_ms": float(np.mean(lib_ms)), "step_ms": step_ms,
                        "kernel_launches_per_solve": t["kernel_launches"]})
        line = {"metric": METRICS[args.solver], "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
                "scaling": "strong" if sharded else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded SURVEY §8(d) generator: A = G diag(sigma), x_true, noise)",
                "config": {"workload": c["desc"] if args.solver == "ihs" else
                           f"{args.solver.upper()} on the {args.config.upper()} data (n={n}, d={d}, nu={nu})",
                           "n": n, "d": d, "nu": nu, "sketch": c["sketch"],
                           **({"mode": c["mode"]} if args.solver == "ihs" else {}), **cfg_extra,
                           "l2": ("inputs larger than L2 (A = %.0f MiB) and L2 flushed between steps"
                                  % (8 * n * d / 2**20)) if 8 * n * d > L2_BYTES else
                                 "L2 flushed (256 MiB write) between timed steps",
                           "parallelism": parallelism},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks,
                "solve": summary,
                "datagen_s": gen_s}
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            pathlib.Path(args.out).write_text(s + "\n")
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
