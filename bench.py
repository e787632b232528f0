#!/usr/bin/env python3
"""Benchmark: adaptive-IHS time-to-1e-10 on the BASELINE configs (B200).

Default workload = C4-SRHT, the largest BASELINE config that fits one GPU (configs[3]: n=2^22, d=2048, A = 64 GiB,
sigma_j = 1/j, nu = 1e-4, adaptive m, Polyak-IHS with the SRHT). A "step" is one complete adaptive_solve
(solver.hpp:242) with A resident in HBM; `value` is the device-timed seconds per solve (lower is better). `e2e`
repeats the step through the public API with the H2D upload of A and b from pinned host memory and the D2H of x
inside the timed region.

"Time to 1e-10": the reference stops at r_t <= eps r_1 (solver.hpp:154,177), a ratio of sketched Newton
decrements, i.e. of SQUARED prediction errors measured under the current sketch. Each config's
(m_initial, eps) is chosen (oracle + device scans) so that the returned x satisfies
  delta = ||Abar (x - x*)|| / ||Abar x*|| <= 1e-10,   Abar = [A; nu I],  x* = device direct_solve,
which every bench line reports as `solve.delta_rel_vs_direct` (with pe_rel = delta^2 = prediction_error(x) /
prediction_error(0), problem.hpp:104-109). C3-C5 start at m_initial = 2d (r_1 measured under a subspace
embedding) with eps = 1e-21; C1 keeps BASELINE's "m starts at 1" with eps = 1e-27; C2 (fixed m = 1024 = 2d)
uses eps = 1e-21.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl b200|reference]
                  [--no-cpu-baseline] [--solver ihs|pcg|cg]

--solver pcg|cg times the paper's comparators on the same data instead (baselines.hpp: sketch-preconditioned
CG with the prescribed sketch size m = d/rho or d ln d/rho at bench.hpp's default rho = 0.1, and plain CG), to
tol 1e-10 on ||H x - A^T b|| <= tol ||A^T b||, max 2000 iterations.

CPU baseline (`cpu_baseline`, and the `--impl reference` arm): the oracle restatement of the reference (pinned
bit-for-bit to the reference's own headers, tests/test_ref_pin.py) on the host, single thread like the
reference. C1 and C2 run whole solves. For C3-C5 a whole single-thread solve takes 10 min to hours, so each
step times bounded samples of the same workload — one SRHT/Gaussian sketch over a few full-length columns, a
gradient over a row block, a factorization + solves of a sketched system — and extrapolates with the solve's
analytic cost counters (types.hpp:18-33; identical on the GPU and the reference, tests/test_gpu_parity.py):
  t = sum over phases of counters[phase] x (host seconds per counter unit measured on the sample).

Multi-GPU (torchrun, one rank per GPU): A is row-sharded over the ranks (strong scaling of the same problem;
--replicas for independent copies), value = max over ranks.
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
# m_initial / eps: see the module docstring and DESIGN.md §4 (chosen so delta <= 1e-10 against direct_solve)
CONFIGS = {
    "c1": dict(desc="C1 SRHT adaptive gradient-IHS n=8192 d=256", n=8192, d=256, spectrum=0, decay=0.95,
               noise=0.01, nu=1e-2, outliers=0.0, sketch="SRHT", mode="GradientOnly", rho=0.1,
               m_initial=1, max_sketch=None, enforce_validity=True, eps=1e-27),
    "c2": dict(desc="C2 Gaussian Polyak-IHS n=65536 d=512 fixed m=1024", n=65536, d=512, spectrum=0, decay=0.98,
               noise=0.01, nu=1e-3, outliers=0.0, sketch="Gaussian", mode="PolyakThenGradient", rho=0.35,
               m_initial=1024, max_sketch=1024, enforce_validity=False, eps=1e-21),
    "c3": dict(desc="C3 SRHT adaptive Polyak-IHS n=2^20 d=1024", n=1 << 20, d=1024, spectrum=0, decay=0.99,
               noise=0.1, nu=1e-3, outliers=0.0, sketch="SRHT", mode="PolyakThenGradient", rho=0.1,
               m_initial=2048, max_sketch=None, enforce_validity=True, eps=1e-21),
    "c4": dict(desc="C4 SRHT adaptive Polyak-IHS n=2^22 d=2048 sigma=1/j", n=1 << 22, d=2048, spectrum=1,
               decay=0.0, noise=0.01, nu=1e-4, outliers=0.0, sketch="SRHT", mode="PolyakThenGradient", rho=0.1,
               m_initial=4096, max_sketch=None, enforce_validity=True, eps=1e-21),
    "c4g": dict(desc="C4 Gaussian adaptive Polyak-IHS n=2^22 d=2048 sigma=1/j (streamed S)", n=1 << 22, d=2048,
                spectrum=1, decay=0.0, noise=0.01, nu=1e-4, outliers=0.0, sketch="Gaussian", mode="PolyakThenGradient",
                rho=0.1, m_initial=4096, max_sketch=None, enforce_validity=True, eps=1e-21),
    "c5": dict(desc="C5 SRHT adaptive Polyak-IHS n=10^6 (pad 2^20) d=4096 +1% x100 outliers", n=10**6, d=4096,
               spectrum=0, decay=0.999, noise=0.01, nu=1e-5, outliers=0.01, sketch="SRHT",
               mode="PolyakThenGradient", rho=0.1, m_initial=8192, max_sketch=None, enforce_validity=True, eps=1e-21),
}
DEFAULT_CONFIG = "c4"
FULL_CPU_SOLVE = ("c1", "c2")  # configs whose whole single-thread oracle solve fits the bench budget
# cost counters of one solve per config (rep.counters: sketch, factor, solve, matvec), recorded from the device
# solve (equal to the reference's by the parity tests); the reference arm multiplies them with its measured host
# rates for configs whose whole CPU solve does not fit the bench budget. The b200 arm checks them live.
REF_COUNTERS_PATH = ROOT / "profiles" / "ref_counters.json"
METRIC = "adaptive-IHS time-to-1e-10 error (||Abar(x - x*)|| / ||Abar x*|| <= 1e-10)"
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


def l2_write_peak():
    """Measured L2-resident write bandwidth (tools/l2_bw.cu -> profiles/l2_bw.json, 96 MiB buffer, whole lines)."""
    try:
        j = json.loads((ROOT / "profiles" / "l2_bw.json").read_text())
        return float(j["96_MiB"]["write_GBps"])
    except Exception:  # noqa: BLE001
        return None


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
                            max_sketch=c["max_sketch"], eps=c["eps"], seed=seed,
                            enforce_validity=c["enforce_validity"])


def oracle_config(O, c, seed=0):
    from paper_2006_05874_b200 import _abi as abi
    return O.default_config(rho=c["rho"], sketch_kind=abi.SKETCH_SRHT if c["sketch"] == "SRHT" else abi.SKETCH_GAUSSIAN,
                            mode=abi.MODE_GRADIENT_ONLY if c["mode"] == "GradientOnly" else abi.MODE_POLYAK_THEN_GRADIENT,
                            m_initial=c["m_initial"], max_sketch=c["max_sketch"] or 0, eps=c["eps"], seed=seed,
                            enforce_validity=int(c["enforce_validity"]))


def config_dict(args, c, world):
    """The `config` object of the JSON line: identical on both arms (same workload, knobs and layout)."""
    n, d = c["n"], c["d"]
    if world > 1:
        parallelism = f"replicas x{world}" if args.replicas else \
            f"row-sharded x{world} (NCCL all-gather/all-reduce of sketch and gradient partials)"
    else:
        parallelism = "single GPU"
    out = {"workload": c["desc"] if args.solver == "ihs" else
           f"{args.solver.upper()} on the {args.config.upper()} data (n={n}, d={d}, nu={c['nu']})",
           "config": args.config, "n": n, "d": d, "nu": c["nu"], "sketch": c["sketch"], "data_seed": 0,
           "solver_seed": 0}
    if args.solver == "ihs":
        out.update({"mode": c["mode"], "rho": c["rho"], "m_initial": c["m_initial"], "max_sketch": c["max_sketch"],
                    "enforce_validity": c["enforce_validity"], "eps": c["eps"],
                    "target": "||Abar(x-x*)||/||Abar x*|| <= 1e-10 (x* = direct_solve)"})
    else:
        out.update({"solver": args.solver, "tol": CG_TOL, "max_iters": CG_MAX_ITERS,
                    **({"rho": PCG_RHO} if args.solver == "pcg" else {})})
    out["l2"] = (("inputs larger than L2 (A = %.0f MiB) and L2 flushed between steps" % (8 * n * d / 2**20))
                 if 8 * n * d > L2_BYTES else "L2 flushed (256 MiB write) between timed steps")
    out["parallelism"] = parallelism
    return out


# --------------------------------------------------------------------- CPU baseline (oracle port, 1 thread)
def host_phase_rates(O, c, m_sample):
    """Host seconds per cost-counter unit of each phase of the reference solve (types.hpp:18-33), measured with
    the oracle restatement (single thread) on bounded samples of this config's workload:
      sketch  SRHT: one srht_sketch over `cs` full-length columns (the FWHT length n_pad and its log factor are
              the config's own; counter unit = butterfly/sign/gather, sketch.hpp:99-106);
              Gaussian: S generation per normal (rng.hpp:35-40) + S*A per multiply-add (sketch.hpp:65-68);
      matvec  8 gradients (problem.hpp:59-69) over a ~128 MiB row block with all d columns (unit = counted MAC);
      factor  SketchedSystem::factorize of a (4 d_s) x d_s sketch, d_s = min(d, 768) (unit = d^2 m + d^3/3);
      solve   SketchedSystem::solve on the same system (unit = d^2 + d).
    Returns ({phase: seconds per unit}, description, seconds spent timing)."""
    import time as _t
    t_start = _t.perf_counter()
    n, d = c["n"], c["d"]
    rates, parts = {}, []
    n_pad = 1 << (n - 1).bit_length()
    logn = n_pad.bit_length() - 1
    if c["sketch"] == "SRHT":
        cs = max(2, min(d, int(round(1e9 / (n_pad * logn)))))
        A_s, _, _ = O.synth(n, cs, spectrum=c["spectrum"], decay=c["decay"], noise_std=0.0, data_seed=0)
        m_s = min(m_sample, n_pad)
        t, cnt = O.time_sketch(A_s, 1, m_s, 0)
        rates["sketch"] = t / cnt.sketch
        parts.append(f"srht_sketch n={n} x {cs} columns, m={m_s}: {t:.3f} s")
        del A_s
    else:
        n_s, d_s, m_s = 8192, min(d, 256), 512
        t_norm = O.time_fill_gaussian(O.derive_seed(0, 0), m_s, n_s) / (m_s * n_s)
        A_s, _, _ = O.synth(n_s, d_s, spectrum=c["spectrum"], decay=c["decay"], noise_std=0.0, data_seed=0)
        t, cnt = O.time_sketch(A_s, 0, m_s, 0)
        t_mac = max(t - t_norm * m_s * n_s, 0.0) / (m_s * n_s * d_s)
        rates["sketch_normal"], rates["sketch"] = t_norm, t_mac
        parts.append(f"gaussian_sketch {m_s}x{n_s} S times {n_s}x{d_s} A: {t:.3f} s ({t_norm * 1e9:.1f} ns/normal)")
    n_g = int(min(n, max(1024, (128 << 20) // (8 * d))))
    A_g, b_g, _ = O.synth(n_g, d, spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"], data_seed=0)
    x_g = np.full(d, 0.5)
    t, cnt = O.time_gradient(A_g, b_g, c["nu"], x_g, 8)
    rates["matvec"] = t / cnt.matvec
    parts.append(f"8 gradients over {n_g}x{d}: {t:.3f} s")
    del A_g, b_g
    d_s = min(d, 768)
    SA = np.asfortranarray(np.random.default_rng(0).standard_normal((4 * d_s, d_s)))
    tf, ts, cnt = O.time_system(SA, c["nu"], np.ones(d_s), 16)
    rates["factor"], rates["solve"] = tf / cnt.factor, ts / cnt.solve
    parts.append(f"factorize {4 * d_s}x{d_s} + 16 solves: {tf + ts:.3f} s")
    return rates, "; ".join(parts), _t.perf_counter() - t_start


def extrapolate(rates, counters, d):
    """Seconds of a reference solve with these cost counters at these host rates (phase by phase)."""
    ph = {"sketch": counters["sketch"] * rates["sketch"]
                    + (counters["sketch"] / d) * rates.get("sketch_normal", 0.0),  # Gaussian: m n normals per m n d
          "factor": counters["factor"] * rates["factor"], "solve": counters["solve"] * rates["solve"],
          "gradient": counters["matvec"] * rates["matvec"]}
    return float(sum(ph.values())), ph


def load_ref_counters():
    try:
        return json.loads(REF_COUNTERS_PATH.read_text())
    except Exception:  # noqa: BLE001
        return {}


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
    """The reference arm: the reference's CPU implementation of the path (the oracle restatement, pinned to the
    reference's own headers by tests/test_ref_pin.py) on the host, single thread like the reference (no OpenMP
    in proj/CMakeLists.txt). C1/C2: one whole adaptive_solve per step. C3-C5: per step a bounded sample of the
    same workload timed phase by phase and extrapolated with the solve's cost counters (module docstring)."""
    from oracle import oracle as O
    if rank != 0:
        return 0
    if args.solver != "ihs" and args.config not in FULL_CPU_SOLVE:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.solver} CPU arm only for "
                          f"{'/'.join(FULL_CPU_SOLVE)}"}), flush=True)
        return 0
    full = args.config in FULL_CPU_SOLVE
    counters = None
    if full:
        A, b, _ = O.synth(c["n"], c["d"], spectrum=c["spectrum"], decay=c["decay"], noise_std=c["noise"],
                          outlier_frac=c["outliers"], data_seed=0)
        cfg = oracle_config(O, c)
    else:
        counters = load_ref_counters().get(args.config)
        if counters is None:
            print(json.dumps({"impl": "reference", "unavailable": f"no recorded cost counters for {args.config} "
                              f"in {REF_COUNTERS_PATH.name}"}), flush=True)
            return 0
    times, extra = [], {}
    warm = min(args.warmup, 1) if full else args.warmup  # a whole-solve step has no state to warm; printed as run
    for i in range(warm + args.steps):
        if full:
            t0 = time.perf_counter()
            if args.solver == "ihs":
                x, rep, log, _ = O.adaptive_solve(A, b, c["nu"], cfg)
                wall = rep.wall_seconds
                extra = {"iterations": int(rep.iterations), "rejections": int(rep.rejections),
                         "final_m": int(rep.final_m)}
            else:
                kind = 1 if c["sketch"] == "SRHT" else 0
                x, _, rep = (O.pcg_solve(A, b, c["nu"], kind, 0, PCG_RHO, CG_TOL, CG_MAX_ITERS)
                             if args.solver == "pcg" else O.cg_solve(A, b, c["nu"], CG_TOL, CG_MAX_ITERS))
                wall = time.perf_counter() - t0
                extra = {"iterations": int(rep.iterations)}
            sample = (f"one whole {args.solver} solve of {args.config.upper()} per step (oracle C++ restatement "
                      "of the reference, 1 thread)")
        else:
            rates, desc, spent = host_phase_rates(O, c, counters["final_m"])
            wall, phases = extrapolate(rates, counters, c["d"])
            extra = {"iterations": counters["iterations"], "rejections": counters["rejections"],
                     "final_m": counters["final_m"], "extrapolated_phase_s": phases,
                     "host_rates_s_per_unit": rates, "sample_seconds": spent}
            sample = (f"extrapolated: per step, bounded samples of {args.config.upper()} ({desc}) timed on the host "
                      "(1 thread), times the solve's cost counters from " + REF_COUNTERS_PATH.name)
        if i >= warm:
            times.append(wall)
    v = float(np.mean(times))
    line = {"impl": "reference", "metric": METRICS[args.solver], "value": v, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong" if world > 1 and not args.replicas else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d) generator)",
            "config": config_dict(args, c, world),
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_s": times, **extra}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- b200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="do not sample nvidia-smi during the timed steps")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of row sharding")
    ap.add_argument("--no-delta", action="store_true", help="skip the direct_solve accuracy check (profiling runs)")
    ap.add_argument("--record-counters", action="store_true",
                    help=f"write this config's solve counters into profiles/{REF_COUNTERS_PATH.name}")
    ap.add_argument("--solver", default="ihs", choices=["ihs", "pcg", "cg"],
                    help="ihs: adaptive Polyak-IHS (the headline); pcg / cg: the baselines.hpp comparators")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
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
    row0, rows = 0, n
    comm = None
    if sharded:
        row0, rows = ihs.shard_rows(n, world, rank)
        uid = [ihs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ihs.NcclComm(uid[0], world, rank, local)
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
        # the end-to-end solve must return what the device-timed one did (same data re-uploaded, same trail)
        same_x = bool(args.solver != "ihs" or np.array_equal(np.asarray(rep_e.x), np.asarray(reps[-1].x)))
        e2e = {"value": v, "unit": "s", "h2d_bytes_per_step": 8 * rows * d + 8 * rows, "d2h_bytes_per_step": 8 * d,
               "timer": "host wall clock around upload_async+solve (includes the H2D copies; work that does not "
                        "depend on the iterates runs chunk by chunk behind them: the SRHT sketches of the first "
                        "system and the next doublings with their Gram products, or the Gaussian S*A)", "x_matches_timed_solve": same_x}

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
    phases = {"gradient": t["gradient_ms"], "sketch": t["sketch_ms"], "factor": t["factor_ms"], "solve": t["solve_ms"],
              "total": t["total_ms"], "host_alloc": t["alloc_ms"], "host_rng": t["host_rng_ms"]}
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
            paths = {"srht_l2_kernel (single launch; T in an L2-resident column ring)": t.get("n_srht_l2", 0),
                     "srht_phase1_tma_kernel + srht_phase2_compact_kernel (compact T)": t.get("n_srht_compact", 0),
                     "srht_phase1_tma_kernel + srht_phase2_r2_kernel (T through HBM)": t.get("n_srht_two_kernel", 0)}
            kern["sketch"] = {"kernel": " | ".join(f"{k} x{v}" for k, v in paths.items() if v) or "srht",
                              "srht_paths": {"l2": paths[next(iter(paths))], "compact": t.get("n_srht_compact", 0),
                                             "two_kernel": t.get("n_srht_two_kernel", 0)},
                              "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                              "algorithmic_bytes_per_launch": t["sketch_bytes"] / t["n_sketch_kernel"],
                              "peak_source": peak_kind}
            # the two-pass transform writes every element twice into L2 (A's fill from HBM, then the phase-1
            # result T into the on-chip ring), and L2 absorbs writes at about the HBM rate: the L2-write roofline
            # (16 n d + 8 m d bytes per sketch against the measured L2 write bandwidth) is the one the launch sits on
            l2w = l2_write_peak()
            n_pad = 1 << (int(c["n"]) - 1).bit_length()
            l2_bytes = t["sketch_bytes"] + t["n_sketch_kernel"] * 8.0 * n_pad * c["d"]
            if l2w:
                a2 = l2_bytes / (sk_ms * 1e-3) / 1e9
                kern["sketch"]["l2_write_roofline"] = {
                    "bytes_per_launch": l2_bytes / t["n_sketch_kernel"], "achieved": a2, "peak": l2w, "unit": "GB/s",
                    "frac": a2 / l2w, "peak_source": "measured (tools/l2_bw.cu: L2-resident whole-line stores, "
                                                     "profiles/l2_bw.json)"}
        else:
            ach = t["sketch_flops"] / (sk_ms * 1e-3) / 1e12
            kern["sketch"] = {"kernel": "dgemm_nn_big_kernel S*A (128x128 cp.async tiles, mma.sync m8n8k4 f64 = "
                                        "DMMA)", "bound": "tensor",
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

    # ---- accuracy of the returned x against the exact minimizer (problem.hpp:73-82, 104-109), off the clock
    acc = {}
    if args.solver == "ihs" and not args.no_delta:
        try:
            x_star = ihs.direct_solve(p)
            pe0 = ihs.prediction_error(p, np.zeros(d), x_star)
            pe = ihs.prediction_error(p, last.x, x_star)
            acc = {"delta_rel_vs_direct": float(np.sqrt(pe / pe0)), "pe_rel": float(pe / pe0),
                   "delta_target": 1e-10, "meets_target": bool(np.sqrt(pe / pe0) <= 1e-10)}
        except Exception as e:  # noqa: BLE001
            acc = {"delta_rel_vs_direct": None, "delta_error": str(e)[:200]}
    counters = {"sketch": last.counters.sketch, "factor": last.counters.factor, "solve": last.counters.solve,
                "matvec": last.counters.matvec} if args.solver == "ihs" else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        if args.config in FULL_CPU_SOLVE:
            t0 = time.perf_counter()
            if args.solver == "ihs":
                x_ref, orep, olog, _ = O.adaptive_solve(A, b, nu, oracle_config(O, c))
                cpu = {"value": float(orep.wall_seconds), "unit": "s", "cores": 1, "kind": "port",
                       "sample": f"one whole adaptive_solve of {args.config.upper()} (oracle C++ restatement of the "
                                 "reference, 1 thread)",
                       "same_m_schedule": bool([(e[0], e[1], e[4]) for e in olog] ==
                                               [(e.t, e.m, int(e.branch)) for e in last.log]),
                       "same_counters": bool((orep.counters.sketch, orep.counters.factor, orep.counters.solve,
                                              orep.counters.matvec) == tuple(counters.values()))}
            else:
                x_ref, _, orep = (O.pcg_solve(A, b, nu, int(kind), 0, PCG_RHO, CG_TOL, CG_MAX_ITERS)
                                  if args.solver == "pcg" else O.cg_solve(A, b, nu, CG_TOL, CG_MAX_ITERS))
                cpu = {"value": time.perf_counter() - t0, "unit": "s", "cores": 1, "kind": "port",
                       "sample": f"one whole {args.solver} solve of {args.config.upper()} (oracle, 1 thread)",
                       "iterations": int(orep.iterations), "same_iterations": int(orep.iterations) == last.iterations}
            Ad = np.concatenate([A @ (last.x - x_ref), nu * (last.x - x_ref)])
            Ar = np.concatenate([A @ x_ref, nu * x_ref])
            cpu["abar_rel_err_vs_oracle"] = float(np.linalg.norm(Ad) / np.linalg.norm(Ar))
        elif args.solver == "ihs":
            rates, desc, spent = host_phase_rates(O, c, last.final_m)
            v, phases = extrapolate(rates, counters, d)
            cpu = {"value": v, "unit": "s", "cores": 1, "kind": "port",
                   "sample": f"extrapolated: bounded samples of {args.config.upper()} ({desc}) timed on the host "
                             "(oracle restatement, 1 thread) x this solve's cost counters",
                   "extrapolated_phase_s": phases, "host_rates_s_per_unit": rates, "sample_seconds": spent}
        else:
            cpu = {"value": None, "unit": "s", "cores": 1, "kind": "port",
                   "sample": f"not run: the single-thread {args.solver} of this config exceeds the bench budget"}

    if rank == 0:
        if args.solver == "ihs":
            summary = {"iterations": last.iterations, "rejections": last.rejections, "final_m": last.final_m,
                       "converged": last.converged, "m_schedule": [e.m for e in last.log if int(e.branch) == 2],
                       **acc, "counters": counters}
            rec = load_ref_counters().get(args.config)
            if rec is not None and world == 1:
                summary["counters_match_recorded"] = rec == {**counters, "iterations": last.iterations,
                                                             "rejections": last.rejections, "final_m": last.final_m}
            if args.record_counters and world == 1:
                allc = load_ref_counters()
                allc[args.config] = {**counters, "iterations": last.iterations, "rejections": last.rejections,
                                     "final_m": last.final_m}
                REF_COUNTERS_PATH.write_text(json.dumps(allc, indent=1, sort_keys=True) + "\n")
        else:
            summary = {"iterations": last.iterations, "converged": last.converged, "m": last.m,
                       "m_capped": last.m_capped, "residual_ratio": last.residuals[-1] / last.residuals[0]}
        summary.update({"lib_total_ms": float(np.mean(lib_ms)), "step_ms": step_ms,
                        "kernel_launches_per_solve": t["kernel_launches"]})
        line = {"metric": METRICS[args.solver], "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
                "scaling": "strong" if sharded else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded SURVEY §8(d) generator: A = G diag(sigma), x_true, noise)",
                "config": config_dict(args, c, world),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks,
                "solve": summary,
                "datagen_s": gen_s}
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            pathlib.Path(args.out).write_text(s + "\n")
    # the NCCL communicator is destroyed explicitly (all work synchronized above), before the process group and
    # before interpreter shutdown could collect it in any order
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
