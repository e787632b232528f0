"""The library's REAL row-sharded code path (world_size > 1) on one device: P emulated ranks
(ihs_gpu_emu_comm_create), one host thread per rank, each with its own problem handle on its shard of the rows
(ihs.shard_rows: rows [r n_loc, (r+1) n_loc) of the padded index space) — the sharded SRHT transform and
exchange, the Gaussian sketch window + all-reduce, the gradient all-reduce and a full adaptive_solve, exactly as
`bench.py --gpus N` runs them over NCCL, with device copies standing in for NCCL (no kernel waits on another).

Checks (sketch.hpp:58-108, problem.hpp:59-69, solver.hpp:106-232):
* every rank holds the same bytes after each collective (SA, gradients, the solution);
* the sharded SRHT sketch — owner-reduce exchange: an all-to-all of owner blocks, the exact butterfly combine by
  each row's owner and an all-gather, ~2 m d doubles received per rank — equals the single-GPU (and oracle)
  sketch bit for bit, including m not divisible by P and m < P;
* Gaussian sketches / gradients equal the single-GPU ones to fp64 tolerance (partial sums in another order);
* the sharded adaptive solve takes the single-GPU solve's m-schedule, branches and counters and returns x within
  1e-10 of it in the Abar norm.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(P, fn):
    out, err = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            err.append((r, e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank thread hung"
    assert not err, err
    return out


def _shards(gpu, A, b, nu, P):
    n = A.shape[0]
    comms = gpu.EmuComm.group(P)
    probs = []
    for r in range(P):
        row0, rows = gpu.shard_rows(n, P, r)
        probs.append(gpu.ProblemInstance(np.asfortranarray(A[row0:row0 + rows]), b[row0:row0 + rows].copy(), nu,
                                         world_size=P, rank=r, comm=comms[r], n_global=n))
    return comms, probs


def _abar_rel(A, nu, x, xr):
    num = np.linalg.norm(np.concatenate([A @ (x - xr), nu * (x - xr)]))
    den = np.linalg.norm(np.concatenate([A @ xr, nu * xr]))
    return num / den


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_sketches_and_gradient(gpu, O, P):
    n, d = 60000, 24  # n_pad = 65536: every rank holds rows, the last one a ragged block
    A, b, _ = gpu.synth_generate(n, d, decay=0.95, noise_std=0.01, data_seed=5)
    nu = 1e-2
    comms, probs = _shards(gpu, A, b, nu, P)
    single = gpu.ProblemInstance(A, b, nu)
    x = np.random.default_rng(P).standard_normal(d)

    def work(r):
        p = probs[r]
        return (gpu.srht_sketch(p, 3000, 7), gpu.srht_sketch(p, 64, 8), gpu.gaussian_sketch(p, 200, 9),
                gpu.gradient(p, x), gpu.srht_sketch(p, 1001, 11), gpu.srht_sketch(p, 1, 12))

    res = _run_ranks(P, work)
    for r in range(1, P):
        for a, b_ in zip(res[0], res[r]):
            assert np.array_equal(a, b_), f"rank {r} differs from rank 0"
    SA_s, SA_s2, SA_g, g, SA_odd, SA_one = res[0]
    assert np.array_equal(SA_s, O.srht_sketch(A, 3000, 7))
    # m not a multiple of P (ragged last owner block) and m = 1 (owners without rows)
    assert np.array_equal(SA_odd, O.srht_sketch(A, 1001, 11))
    assert np.array_equal(SA_one, O.srht_sketch(A, 1, 12))
    assert np.array_equal(SA_s2, gpu.srht_sketch(single, 64, 8))
    ref = gpu.gaussian_sketch(single, 200, 9)
    assert np.max(np.abs(SA_g - ref)) <= 1e-12 * np.max(np.abs(ref))
    g1 = gpu.gradient(single, x)
    assert np.max(np.abs(g - g1)) <= 1e-12 * np.max(np.abs(g1))
    del probs, comms


@pytest.mark.parametrize("P,n", [(2, (1 << 21) - 3), (4, (1 << 22) - 5), (2, (1 << 23) - 7)])
def test_sharded_srht_l2_resident(gpu, O, P, n):
    """Shards of 2^20..2^22 padded rows (10..12 high bits) take the L2-resident launch with the owner-block
    emission: bit-identical to the single-GPU sketch, and to the oracle, with ragged last shards."""
    d = 2
    A = np.asfortranarray(np.random.default_rng(n % 97).standard_normal((n, d)))
    b = np.zeros(n)
    comms, probs = _shards(gpu, A, b, 1e-2, P)
    single = gpu.ProblemInstance(A, b, 1e-2)
    ms = (4097, 70001)

    def work(r):
        return [gpu.srht_sketch(probs[r], m, 31 + m) for m in ms]

    res = _run_ranks(P, work)
    for r in range(1, P):
        for a, b_ in zip(res[0], res[r]):
            assert np.array_equal(a, b_), f"rank {r} differs from rank 0"
    for m, SA in zip(ms, res[0]):
        assert np.array_equal(SA, gpu.srht_sketch(single, m, 31 + m)), f"m={m}: sharded L2 sketch differs"
    assert np.array_equal(res[0][0], O.srht_sketch(A, ms[0], 31 + ms[0]))
    del probs, comms


@pytest.mark.parametrize("P,kind", [(2, "SRHT"), (4, "SRHT"), (8, "SRHT"), (2, "Gaussian"), (4, "Gaussian")])
def test_sharded_adaptive_solve(gpu, P, kind):
    n, d = 60000, 48
    A, b, _ = gpu.synth_generate(n, d, decay=0.97, noise_std=0.01, data_seed=6)
    nu = 1e-3
    cfg = gpu.SolverConfig(sketch_kind=getattr(gpu.SketchKind, kind), m_initial=2 * d, eps=1e-21, seed=3)
    comms, probs = _shards(gpu, A, b, nu, P)
    reps = _run_ranks(P, lambda r: gpu.adaptive_solve(probs[r], cfg))
    ref = gpu.adaptive_solve(gpu.ProblemInstance(A, b, nu), cfg)
    for r in range(P):
        assert np.array_equal(reps[r].x, reps[0].x)
        assert [(e.t, e.m, int(e.branch)) for e in reps[r].log] == [(e.t, e.m, int(e.branch)) for e in ref.log]
        c, c1 = reps[r].counters, ref.counters
        assert (c.sketch, c.factor, c.solve, c.matvec) == (c1.sketch, c1.factor, c1.solve, c1.matvec)
    assert reps[0].converged and reps[0].iterations > 1
    assert _abar_rel(A, nu, reps[0].x, ref.x) <= 1e-10
    del probs, comms


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_gaussian_generation_is_one_pth(gpu, P):
    """Each shard counts only its share of the stream's substreams (counts all-gathered) and emits only the
    substreams reaching into its own window, so its generation work is ~2/P of the single-GPU generator's
    (which counts and emits the whole stream), and the sketch is unchanged."""
    n, d, m = 60000, 16, 512
    A, b, _ = gpu.synth_generate(n, d, decay=0.95, noise_std=0.01, data_seed=7)
    comms, probs = _shards(gpu, A, b, 1e-2, P)

    def work(r):
        d0 = gpu.thread_generated_draws()
        SA = gpu.gaussian_sketch(probs[r], m, 21)
        return SA, gpu.thread_generated_draws() - d0

    res = _run_ranks(P, work)
    single = gpu.ProblemInstance(A, b, 1e-2)
    d0 = gpu.thread_generated_draws()
    ref = gpu.gaussian_sketch(single, m, 21)
    total = gpu.thread_generated_draws() - d0
    for SA, _ in res:
        assert np.array_equal(SA, res[0][0])
    assert np.max(np.abs(res[0][0] - ref)) <= 1e-12 * np.max(np.abs(ref))
    # one pass over the stream = total / 2 draws; shard r counts a 1/P share of the substreams and emits those
    # covering its rows (rows_r / n of the stream: shards are n_pad / P rows, the last ones shorter), plus at most
    # a couple of boundary substreams
    one_pass = total / 2
    for r, (_, draws) in enumerate(res):
        rows = gpu.shard_rows(n, P, r)[1]
        bound = one_pass * (1.0 / P + rows / n) + 4 * (1 << 18)
        assert draws <= bound, (r, draws, bound, total, P)
        assert draws < 0.8 * total  # well below the single-GPU generator's work
    del probs, comms


def test_sharded_gaussian_two_level_plan(gpu):
    """Long streams count over few jump substreams and dump the emitting windows (IHS_GAUSS_MAX_JUMP_SUBS forces
    that plan here): the sharded Gaussian sketch still equals the single-GPU one on every rank."""
    import os
    import subprocess
    import sys
    code = ("import sys, threading\n"
            "sys.path.insert(0, 'tests')\n"
            "import numpy as np\n"
            "from paper_2006_05874_b200 import ihs\n"
            "import test_gpu_sharded_emu as T\n"
            "A, b, _ = ihs.synth_generate(60000, 8, decay=0.95, noise_std=0.01, data_seed=9)\n"
            "ref = ihs.gaussian_sketch(ihs.ProblemInstance(A, b, 1e-2), 300, 5)\n"
            "for P in (2, 4):\n"
            "    comms, probs = T._shards(ihs, A, b, 1e-2, P)\n"
            "    res = T._run_ranks(P, lambda r: ihs.gaussian_sketch(probs[r], 300, 5))\n"
            "    for SA in res:\n"
            "        assert np.array_equal(SA, res[0]) and np.max(np.abs(SA - ref)) <= 1e-12 * np.max(np.abs(ref))\n"
            "print('ok')\n")
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root,
                       env=dict(os.environ, IHS_GAUSS_MAX_JUMP_SUBS="5"))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
