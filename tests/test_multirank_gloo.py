"""The N > 1 path's host-side math on CPU, with real multi-process exchange
(torch.distributed, gloo, world_size 2 and 4).

Each rank takes its row shard (ihs.shard_rows: rows [r*n_loc, (r+1)*n_loc) of
the padded index space), computes what the CUDA shard kernels compute — the
sign flip and the low-bit butterflies of its block, the unscaled partial at
r_lo(k) for every sampled row, and the gradient partial A_r^T(A_r x - b_r) —
exchanges them (all_gather / all_reduce, the NCCL collectives of the device
path), and combines them in the reference's stage order. The combined SRHT
sketch must equal the oracle's single-process srht_sketch bit for bit, and
the gradient must match to fp64 tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def fwht_unnormalized(v):
    """Radix-2 butterflies h = 1, 2, ... (sketch.hpp:37-46) along axis 0, no scaling."""
    v = v.copy()
    n = v.shape[0]
    h = 1
    while h < n:
        w = v.reshape(n // (2 * h), 2, h, *v.shape[1:])
        a = w[:, 0].copy()
        b = w[:, 1].copy()
        w[:, 0] = a + b
        w[:, 1] = a - b
        h *= 2
    return v


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        from oracle import oracle as O
        from paper_2006_05874_b200 import ihs

        n, d, m, seed, nu = case
        A, b, _ = O.synth(n, d, decay=0.9, noise_std=0.05, outlier_frac=0.01, data_seed=3)
        n_pad = O.next_pow2(n)
        row0, rows = ihs.shard_rows(n, world, rank)
        n_loc = n_pad // world
        assert row0 == rank * n_loc and rows == min(n_loc, n - row0)
        # ---- SRHT partial of this shard (what srht_plan_shard + srht_run_device compute)
        eps = O.rademacher(O.derive_seed(seed, 1), n_pad)
        P = O.sample_without_replacement(O.derive_seed(seed, 2), n_pad, m)
        B = np.zeros((n_loc, d))
        B[:rows] = eps[row0:row0 + rows, None] * A[row0:row0 + rows]
        T = fwht_unnormalized(B)
        U_r = np.ascontiguousarray(T[P % n_loc])  # m x d, unscaled
        parts = [torch.zeros(m, d, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(U_r))
        U = np.stack([t.numpy() for t in parts])  # [P][m][d], rank-major like ncclAllGather
        V = fwht_unnormalized(U)  # top log2(P) stages over the shard index, in order
        hi = P // n_loc
        comb = V[hi, np.arange(m)]
        s1 = 1.0 / np.sqrt(float(n_pad))
        s2 = np.sqrt(float(n_pad) / float(m))
        SA = (comb * s1) * s2
        ok_srht = bool(np.array_equal(SA, O.srht_sketch(A, m, seed)))
        # ---- owner-reduce exchange (the device path, runtime.cpp device_sketch): row k is owned by rank
        # k // mq; an all-to-all hands each owner the P partials of its rows, the owner runs the top stages over
        # the shard index in order, and an all-gather assembles SA on every rank
        mq = -(-m // world)
        send = np.zeros((world, mq, d))
        for k in range(m):
            send[k // mq, k % mq] = U_r[k]
        recv = torch.zeros(world * mq * d, dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send.reshape(-1)))
        Vq = fwht_unnormalized(recv.numpy().reshape(world, mq, d))  # [source rank p][my rows][d]
        mine = np.zeros((mq, d))
        for kk in range(mq):
            k = rank * mq + kk
            if k < m:
                mine[kk] = (Vq[hi[k], kk] * s1) * s2
        blocks = [torch.zeros(mq * d, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(blocks, torch.from_numpy(mine.reshape(-1)))
        SA_or = np.concatenate([t.numpy().reshape(mq, d) for t in blocks])[:m]
        ok_srht = ok_srht and bool(np.array_equal(SA_or, SA))
        # ---- split SYRK (system_factorize with split_comm): this rank's ceil(m/P) rows of the replicated SA
        # (Gram), or its ceil(d/P) columns (Woodbury inner), then an all-reduce of the k x k partials
        r0 = min(m, rank * mq)
        G = torch.from_numpy(np.ascontiguousarray(SA[r0:r0 + mq].T @ SA[r0:r0 + mq]))
        dist.all_reduce(G)
        dq = -(-d // world)
        c0 = min(d, rank * dq)
        Ii = torch.from_numpy(np.ascontiguousarray(SA[:, c0:c0 + dq] @ SA[:, c0:c0 + dq].T))
        dist.all_reduce(Ii)
        G_ref, I_ref = SA.T @ SA, SA @ SA.T
        ok_srht = ok_srht and bool(np.linalg.norm(G.numpy() - G_ref) <= 1e-13 * np.linalg.norm(G_ref) * world)
        ok_srht = ok_srht and bool(np.linalg.norm(Ii.numpy() - I_ref) <= 1e-13 * np.linalg.norm(I_ref) * world)
        # ---- gradient partial + all_reduce (+ nu^2 x once)
        x = np.random.default_rng(7).standard_normal(d)
        Ar, br = A[row0:row0 + rows], b[row0:row0 + rows]
        g = torch.from_numpy(Ar.T @ (Ar @ x - br))
        dist.all_reduce(g)
        g = g.numpy() + nu * nu * x
        g_ref = O.gradient(A, b, nu, x)
        ok_grad = bool(np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref) * np.sqrt(n))
        q.put((rank, ok_srht, ok_grad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (1000, 5, 64, 11, 0.1)),        # n not a power of two: the last shard is partly virtual
    (2, (4096, 3, 4096, 2, 0.05)),      # full sampling
    (4, (3500, 4, 333, 5, 0.2)),
    (4, (8192, 2, 1000, 9, 0.3)),
])
def test_sharded_srht_and_gradient_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in results) == list(range(world))
    assert all(r[1] for r in results), "sharded SRHT / owner-reduce / split Gram differs from the single process"
    assert all(r[2] for r in results), "sharded gradient differs from the oracle"


def test_shard_rows_rules(ihs):
    assert ihs.shard_rows(1 << 20, 8, 3) == (3 << 17, 1 << 17)
    assert ihs.shard_rows(10**6, 8, 7) == (7 << 17, 10**6 - (7 << 17))
    with pytest.raises(ihs.InvalidInput):
        ihs.shard_rows(100, 8, 0)  # fewer than 32 padded rows per shard
    with pytest.raises(ihs.InvalidInput):
        ihs.shard_rows(3000, 4, 3)  # n_pad = 4096: shard 3 = [3072, 4096) holds no real row
    assert ihs.shard_rows(600, 2, 1) == (512, 88)
