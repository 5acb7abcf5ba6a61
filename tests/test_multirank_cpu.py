"""World-size-2 gloo tests (CPU) of the query-sharded multi-GPU design.

The GPU path shards queries in Morton order with `wn_shard_range`, exchanges the owned rows after each
traversal and reduces the per-256-query-block Σ partials in a fixed global order, so every rank — and
every world size — follows the single-GPU trajectory bit for bit.  Here each rank runs the same
schedule with the oracle's operators on its own shard, exchanges through torch.distributed (gloo), and
the result must equal the world-size-1 run exactly.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import OP_A, OP_AT, OP_G
from paper_2405_16634_b200 import synth

BLOCK = 256


def _shard(n, rank, world):
    import paper_2405_16634_b200.wn as wn  # host-only call: no GPU needed

    return wn.wn_shard_range(n, rank, world)


def _allgather_rows(local, n, rank, world, dim):
    """Owned rows [b, e) of a sorted-order n×dim array → the full array on every rank."""
    full = torch.zeros(n * dim, dtype=torch.float64)
    b, e = _shard(n, rank, world)
    full[b * dim:e * dim] = torch.from_numpy(local.reshape(-1))
    if world > 1:
        dist.all_reduce(full)  # disjoint rows: the sum is the concatenation (exact: x + 0 = x)
    return full.numpy().reshape(n, dim) if dim > 1 else full.numpy()


def _sharded_solve(rank, world, pts, iters):
    cl = oracle.Cloud(pts)
    t = cl.t
    perm = t.export()["perm"].astype(np.int64)  # Morton order (the GPU's query order)
    n = len(pts)
    b, e = _shard(n, rank, world)
    nb = (n + BLOCK - 1) // BLOCK
    mu = np.zeros((n, 3))  # normalized frame, caller order
    w1, w2 = float(np.float32(0.002)), float(np.float32(0.016))
    alphas = []
    for k in range(1, iters + 1):
        w = float(np.float32(oracle.width_schedule(k, 40, w1, w2)))
        q = perm[b:e]

        def partials(vals):  # Σ over globally aligned 256-query blocks (sorted order), fixed order
            loc = np.zeros(nb)
            for i, v in zip(range(b, e), vals):
                loc[i // BLOCK] += v
            out = torch.from_numpy(loc)
            if world > 1:
                dist.all_reduce(out)  # each block is owned by exactly one rank
            return out.numpy()

        s_loc = 0.5 - t.tree(OP_A, mu, w, 2.0, qidx=q)
        s_sorted = _allgather_rows(s_loc, n, rank, world, 1)
        ps = partials(s_loc ** 2)
        s = np.empty(n)
        s[perm] = s_sorted
        r_loc = t.tree(OP_AT, s, w, 2.0, qidx=q)
        r_sorted = _allgather_rows(r_loc, n, rank, world, 3)
        pr = partials(np.sum(r_loc ** 2, axis=1))
        r = np.empty((n, 3))
        r[perm] = r_sorted
        qv = t.tree(OP_A, r, w, 2.0, qidx=q)
        pq = partials(qv ** 2)
        rr, qq = float(np.sum(pr)), float(np.sum(pq))  # fixed order over all blocks
        alpha = rr / qq if qq > 0 else 0.0
        alphas.append((float(np.sum(ps)), alpha))
        mp_ = mu + alpha * r
        g_loc = t.tree(OP_G, mp_, w, 2.0, qidx=q)
        a = np.linalg.norm(mp_[q], axis=1)
        h = np.linalg.norm(g_loc, axis=1)
        new_loc = np.where(h[:, None] > 0, g_loc * (a / np.where(h > 0, h, 1))[:, None], mp_[q])
        mu_sorted = _allgather_rows(new_loc, n, rank, world, 3)
        mu = np.empty((n, 3))
        mu[perm] = mu_sorted
    return mu, alphas


def _worker(rank, world, port, pts, iters, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mu, alphas = _sharded_solve(rank, world, pts, iters)
        np.save(os.path.join(outdir, f"mu_{rank}.npy"), mu)
        np.save(os.path.join(outdir, f"alpha_{rank}.npy"), np.array(alphas))
    finally:
        dist.destroy_process_group()


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [1500, 3001])
def test_two_rank_sharded_iteration_is_bit_identical(n):
    pts = synth.sphere(n, seed=21)[0]
    iters = 3
    ref_mu, ref_alpha = _sharded_solve(0, 1, pts, iters)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), pts, iters, d), nprocs=2, join=True, start_method="spawn")
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"mu_{r}.npy")), ref_mu)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"alpha_{r}.npy")), np.array(ref_alpha))
    # and the sharded schedule is the oracle's own solver up to summation order
    cl = oracle.Cloud(pts)
    mu_o, st = cl.t.solve(iters=iters, total_iters=40, w1=float(np.float32(0.002)), w2=float(np.float32(0.016)))
    np.testing.assert_allclose(ref_mu, mu_o, rtol=1e-9, atol=1e-12 * np.abs(mu_o).max())
    np.testing.assert_allclose([a for _, a in ref_alpha], st[:, 1], rtol=1e-9)


def test_shards_align_to_partial_blocks():
    for n in (1000, 500000):
        for world in (2, 4, 8):
            for r in range(world):
                b, e = _shard(n, r, world)
                assert b % BLOCK == 0 and (e % BLOCK == 0 or e == n)
