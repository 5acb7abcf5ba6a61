"""The NCCL exchange path of wnnc_iterate on the one GPU of this run (a world-size-1 communicator):
every collective runs (grouped broadcasts, schedule pack / unpack, partial exchange) and the trajectory
must be bit-identical to the single-GPU path.  Multi-rank logic: tests/test_multirank_cpu.py."""
import numpy as np
import pytest

from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wn():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    return wn


def test_world1_comm_matches_single_gpu(wn):
    # single GPU; peer-memory exchange (default: epilogue stores into every replica + signal / wait),
    # with and without the CUDA graph; NCCL broadcasts, with and without the graph — one trajectory
    uid = wn.wn_comm_unique_id()
    assert len(uid) == 128
    comm = wn.wn_comm_init(0, 1, uid)
    p = torch.from_numpy(synth.config("C2")["points"]).cuda()
    outs = []
    G, NC = wn.WN_FLAG_GRAPH, wn.WN_FLAG_COMM_NCCL
    for c, flags in ((None, 0), (comm, 0), (comm, G), (comm, NC), (comm, NC | G), (comm, G)):
        t = wn.wn_build_tree(p)
        mu = torch.zeros(len(p), 3, device="cuda")
        st = wn.wnnc_iterate(t, mu, comm=c, stats=True, iters=5, total_iters=40, flags=flags)
        outs.append((mu.cpu().numpy(), [s["alpha"] for s in st]))
    for m, a in outs[1:]:
        np.testing.assert_array_equal(m, outs[0][0])
        assert a == outs[0][1]
    comm.close()


def _close(a, b):
    # two transpose-mode trajectories: the scatter's fp64 atomics add in a run-dependent order, so equal up to
    # rounding (after 5 iterations: 1e-4 of the largest |μ| per entry) and every orientation the same
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-4 * np.abs(b).max())
    assert np.all(np.sum(a * b, axis=1) > 0)


def test_world1_comm_transpose(wn):
    # the multi-GPU form of the transpose-mode adjoint on a world-1 communicator: peer path (scatter into the
    # arena's accumulators, signal, wait, rank-order sum, replicated push-down; stream and graph) and NCCL
    # (all-reduce of the accumulators) — the single-GPU transpose trajectory up to the atomics' rounding
    comm = wn.wn_comm_init(0, 1, wn.wn_comm_unique_id())
    p = torch.from_numpy(synth.config("C2")["points"]).cuda()
    T, G, NC = wn.WN_ADJ_TRANSPOSE, wn.WN_FLAG_GRAPH, wn.WN_FLAG_COMM_NCCL
    outs = []
    for c, flags in ((None, 0), (comm, 0), (comm, G), (comm, NC)):
        t = wn.wn_build_tree(p)
        mu = torch.zeros(len(p), 3, device="cuda")
        wn.wnnc_iterate(t, mu, comm=c, iters=5, total_iters=40, flags=flags, adjoint_mode=T)
        outs.append(mu.cpu().numpy())
    for m in outs[1:]:
        _close(m, outs[0])
    comm.close()


@pytest.mark.parametrize("world,n", [(2, 30011), (3, 70001), (8, 30011), (8, 1000)])
def test_emulated_ranks_transpose(wn, world, n):
    # W emulated ranks, transpose-mode adjoint (SURVEY §8(e) + row a7): each rank scatters its shard into its
    # own accumulators, every rank adds all ranks' in rank order and pushes down for all points — every
    # replica is the same bit for bit, and the trajectory is the single-GPU transpose one up to rounding
    # (1000 points over 8 ranks: shards of 256 queries, so some ranks have none and only signal)
    p = torch.from_numpy(synth.config("C2" if n <= 50000 else "C3")["points"][:n]).cuda()
    t = wn.wn_build_tree(p)
    T = wn.WN_ADJ_TRANSPOSE
    ref = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, ref, iters=5, total_iters=40, adjoint_mode=T)
    mu = torch.zeros(len(p), 3, device="cuda")
    reps = wn.wnnc_iterate_emulated(t, mu, world, iters=5, total_iters=40, adjoint_mode=T).cpu().numpy()
    for r in range(1, world):
        np.testing.assert_array_equal(reps[r], reps[0])
    _close(reps[0], ref.cpu().numpy())


def test_peer_arena_grows_with_n(wn):
    # one communicator, clouds of increasing size: the peer-memory arena is rebuilt (collectively) and the
    # cached graph re-captured; every run still equals the single-GPU trajectory
    comm = wn.wn_comm_init(0, 1, wn.wn_comm_unique_id())
    for cfg, n in (("C1", None), ("C2", 20000), ("C2", None), ("C1", None)):
        pts = synth.config(cfg)["points"]
        p = torch.from_numpy(pts[:n] if n else pts).cuda()
        res = []
        for c in (None, comm):
            t = wn.wn_build_tree(p)
            mu = torch.zeros(len(p), 3, device="cuda")
            wn.wnnc_iterate(t, mu, comm=c, iters=3, total_iters=40, flags=wn.WN_FLAG_GRAPH)
            res.append(mu.cpu().numpy())
        np.testing.assert_array_equal(res[1], res[0])
    comm.close()


@pytest.mark.parametrize("world,n", [(2, 30011), (3, 30011), (8, 30011), (3, 70001)])
def test_emulated_ranks_match_single_gpu(wn, world, n):
    # W ranks of the peer-memory exchange emulated on this GPU (each rank's shard reads its own replica
    # and stores into all W replicas; signals / waits with world-W targets; ping-pong μ): every replica
    # must hold the single-GPU trajectory bit for bit — below 60k queries through the split traversal,
    # above through the one-warp kernel
    p = torch.from_numpy(synth.config("C2" if n <= 50000 else "C3")["points"][:n]).cuda()
    t = wn.wn_build_tree(p)
    ref = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, ref, iters=5, total_iters=40)
    mu = torch.zeros(len(p), 3, device="cuda")
    reps = wn.wnnc_iterate_emulated(t, mu, world, iters=5, total_iters=40)
    np.testing.assert_array_equal(mu.cpu().numpy(), ref.cpu().numpy())
    for r in range(world):
        np.testing.assert_array_equal(reps[r].cpu().numpy(), ref.cpu().numpy())


@pytest.mark.parametrize("order", [0, 1])
def test_mu_zero_flag_is_exact(wn, order):
    # WN_FLAG_MU_ZERO (iteration 1 takes A(0) = 0, s = ½, without the traversal) reproduces the computed
    # first iteration bit for bit: single GPU (stream and graph), NCCL world 1, 3 emulated ranks
    p = torch.from_numpy(synth.config("C2")["points"][:20011]).cuda()
    t = wn.wn_build_tree(p)
    wn.wn_tree_set_far_order(t, order)
    Z, G = wn.WN_FLAG_MU_ZERO, wn.WN_FLAG_GRAPH
    out = []
    for flags in (0, Z, Z | G):
        mu = torch.zeros(len(p), 3, device="cuda")
        st = wn.wnnc_iterate(t, mu, stats=True, iters=4, total_iters=40, flags=flags)
        out.append((mu.cpu().numpy(), [(x["E"], x["alpha"]) for x in st]))
    comm = wn.wn_comm_init(0, 1, wn.wn_comm_unique_id())
    mu = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, mu, comm=comm, iters=4, total_iters=40, flags=Z | wn.WN_FLAG_COMM_NCCL)
    out.append((mu.cpu().numpy(), out[0][1]))
    comm.close()
    mu = torch.zeros(len(p), 3, device="cuda")
    reps = wn.wnnc_iterate_emulated(t, mu, 3, iters=4, total_iters=40, flags=Z)
    out.append((reps[2].cpu().numpy(), out[0][1]))
    for m, st in out[1:]:
        np.testing.assert_array_equal(m, out[0][0])
        assert st == out[0][1]


def test_emulated_ranks_first_order(wn):
    # the first-order far field (row f2) through the sharded peer exchange: 3 emulated ranks, one trajectory
    p = torch.from_numpy(synth.config("C2")["points"][:30011]).cuda()
    t = wn.wn_build_tree(p)
    wn.wn_tree_set_far_order(t, 1)
    ref = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, ref, iters=4, total_iters=40)
    mu = torch.zeros(len(p), 3, device="cuda")
    reps = wn.wnnc_iterate_emulated(t, mu, 3, iters=4, total_iters=40)
    for r in range(3):
        np.testing.assert_array_equal(reps[r].cpu().numpy(), ref.cpu().numpy())


def test_shard_plan_balances_work(wn):
    # the work-weighted shards of an 8-rank solve of the non-uniform C3 cloud: block-aligned, covering,
    # and balanced on the actual per-query work (node tests and live terms of A) where equal counts are not
    c = synth.config("C3")
    p = torch.from_numpy(c["points"]).cuda()
    n = len(p)
    t = wn.wn_build_tree(p)
    pl = wn.wn_shard_plan(t, 8)
    assert pl[0] == 0 and pl[-1] == n and all(b % 256 == 0 for b in pl[:-1]) and pl == sorted(pl)
    mu = torch.from_numpy((synth.random_signs(c["normals"], 7) * (4 * np.pi / n)).astype(np.float32)).cuda()
    cnt = wn.wn_query_work(t, mu, 0.004, op=0).cpu().numpy().astype(np.int64)
    perm = wn.wn_tree_export(t)["perm"].cpu().numpy()
    work = (cnt[:, 0] * 13 + cnt[:, 3] * 10)[perm[wn.wn_tree_schedule(t).cpu().numpy()]]
    wp = np.array([work[pl[r]:pl[r + 1]].sum() for r in range(8)])
    we = np.array([work[b:e].sum() for b, e in (wn.wn_shard_range(n, r, 8) for r in range(8))])
    assert wp.max() / wp.mean() < 1.02 < we.max() / we.mean()


def test_comm_init_errors(wn):
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wn_comm_init(2, 2, bytes(128))
