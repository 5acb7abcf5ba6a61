"""The multi-GPU peer-memory exchange across real processes (needs a GPU).

SURVEY §8(e) / DESIGN.md §8: every rank traverses its shard of the query schedule and its traversal epilogues
store the owned rows and Σ partials straight into every rank's replica (CUDA IPC mappings), the last block
of each launch signals every rank with a system-scope atomic, and the next step waits for all signals.
This test runs that code — cudaIpcGetMemHandle / cudaIpcOpenMemHandle between processes, remote stores into
another process's allocation, cross-process `atomicAdd_system` signals, the work-weighted shard plan — with
W processes on ONE GPU.  Kernels of different processes must never wait on one another on one GPU (they may
not run concurrently; the profiling guide records Xid 109 for exactly that), so the ranks use
WN_FLAG_HOST_WAIT: the host synchronizes its stream and polls its signal word, and every kernel finishes on
its own.  The arena handles travel through torch.distributed (gloo), since NCCL refuses two ranks on one
device.  Every rank must end with the single-GPU trajectory, bit for bit (the sharding only decides which
rank computes which rows; partials are reduced in one fixed order).
"""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_PTS, ITERS = 100003, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_dir, adjoint_mode=0):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2405_16634_b200.wn as wn

        p = synth.config("C3", n=N_PTS)["points"]
        tree = wn.wn_build_tree(torch.from_numpy(p).cuda())
        comm = wn.wn_comm_init_local(rank, world)
        h = wn.wn_comm_arena_export(comm, tree.n)
        handles = [None] * world
        dist.all_gather_object(handles, h)
        wn.wn_comm_arena_import(comm, handles)
        dist.barrier()  # every rank mapped every replica before anyone stores into a peer
        mu = torch.zeros(tree.n, 3, device="cuda")
        st = wn.wnnc_iterate(tree, mu, comm=comm, stats=True, iters=ITERS, total_iters=40,
                             flags=wn.WN_FLAG_HOST_WAIT | wn.WN_FLAG_MU_ZERO, adjoint_mode=adjoint_mode)
        np.save(os.path.join(out_dir, f"mu{rank}.npy"), mu.cpu().numpy())
        np.save(os.path.join(out_dir, f"alpha{rank}.npy"), np.array([s["alpha"] for s in st]))
        bounds = wn.wn_shard_plan(tree, world)
        np.save(os.path.join(out_dir, f"bounds{rank}.npy"), np.asarray(bounds))
        dist.barrier()  # no rank unmaps its arena while a peer may still store into it
        comm.close()
        tree.close()
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    p = synth.config("C3", n=N_PTS)["points"]
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    mu = torch.zeros(t.n, 3, device="cuda")
    st = wn.wnnc_iterate(t, mu, stats=True, iters=ITERS, total_iters=40, flags=wn.WN_FLAG_MU_ZERO)
    return mu.cpu().numpy(), np.array([s["alpha"] for s in st])


@pytest.mark.parametrize("world", [2, 3])
def test_processes_exchange_over_ipc_bit_identical(single_gpu, world):
    import torch.multiprocessing as mp

    ref_mu, ref_alpha = single_gpu
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True,
                           start_method="spawn")
        bounds = [np.load(os.path.join(d, f"bounds{r}.npy")) for r in range(world)]
        for r in range(world):
            np.testing.assert_array_equal(bounds[r], bounds[0])  # every rank planned the same shards
            assert len(np.unique(bounds[0])) == world + 1  # nobody's shard is empty here
            np.testing.assert_array_equal(np.load(os.path.join(d, f"alpha{r}.npy")), ref_alpha)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"mu{r}.npy")), ref_mu)


def test_processes_transpose_adjoint():
    # the transpose-mode adjoint across 2 processes: each scatters its shard into the accumulators of its own
    # arena, signals; after both signals each adds both ranks' accumulators (IPC reads of the peer's block) in
    # rank order and pushes down — both ranks end with the same μ bit for bit, the single-GPU transpose
    # trajectory up to the scatter atomics' rounding
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    p = synth.config("C3", n=N_PTS)["points"]
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    ref = torch.zeros(t.n, 3, device="cuda")
    wn.wnnc_iterate(t, ref, iters=ITERS, total_iters=40, flags=wn.WN_FLAG_MU_ZERO, adjoint_mode=wn.WN_ADJ_TRANSPOSE)
    ref = ref.cpu().numpy()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(2, _free_port(), d, wn.WN_ADJ_TRANSPOSE), nprocs=2, join=True,
                           start_method="spawn")
        mus = [np.load(os.path.join(d, f"mu{r}.npy")) for r in range(2)]
        np.testing.assert_array_equal(mus[1], mus[0])
        np.testing.assert_array_equal(np.load(os.path.join(d, "alpha1.npy")), np.load(os.path.join(d, "alpha0.npy")))
        np.testing.assert_allclose(mus[0], ref, rtol=0, atol=1e-4 * np.abs(ref).max())
        assert np.all(np.sum(mus[0] * ref, axis=1) > 0)
