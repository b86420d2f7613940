"""Per-GPU batch sharder: split arithmetic and the multi-process (world_size 2,
gloo on CPU) shard -> compute -> gather path. The per-shard compute stand-in
is the CPU oracle (tests may use it as the checker); on GPUs each rank runs
the same code with the CUDA kernels and NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2108_13656_b200 import sharder


@pytest.mark.parametrize("n,world", [(0, 1), (1, 1), (7, 2), (8, 8), (256, 3), (1024, 8), (5, 8)])
def test_shard_range_partitions(n, world):
    spans = [sharder.shard_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == n
    assert sizes == sharder.shard_sizes(n, world)


def test_shard_range_rejects():
    with pytest.raises(ValueError):
        sharder.shard_range(4, 0, 0)
    with pytest.raises(ValueError):
        sharder.shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        sharder.shard_range(-1, 2, 0)


def test_run_on_devices_order_and_invariance():
    from oracle import oracle

    batch = oracle.synth_uniform_u8(7, 5, 6, seed=4)
    whole = oracle.decolor_u8(batch)
    for ndev in (1, 2, 3, 8):
        got = sharder.run_on_devices(lambda shard, dev: oracle.decolor_u8(shard), batch, list(range(ndev)))
        assert np.array_equal(got, whole)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_images, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = sharder.shard_range(n_images, world, rank)
        # every rank regenerates only its own images (first_image = a), as the bench does
        rgb = oracle.synth_uniform_u8(b - a, 6, 10, seed=9, first_image=a)
        local = torch.from_numpy(oracle.decolor_u8(rgb))
        full = sharder.gather_to_root(local, n_images)
        if rank == 0:
            q.put(full.numpy())
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_images", [5, 8])
def test_gloo_world2_shard_and_gather(n_images):
    from oracle import oracle

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_images, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = q.get()
    want = oracle.decolor_u8(oracle.synth_uniform_u8(n_images, 6, 10, seed=9))
    assert np.array_equal(got, want)
