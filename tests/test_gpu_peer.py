"""The optional final gather fused into the launch (SURVEY.md 8 e): the root's
output buffer mapped into every rank over CUDA IPC (sharder.PeerBuffer), each
rank's decolor / tone kernels storing their shard straight into it.

On the single-GPU test box the two ranks are two processes on the same device
(the IPC mapping and the remote stores are the same code path as across
NVLink peers; no kernel waits on another rank). The root's assembled batch must
equal one single-process launch over the whole batch, byte for byte.
"""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, h, w, result_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import sharder, synth

    dev = torch.device("cuda", 0)
    first, last = sharder.shard_range(n_total, world, rank)
    rgb = torch.empty((last - first, h, w, 3), dtype=torch.uint8, device=dev)
    synth.fill_uniform_u8(rgb, seed=3, first_image=first)
    gray = sharder.PeerBuffer(n_total, (h, w), 0)
    toned = sharder.PeerBuffer(n_total, (h, w), 0)
    wg.decolor(rgb, out=gray.view(first, last - first))  # a tensor view (same device here)
    from paper_2108_13656_b200 import _lib  # and the raw address through the C ABI (any device)

    _lib.call("wg_decolor_tone_u8", rgb.data_ptr(), toned.ptr_at(first), None, rgb.numel() // 3, 0.55, 0.8, 0.5, 8.0,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        full = torch.empty((n_total, h, w, 3), dtype=torch.uint8, device=dev)
        synth.fill_uniform_u8(full, seed=3, first_image=0)
        ok = torch.equal(gray.full(), wg.decolor(full)) and torch.equal(toned.full(), wg.decolor_tone(full))
        with open(os.path.join(result_dir, "result.txt"), "w") as f:
            f.write("ok" if ok else "mismatch")
    gray.close()
    toned.close()
    dist.destroy_process_group()


def test_decolor_into_root_buffer(tmp_path):
    import torch.multiprocessing as mp

    # 5 images over 2 ranks (3 + 2, unequal shards), 4K-wide rows
    mp.spawn(_worker, args=(2, _free_port(), 5, 270, 3840, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "result.txt").read_text() == "ok"


def _bench_gather_worker(rank, world, port, result_dir):
    import sys

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_2108_13656_b200 as wg
    from paper_2108_13656_b200 import _lib, sharder, synth

    dev = torch.device("cuda", 0)
    n_total, h, w = 3, 180, 320
    first, last = sharder.shard_range(n_total, world, rank)
    rgb = torch.empty((last - first, h, w, 3), dtype=torch.uint8, device=dev)
    synth.fill_uniform_u8(rgb, seed=9, first_image=first)
    out = wg.decolor(rgb)
    stream = torch.cuda.current_stream(dev)

    def step_into(ptr, _n=rgb.numel() // 3):
        _lib.call("wg_decolor_u8", rgb.data_ptr(), ptr, _n, 0.55, 0.8, stream.cuda_stream)

    res = bench.run_gather(torch, sharder, out, n_total, world, step_into, first, stream)
    if rank == 0:
        with open(os.path.join(result_dir, "gather.txt"), "w") as f:
            f.write(repr(res))
    dist.destroy_process_group()


def test_bench_gather_paths_two_ranks(tmp_path):
    """bench.run_gather (strong scaling, N > 1): the sharder's gather and the
    fused peer-buffer launch, with two ranks on one device over gloo -- the
    fused launch reproduces the root's own shard."""
    import torch.multiprocessing as mp

    mp.spawn(_bench_gather_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    res = eval((tmp_path / "gather.txt").read_text())
    assert res["gather_ms"] >= 0 and res["fused"]["root_shard_equal"] is True, res
