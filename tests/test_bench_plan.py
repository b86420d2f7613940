"""bench.py's sharding plan on CPU: strong scaling shards the fixed C5 batch
(BASELINE configs[4], 1024 images) over the ranks of a torchrun job, weak
scaling gives every rank a full batch (run over gloo, world_size 1 and 2)."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan(nproc, *extra):
    if nproc == 1:
        cmd = [sys.executable, "bench.py", "--plan", *extra]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus",
               str(nproc), "--plan", *extra]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="1")
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    return lines[0]


@pytest.mark.parametrize("nproc", [1, 2])
def test_c5_strong_scaling_plan(nproc):
    p = _plan(nproc, "--workload", "C5")
    assert p["scaling"] == "strong" and p["n_gpus"] == nproc
    assert p["config"]["images_total"] == 1024
    assert "1024 x 7680x4320" in p["config"]["workload"]
    shards = p["config"]["shards"]
    assert shards[0][0] == 0 and shards[-1][1] == 1024
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))  # contiguous, in rank order


def test_weak_scaling_plan_world2():
    p = _plan(2, "--workload", "C3")
    assert p["scaling"] == "weak"
    assert p["config"]["shards"] == [[0, 256], [256, 512]]
    p = _plan(2, "--workload", "C5", "--scaling", "weak", "--images", "8")
    assert p["config"]["shards"] == [[0, 8], [8, 16]]
