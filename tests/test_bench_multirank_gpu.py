"""bench.py's multi-rank path end to end (-m gpu): two ranks under torchrun share the one GPU of the test box,
gloo carries the all-reduce of dL/dp0 (PA_BENCH_BACKEND=gloo; a functional check of the code the driver's
N = 2/4/8 NCCL runs take — frame sharding, the all-reduce callback inside pa_step, barriers, max-over-ranks
timing, rank 0's JSON line — not a measurement).  Also a rank that owns no frame (F = 0 on that rank)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("frames", [4, 1])
def test_two_ranks_bench_line(frames):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, PA_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
           "c2", "--frames", str(frames), "--steps", "1", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["frames_per_rank"] in (frames // 2, (frames + 1) // 2)
    assert "gloo" in d["config"]["parallelism"]
