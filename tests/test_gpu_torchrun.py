"""bench.py under torchrun with 2 ranks on one GPU (TT_BENCH_ONE_GPU=1: gloo group,
every rank on cuda:0): the sharded multi-rank path end to end — each rank creates its
UE block's handle, times its slots, the max/sum reductions run, rank 0 prints one JSON
line for n_gpus = 2. (The throughput of two processes sharing one GPU is not a
scaling number; only the plumbing is checked.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_bench_on_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, TT_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "c3", "--steps", "5",
           "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "ue-shard x2"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 5
