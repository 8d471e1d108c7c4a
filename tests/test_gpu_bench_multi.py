"""bench.py's N > 1 path as the driver launches it (torch.distributed.run,
two ranks) on a one-GPU box: NRC_BENCH_SHARED_GPU=1 puts both ranks on
cuda:0 with gloo (a code-path test: the timings mean nothing).  Every
training partition runs, the replicas stay bitwise identical, and rank 0
prints one contract JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["dp", "replicated", "allreduce-peer", "allreduce-sym"])
def test_bench_two_ranks_shared_gpu(mode):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    env = dict(os.environ, NRC_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--train-mode", mode]
    if mode != "dp":
        cmd.append("--no-mode-table")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["config"]["parallelism"] == f"{mode}2"
    assert line["replicas"].startswith("identical")
    assert line["gpu_launches"] > 0 and line["value"] > 0
    if mode == "dp":  # the N3 comparison: every partition trained the frame (NVLS where multicast exists)
        tm = line["train_modes"]
        assert set(tm) == {"dp", "replicated", "allreduce-peer", "allreduce-sym", "allreduce-nvls"}
        for m in ("dp", "replicated", "allreduce-peer"):
            assert tm[m]["train_ms"] > 0 and tm[m]["replicas"].startswith("identical"), tm
