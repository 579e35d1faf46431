"""bench.py under torchrun with 2 ranks (the driver's scaling run), on a one-GPU box: ranks share the GPU
(KS_BENCH_SHARE_GPU=1, gloo plumbing; independent problems, so no rank's kernels wait on another's). Checks
the launch path end to end: exactly one JSON line (rank 0) with n_gpus = 2, weak scaling and positive
whole-job throughput; the reference arm prints one line from rank 0 and the other rank exits 0 silently."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(extra):
    env = dict(os.environ, KS_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--config", "1", "--steps", "2", "--warmup", "3"] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return lines


def test_bench_two_ranks():
    lines = _run(["--no-cpu-baseline", "--no-e2e"])
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["steps"] == 2


def test_reference_arm_two_ranks():
    lines = _run(["--impl", "reference", "--ref-budget-s", "5"])
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
