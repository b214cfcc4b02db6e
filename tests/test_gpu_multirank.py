"""The N > 1 paths on a real device: tests/gpu_dist_check.py (broadcast structure, per-rank
shards, concatenation == single rank) and bench.py's torchrun leg, both with two ranks.  A
one-GPU box runs both ranks on cuda:0 over gloo; with one GPU per rank the same code runs over
NCCL.  These check correctness and that the launch contract holds, not multi-GPU speed."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, env_extra, timeout):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_sharded_search_equals_single_rank():
    r = _torchrun([os.path.join(ROOT, "tests", "gpu_dist_check.py")], {}, 600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "DIST_CHECK PASS" in r.stdout


@pytest.mark.parametrize("replicate", ["0", "1"])  # structure broadcast from rank 0 / built on every rank
def test_bench_two_ranks_contract(replicate):
    r = _torchrun(["bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
                   "--config", "cfg0"],
                  {"LO_BENCH_SAME_DEVICE": "1", "LO_BENCH_DIST_BACKEND": "gloo",
                   "LO_BENCH_REPLICATE": replicate}, 900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
