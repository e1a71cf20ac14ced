"""bench.py's multi-rank entry point on the one GPU this run has: `--gpus 2
--share-gpu` relaunches itself under torch.distributed.run (two ranks on
GPU 0, gloo group) and runs the row-sharded C5 leg -- S local, S' through
the p2p peer-store exchange -- printing one JSON line with n_gpus 2."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_shared_gpu(cuda):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--share-gpu",
           "--steps", "3", "--warmup", "3", "--no-cpu", "--configs", "c5", "--c5-n", "8192"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    c5 = line["configs"]["c5"]
    assert c5["rows_per_rank"] == 4096 and c5["transport"] == "p2p"
    assert c5["sjlt"]["S_ms"] > 0 and c5["sjlt"]["St_ms"] > 0
