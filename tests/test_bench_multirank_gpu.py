"""bench.py's N-rank flow (torchrun, sharded generation, execute_sharded
exchange, max-over-ranks timing, one JSON line from rank 0) run with two
ranks sharing cuda:0 over gloo (TQP_BENCH_SHARE_GPU=1) - a functional check
on a one-GPU box, not a measurement."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, TQP_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--sf", "0.2", "--no-cpu-baseline", "--no-csv", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["lineitem_rows_per_gpu"] * 2 >= 2_390_000
