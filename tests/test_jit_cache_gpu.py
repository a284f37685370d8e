"""The NVRTC kernel cache is bounded (jit.cu: least-recently-used libraries
unloaded at TQP_JIT_CACHE). With room for two libraries, running the four
TPC-H queries twice (every fused unit on NVRTC kernels, TQP_JIT=1) unloads and
recompiles kernels between executions; every result must still match the
reference (the per-unit memo and the attribute caches notice the unload)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests"); sys.path.insert(0, {root!r} + "/oracle")
from paper_2209_04579_b200 import tqp
from conftest import load_tpch_golden
from test_oracle import compare_tables
gold = load_tpch_golden()
ctx = tqp.Context(0)
tables = {{n: tqp.Table.generate(n, gold["sf"], gold["seed"], ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}}
execs = {{q: tqp.Executor(json.loads(open({root!r} + "/paper_2209_04579_b200/plans/" + q + ".opplan.json").read()), ctx=ctx)
         for q in ("q1", "q6", "q14", "q3")}}
for rnd in range(2):
    for q, ex in execs.items():
        compare_tables(ex.execute(tables).to_numpy(), gold["results"][q])
        assert ex.fallbacks == 0, q
print("ok")
"""


def test_jit_cache_bound_evicts_and_recompiles():
    env = dict(os.environ, TQP_JIT_CACHE="2", TQP_JIT="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
