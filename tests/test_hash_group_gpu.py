"""Fused hash-group parity: queries/qg.sql - GROUP BY
l_partkey with a date filter, SUM(l_extendedprice * (1 - l_discount)),
SUM(l_quantity), COUNT(*) - lowered by the reference (plans/qg.opplan.json)
and run by the fused MODE_HASH unit (direct-address group table over the
l_partkey range, exact Q64.64 limb sums, output in ascending key order as the
reference's sort-based lowering, operator_plan.cpp:309-388).

* against the reference executor's own results (tests/golden/qg_results_sf*,
  oracle/make_golden.sh) at SF0.05 and SF1: keys, counts and int64 sums exact,
  fp64 sums within 1e-9 relative;
* at SF10 (2 M groups) against the device per-instruction path (the
  reference's sort-based lowering executed as written), exactly the same;
* the unit stays fused (no exact-path fallback) and is a hash-group unit.
Wider shapes (dictionary keys, 1:N and non-dense joins, NaN, ties) are
covered by the random group plans (test_random_plans_gpu.py)."""
import gzip
import json

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from test_oracle import compare_tables

pytestmark = pytest.mark.gpu
PLAN = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / "qg.opplan.json").read_text())


def golden(sf):
    with gzip.open(GOLDEN / f"qg_results_sf{sf}.json.gz", "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("sf", ["0.05", "1"])
def test_qg_matches_reference(ctx, sf):
    from paper_2209_04579_b200 import tqp
    gold = golden(sf)
    li = tqp.Table.generate("lineitem", float(sf), 7)
    assert li.rows == gold["lineitem_rows"]
    ex = tqp.Executor(PLAN)
    got = ex.execute({"lineitem": li}).to_numpy()
    compare_tables(got, gold["results"]["qg"])
    assert ex.fallbacks == 0
    assert "hash-group" in json.dumps(ex.explain())


def test_qg_sf10_fused_equals_per_instruction(ctx):
    from paper_2209_04579_b200 import tqp
    li = {"lineitem": tqp.Table.generate("lineitem", 10.0, 7)}
    fused = tqp.Executor(PLAN)
    a = fused.execute(li).to_numpy()
    b = tqp.Executor(PLAN, fuse=False).execute(li).to_numpy()
    assert fused.fallbacks == 0
    assert a[0][2].shape[0] > 1_900_000  # ~2 M l_partkey groups
    for (na, ta, xa), (nb, tb, xb) in zip(a, b):
        assert (na, ta) == (nb, tb)
        if xa.dtype.kind == "f":
            np.testing.assert_allclose(xa, xb, rtol=1e-9, atol=0)
        else:
            assert np.array_equal(xa, xb), na
    # the fused unit is deterministic run to run (order-independent exact sums)
    c = fused.execute(li).to_numpy()
    for (na, _, xa), (_, _, xc) in zip(a, c):
        assert np.array_equal(xa.view(np.uint8), xc.view(np.uint8)), na


def test_qg_hash_instances_agree(ctx, monkeypatch):
    """The three kernels a lean hash-group unit can run - the NVRTC pipeline
    (q_tile<hash-lean>), the lean template instance (TQP_JIT=0) and the
    general k_tile<MODE_HASH> (TQP_HASH_NOLEAN) - produce the same bits."""
    from paper_2209_04579_b200 import tqp
    li = {"lineitem": tqp.Table.generate("lineitem", 1.0, 7)}
    runs = {}
    for name, env in (("jit", {}), ("lean", {"TQP_JIT": "0"}), ("general", {"TQP_JIT": "0", "TQP_HASH_NOLEAN": "1"})):
        for k in ("TQP_JIT", "TQP_HASH_NOLEAN"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ex = tqp.Executor(PLAN)
        ex.set_timing(True)
        runs[name] = ex.execute(li).to_numpy()
        kernels = [k for k in ex.timings() if k.startswith("kernel:")]
        want = {"jit": "q_tile<hash-lean", "lean": "k_tile<hash-lean", "general": "k_tile<hash-direct"}[name]
        assert any(want in k for k in kernels), (name, kernels)
        assert ex.fallbacks == 0
    for name in ("lean", "general"):
        for (na, ta, xa), (nb, tb, xb) in zip(runs["jit"], runs[name]):
            assert (na, ta) == (nb, tb)
            assert np.array_equal(xa.view(np.uint8), xb.view(np.uint8)), (name, na)
