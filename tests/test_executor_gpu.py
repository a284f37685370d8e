"""Executor parity: lowered reference OperatorPlans run on the B200 executor
(fused and per-instruction) against the reference executor's own results."""
import json

import numpy as np
import pytest

import tqp_oracle as O
from conftest import ROOT, load_tpch_golden
from test_oracle import compare_tables

pytestmark = pytest.mark.gpu
PLANS = ROOT / "paper_2209_04579_b200" / "plans"


def device_tables(tqp, tables_json):
    out = {}
    for name, t in O.tables_from_json(tables_json).items():
        out[name] = tqp.Table.from_columns([(c, typ, arr) for c, (typ, arr) in t.items()])
    return out


def as_numpy(result):
    return [(n, t, a) for n, t, a in result.to_numpy()]


@pytest.mark.parametrize("fuse", [False, True])
def test_golden_plans(ctx, golden_plans, fuse):
    from paper_2209_04579_b200 import tqp
    for case in golden_plans:
        tables = device_tables(tqp, case["tables"])
        ex = tqp.Executor(case["opplan"], fuse=fuse)
        if "error" in case:
            with pytest.raises(tqp.ExecError) as ei:
                ex.execute(tables)
            assert str(ei.value) == case["error"], case["name"]
            continue
        got = as_numpy(ex.execute(tables))
        compare_tables(got, case["result"])


@pytest.mark.parametrize("fuse", [False, True])
def test_tpch_sf0005_matches_reference(ctx, fuse):
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    tables = device_tables(tqp, gold["tables"])
    for q in ("q1", "q3", "q6", "q14"):
        ex = tqp.Executor(json.loads((PLANS / f"{q}.opplan.json").read_text()), fuse=fuse)
        compare_tables(as_numpy(ex.execute(tables)), gold["results"][q])


def test_device_generator_is_bit_identical_to_host(ctx):
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    for name, t in O.tables_from_json(gold["tables"]).items():
        dev = tqp.Table.generate(name, gold["sf"], gold["seed"]).to_numpy()
        for c, (typ, arr) in t.items():
            np.testing.assert_array_equal(dev[c], arr, err_msg=f"{name}.{c}")


def test_generator_shards_partition_the_table(ctx):
    from paper_2209_04579_b200 import tqp
    full = tqp.Table.generate("lineitem", 0.01).to_numpy()
    parts = [tqp.Table.generate("lineitem", 0.01, shard=s, nshards=3).to_numpy() for s in range(3)]
    for c in full:
        np.testing.assert_array_equal(np.concatenate([p[c] for p in parts]), full[c])
    # order-aligned: no orderkey spans two shards
    last = [p["l_orderkey"][-1, 0] for p in parts[:-1]]
    first = [p["l_orderkey"][0, 0] for p in parts[1:]]
    assert all(a < b for a, b in zip(last, first))


def test_input_binding_errors(ctx):
    from paper_2209_04579_b200 import tqp
    ex = tqp.Executor(json.loads((PLANS / "q6.opplan.json").read_text()))
    with pytest.raises(tqp.ExecError, match="no input table"):
        ex.execute({})
    bad = tqp.Table.from_columns([("l_orderkey", "float64", np.zeros(1))])
    with pytest.raises(tqp.ExecError, match="the plan expects"):
        ex.execute({"lineitem": bad})


def test_profile_trace(ctx):
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    tables = device_tables(tqp, gold["tables"])
    ex = tqp.Executor(json.loads((PLANS / "q6.opplan.json").read_text()), fuse=False)
    res, trace = ex.profile_execute(tables)
    ops = [e for e in trace if e["cat"] == "operator"]
    assert [e["name"] for e in ops] == ["scan#0", "filter#0", "aggregate#0", "project#0"]
    assert all(e["ph"] == "X" for e in trace)
