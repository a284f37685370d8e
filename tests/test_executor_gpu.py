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


def test_q14_scalar_epilogue(ctx):
    """Q14's final projection (100.00 * promo / total) runs inside the fused
    unit's finalize kernel; with no qualifying row the exact path reports the
    reference's division-by-zero error, fused or not, and the sharded merge
    raises the same text."""
    from paper_2209_04579_b200 import tqp
    plan = json.loads((PLANS / "q14.opplan.json").read_text())
    gold = load_tpch_golden()
    tables = {n: tqp.Table.generate(n, gold["sf"], gold["seed"]) for n in ("lineitem", "part")}
    fused = tqp.Executor(plan, fuse=True)
    fused.set_timing(True)
    got = as_numpy(fused.execute(tables))
    assert not [k for k in fused.timings() if k.startswith("step:")], fused.timings()
    compare_tables(got, gold["results"]["q14"])
    exact = as_numpy(tqp.Executor(plan, fuse=False).execute(tables))
    np.testing.assert_allclose(got[0][2], exact[0][2], rtol=1e-12)
    # every price 0.0: both sums are 0.0 -> 100.00 * 0.0 / 0.0
    host = tables["lineitem"].to_numpy()
    cols = []
    for name, lt in tables["lineitem"].columns():
        a = host[name]
        if name == "l_extendedprice":
            a = np.zeros_like(a)
        cols.append((name, lt, a))
    empty = {"lineitem": tqp.Table.from_columns(cols), "part": tables["part"]}
    msgs = []
    for fuse in (True, False):
        with pytest.raises(tqp.ExecError) as ei:
            tqp.Executor(plan, fuse=fuse).execute(empty)
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1] and msgs[0].endswith("arith: division by zero at row 0"), msgs
    ex = tqp.Executor(plan, fuse=True)
    with pytest.raises(tqp.ExecError) as ei:
        ex.finish([ex.execute_partial(empty)])
    assert str(ei.value) == msgs[0]


def test_one_executor_over_several_table_sets(ctx):
    """An executor reused across table sets (its per-unit kernel memo keyed by
    the generator arguments) gives each table set the result a fresh executor
    gives it, in either order and repeatedly."""
    from paper_2209_04579_b200 import tqp
    import os
    old = os.environ.get("TQP_JIT")
    os.environ["TQP_JIT"] = "1"  # the NVRTC kernels (and their memo) at test sizes
    try:
        sets = [{n: tqp.Table.generate(n, sf, seed) for n in ("lineitem", "orders", "customer", "part")}
                for sf, seed in ((0.02, 7), (0.02, 8), (0.03, 7))]
        for q in ("q1", "q6", "q14", "q3"):
            plan = json.loads((PLANS / f"{q}.opplan.json").read_text())
            fresh = [as_numpy(tqp.Executor(plan).execute(t)) for t in sets]
            ex = tqp.Executor(plan)
            for i in (0, 1, 2, 1, 0, 0, 2):
                got = as_numpy(ex.execute(sets[i]))
                for (n, _, g), (_, _, w) in zip(got, fresh[i]):
                    np.testing.assert_array_equal(g, w, err_msg=f"{q} set {i} {n}")
            assert ex.fallbacks == 0
    finally:
        if old is None:
            del os.environ["TQP_JIT"]
        else:
            os.environ["TQP_JIT"] = old


def _with_column(tqp, table, name, fn):
    host = table.to_numpy()
    return tqp.Table.from_columns([(c, lt, fn(host[c]) if c == name else host[c]) for c, lt in table.columns()])


@pytest.mark.parametrize("scale", [1e-25, 1e15])
def test_buildgroup_fixed_point_guards(ctx, scale):
    """Q3's build-group sums are exact Q64.64 fixed point. A value with bits
    below 2^-64 (scale 1e-25) or a column whose max|v| x rows may reach 2^62
    (scale 1e15) must not be summed there: the unit hands its steps to the
    exact path (one fallback) and the result is the per-instruction one."""
    from paper_2209_04579_b200 import tqp
    plan = json.loads((PLANS / "q3.opplan.json").read_text())
    base = {n: tqp.Table.generate(n, 0.005, 7) for n in ("lineitem", "orders", "customer")}
    tables = dict(base, lineitem=_with_column(tqp, base["lineitem"], "l_extendedprice", lambda a: a * scale))
    fused = tqp.Executor(plan, fuse=True)
    got = as_numpy(fused.execute(tables))
    assert fused.fallbacks == 1
    want = as_numpy(tqp.Executor(plan, fuse=False).execute(tables))
    for (n, _, g), (_, _, w) in zip(got, want):
        np.testing.assert_array_equal(g, w, err_msg=n)
    # the unscaled tables stay on the fused path
    ok = tqp.Executor(plan, fuse=True)
    ok.execute(base)
    assert ok.fallbacks == 0


def test_typed_scalar_access_checks_dtype(ctx):
    """last_or_zero / iota_len / segmented_reduce's count read a 1x1 int64
    (Tensor::data<int64_t>, tensor.cpp:35-39): other dtypes raise the
    reference's KernelError instead of reading 8 bytes of something else."""
    from paper_2209_04579_b200 import tqp
    for arr, dt, name in ((np.array([[1.5]]), tqp.F64, "float64"), (np.array([[1]], np.int32), tqp.I32, "int32"),
                          (np.array([[1]], np.uint8), tqp.BOOL, "bool")):
        t = tqp.Tensor.from_numpy(arr, dt)
        with pytest.raises(tqp.KernelError, match=f"tensor: dtype is {name}, accessed as int64"):
            tqp.last_or_zero(t)
    np.testing.assert_array_equal(tqp.last_or_zero(tqp.Tensor.from_numpy(np.array([[3], [9]], np.int64))).numpy(),
                                  [[9]])


def test_execute_async_matches_execute(ctx):
    """execute_async + result() (queries submitted back to back, results
    taken afterwards) gives the golden results; a fused unit whose deferred
    check flags its data (Q64.64 range, see the fixed-point guards test)
    re-runs on the checked path inside result() and returns the exact
    path's result."""
    import json
    from conftest import load_tpch_golden
    from test_oracle import compare_tables
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    tables = {n: tqp.Table.generate(n, gold["sf"], gold["seed"], ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
    execs = {q: tqp.Executor(json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text()), ctx=ctx)
             for q in ("q1", "q6", "q14", "q3")}
    for _ in range(3):
        pend = {q: ex.execute_async(tables) for q, ex in execs.items()}
        for q, p in pend.items():
            compare_tables(p.result().to_numpy(), gold["results"][q])
    p = execs["q6"].execute_async(tables)
    del p  # freed without a result
    ctx.sync()
    plan = json.loads((PLANS / "q3.opplan.json").read_text())
    base = {n: tqp.Table.generate(n, 0.005, 7) for n in ("lineitem", "orders", "customer")}
    scaled = dict(base, lineitem=_with_column(tqp, base["lineitem"], "l_extendedprice", lambda a: a * 1e15))
    fused = tqp.Executor(plan, fuse=True)
    got = as_numpy(fused.execute_async(scaled).result())
    assert fused.fallbacks == 1
    want = as_numpy(tqp.Executor(plan, fuse=False).execute(scaled))
    for (n, _, g), (_, _, w) in zip(got, want):
        np.testing.assert_array_equal(g, w, err_msg=n)
