"""Sharded execution simulated on one GPU: N shards of
lineitem (order-aligned) each run phase 1, the partials merge in shard order,
and the result must equal the unsharded run: bit-exact for integers, keys,
counts and build-grouped (Q64.64) sums; fp64 scan sums within 1e-9."""
import json

import numpy as np
import pytest

import tqp_oracle as O
from conftest import ROOT, load_tpch_golden
from test_oracle import compare_tables

pytestmark = pytest.mark.gpu
PLANS = ROOT / "paper_2209_04579_b200" / "plans"
SF = 0.05


def plan(q):
    return json.loads((PLANS / f"{q}.opplan.json").read_text())


def tables(tqp, shard, nshards, orders_whole=False):
    t = {}
    for name in ("lineitem", "orders", "customer", "part"):
        sharded = name == "lineitem" or (name == "orders" and not orders_whole)
        t[name] = tqp.Table.generate(name, SF, 7, shard=shard if sharded else 0, nshards=nshards if sharded else 1)
    return t


def assert_same(got, want, exact):
    assert [(n, t) for n, t, _ in got] == [(n, t) for n, t, _ in want]
    for (n, _, g), (_, _, w) in zip(got, want):
        assert g.shape == w.shape, n
        if g.dtype == np.float64 and not exact:
            np.testing.assert_allclose(g, w, rtol=1e-9, atol=0, err_msg=n)
        else:
            np.testing.assert_array_equal(g, w, err_msg=n)


@pytest.mark.parametrize("nshards", [1, 2, 3, 8])
@pytest.mark.parametrize("q", ["q1", "q6", "q14", "q3"])
def test_sharded_equals_unsharded(ctx, q, nshards):
    from paper_2209_04579_b200 import tqp
    ex = tqp.Executor(plan(q))
    ok, why = ex.shardable()
    assert ok, why
    want = ex.execute(tables(tqp, 0, 1)).to_numpy()
    parts = [ex.execute_partial(tables(tqp, s, nshards)) for s in range(nshards)]
    got = ex.finish(parts).to_numpy()
    assert_same(got, want, exact=q == "q3")


def test_q3_groups_split_across_shards(ctx):
    """orders whole on every shard, lineitem cut at arbitrary rows: an order's
    lines land on several shards and the merge must add them exactly."""
    from paper_2209_04579_b200 import tqp
    ex = tqp.Executor(plan("q3"))
    full = tables(tqp, 0, 1)
    want = ex.execute(full).to_numpy()
    li = full["lineitem"].to_numpy()
    n = full["lineitem"].rows
    cuts = [0, n // 3 + 1, n // 2 + 2, n]  # not order-aligned
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        cols = [(c, t, li[c][a:b]) for c, t in full["lineitem"].columns()]
        shard = dict(full)
        shard["lineitem"] = tqp.Table.from_columns(cols)
        parts.append(ex.execute_partial(shard))
    assert_same(ex.finish(parts).to_numpy(), want, exact=True)


def test_sharded_matches_reference_golden(ctx):
    """The merged result of 4 shards of the SF0.005 golden tables equals the
    reference executor's own result."""
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    host = O.tables_from_json(gold["tables"])
    n = len(host["lineitem"]["l_orderkey"][1])
    keys = host["lineitem"]["l_orderkey"][1][:, 0]
    # order-aligned cuts near n/4, n/2, 3n/4
    cuts = [0]
    for f in (0.25, 0.5, 0.75):
        i = int(n * f)
        while 0 < i < n and keys[i] == keys[i - 1]:
            i += 1
        cuts.append(i)
    cuts.append(n)
    dev = {name: tqp.Table.from_columns([(c, typ, arr) for c, (typ, arr) in t.items()]) for name, t in host.items()}
    for q in ("q1", "q6", "q14", "q3"):
        ex = tqp.Executor(plan(q))
        parts = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            shard = dict(dev)
            shard["lineitem"] = tqp.Table.from_columns(
                [(c, typ, arr[a:b]) for c, (typ, arr) in host["lineitem"].items()])
            parts.append(ex.execute_partial(shard))
        got = [(nm, t, a) for nm, t, a in ex.finish(parts).to_numpy()]
        compare_tables(got, gold["results"][q])


def test_partials_travel_as_torch_words(ctx):
    """Partials copied into torch CUDA tensors (what the NCCL all-gather hands
    back) merge like the library's own tensors."""
    import torch
    from paper_2209_04579_b200 import tqp
    ex = tqp.Executor(plan("q1"))
    want = ex.execute(tables(tqp, 0, 1)).to_numpy()
    parts = [torch.as_tensor(ex.execute_partial(tables(tqp, s, 2)), device="cuda").reshape(-1).clone()
             for s in range(2)]
    torch.cuda.synchronize()
    assert_same(ex.finish(parts).to_numpy(), want, exact=False)


def test_partial_errors(ctx):
    from paper_2209_04579_b200 import tqp
    t = tables(tqp, 0, 1)
    nofuse = tqp.Executor(plan("q6"), fuse=False)
    ok, why = nofuse.shardable()
    assert not ok and "fused" in why
    with pytest.raises(tqp.ExecError, match="not shardable"):
        nofuse.execute_partial(t)
    q6, q1 = tqp.Executor(plan("q6")), tqp.Executor(plan("q1"))
    p6 = q6.execute_partial(t)
    with pytest.raises(tqp.TqpError, match="not produced by this plan"):
        q1.finish([p6])
    with pytest.raises(tqp.TqpError, match="at least one partial"):
        q1.finish([])
