"""One-call sharded execution through the C ABI (tqp_executor_execute_sharded,
SURVEY.md §8(e)) with ranks that are threads of this process sharing one
B200 (tqp_comm_init_local: the same exchange code paths NCCL runs between
GPUs, which NCCL itself cannot run with two ranks on one device).

Layout as the generator shards TPC-H: lineitem and orders cut on order
boundaries (co-partitioned), part and customer cut by rows (row shards whose
build sides are exchanged as presence / flag bitmaps over the global key
range). Every rank must return the reference's SF1 result and stay on the
fused path. Also covered: an orders shard that is NOT aligned with the
lineitem shard (the group build's rows are re-aligned by an all-to-all on
l_orderkey ranges), and a plan that cannot shard (tables gathered to every
rank, reference result)."""
import json
import threading

import pytest

from conftest import GOLDEN, ROOT
from test_oracle import compare_tables

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
PLANS = ROOT / "paper_2209_04579_b200" / "plans"


def plan(q):
    return json.loads((PLANS / f"{q}.opplan.json").read_text())


def gold(sf=1):
    return json.loads((GOLDEN / f"tpch_results_sf{sf}.json").read_text())["results"]


def run_ranks(n, body):
    """body(rank, comm, ctx) on n threads; returns the per-rank results"""
    from paper_2209_04579_b200 import tqp
    comms = tqp.Comm.local_group(n)
    out, errs = [None] * n, [None] * n

    def work(r):
        try:
            ctx = tqp.Context(0)
            out[r] = body(r, comms[r], ctx)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=500)
    for e in errs:
        if e is not None:
            raise e
    return out


def tables_for(tqp, ctx, sf, rank, n, orders_shard=None):
    t = {}
    for name in ("lineitem", "orders", "part", "customer"):
        s = rank if name != "orders" or orders_shard is None else orders_shard
        t[name] = tqp.Table.generate(name, sf, 7, shard=s, nshards=n, ctx=ctx)
    return t


@pytest.mark.parametrize("n", [2, 4])
def test_sharded_queries_match_reference(n):
    from paper_2209_04579_b200 import tqp
    want = gold(1)

    def body(r, comm, ctx):
        tabs = tables_for(tqp, ctx, 1, r, n)
        res = {}
        for q in ("q1", "q6", "q14", "q3"):
            ex = tqp.Executor(plan(q), ctx=ctx)
            res[q] = (ex.execute_sharded(tabs, comm).to_numpy(), ex.fallbacks, ex.shard_stats())
        return res

    for r, res in enumerate(run_ranks(n, body)):
        for q, (got, fb, stats) in res.items():
            compare_tables(got, want[q])
            assert fb == 0, (r, q)
            assert stats["path"] == "fused", (r, q, stats)
        # the part (Q14) and customer (Q3) build sides were exchanged as bitmaps
        assert res["q14"][2]["bitmap_merges"] == 1 and res["q3"][2]["bitmap_merges"] == 1
        assert res["q1"][2]["bitmap_merges"] == 0


def test_sharded_unaligned_orders_are_realigned():
    """orders shards rotated against the lineitem shards and declared row
    shards: Q3's group build (orders) is re-aligned to each rank's l_orderkey
    range with a grouped send/recv all-to-all before the build"""
    from paper_2209_04579_b200 import tqp
    n = 3
    want = gold(1)
    kinds = dict(tqp.TPCH_SHARD_KINDS, orders=tqp.SHARD_ROWS)

    def body(r, comm, ctx):
        tabs = tables_for(tqp, ctx, 1, r, n, orders_shard=(r + 1) % n)
        ex = tqp.Executor(plan("q3"), ctx=ctx)
        return ex.execute_sharded(tabs, comm, kinds).to_numpy(), ex.fallbacks, ex.shard_stats()

    for got, fb, stats in run_ranks(n, body):
        compare_tables(got, want["q3"])
        assert fb == 0
        assert stats["path"] == "fused" and stats["shuffled_tables"] == 1, stats


def test_sharded_unshardable_plan_gathers():
    """per-instruction executors have no fused unit to shard: every rank
    gathers the shards and runs the plan whole (the reference's result)"""
    from paper_2209_04579_b200 import tqp
    n = 2
    want = gold(1)

    def body(r, comm, ctx):
        tabs = tables_for(tqp, ctx, 1, r, n)
        ex = tqp.Executor(plan("q14"), fuse=False, ctx=ctx)
        return ex.execute_sharded(tabs, comm).to_numpy(), ex.shard_stats()

    for got, stats in run_ranks(n, body):
        compare_tables(got, want["q14"])
        assert stats["path"] == "gathered", stats
