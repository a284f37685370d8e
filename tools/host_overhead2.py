import json, sys, time
from pathlib import Path
sys.path.insert(0, "/root/repo")
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
for q in ("q6", "q1"):
    ex = tqp.Executor(json.loads(Path(f"/root/repo/paper_2209_04579_b200/plans/{q}.opplan.json").read_text()), ctx=ctx)
    for _ in range(5): ex.execute(tables)
    ctx.sync()
    n = 100
    t0 = time.perf_counter()
    for _ in range(n): r = ex.execute(tables)
    wall = (time.perf_counter() - t0) / n * 1e6
    cn, th, k = ex._args(tables)
    st = tqp.Status()
    t0 = time.perf_counter()
    for _ in range(n):
        h = tqp.lib.tqp_executor_execute(ex.h, cn, th, k, tqp.C.byref(st)); tqp.lib.tqp_result_free(h)
    craw = (time.perf_counter() - t0) / n * 1e6
    print(f"{q}: python execute {wall:.1f} us, raw C call {craw:.1f} us")
