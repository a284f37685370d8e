"""Runs Q3 repeatedly at SF10 and reports executions that left the fused
path (debug aid for the fused unit's precondition flags)."""
import json, sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
ex = tqp.Executor(json.load(open("paper_2209_04579_b200/plans/q3.opplan.json")), ctx=ctx)
ex.set_timing(True)
slow = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    t0 = time.perf_counter(); ex.execute(tables); ctx.sync(); ms = (time.perf_counter() - t0) * 1e3
    if ms > 5: slow.append((i, round(ms, 1)))
t = ex.timings()
print("slow executions:", slow, "fused calls:", t.get("fused_probe_build-group_topk", {}).get("calls"))
