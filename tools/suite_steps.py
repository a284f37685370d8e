"""Per-step, per-query device times of the 4-query suite (debug aid for
outlier steps)."""
import json, sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import torch
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
ex = {q: tqp.Executor(json.load(open(f"paper_2209_04579_b200/plans/{q}.opplan.json")), ctx=ctx) for q in ("q1", "q6", "q14", "q3")}
for q in ex: ex[q].set_timing(True)
for _ in range(3):
    for q in ex: ex[q].execute(tables)
ctx.sync()
for q in ex: ex[q].reset_timings()
for step in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    row = []
    for q in ex:
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); ex[q].execute(tables); b.record(stream); b.synchronize()
        ms = a.elapsed_time(b)
        if ms > 3: row.append((q, round(ms, 2)))
    if row: print("step", step, row, flush=True)
for q in ex:
    print(q, {k: (v["calls"], round(v["total_ms"], 2)) for k, v in ex[q].timings().items()})
