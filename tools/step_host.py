"""Host-phase marks (TQP_HOST_PROF=1) of one asynchronous 4-query suite step
at SF10, as bench.py submits it:  TQP_HOST_PROF=1 python tools/step_host.py"""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
Q = ("q1", "q6", "q14", "q3")
ex = {q: tqp.Executor(json.loads((ROOT / f"paper_2209_04579_b200/plans/{q}.opplan.json").read_text()), ctx=ctx) for q in Q}
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
def step():
    pend = [ex[q].execute_async(tables) for q in Q]
    for p in pend: p.result()
for _ in range(5): step()
ctx.sync()
ms = []
for i in range(20):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    if i == 19: print("---- last step", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    a.record(stream); step(); b.record(stream); b.synchronize(); ms.append(a.elapsed_time(b))
    if i == 19: print("wall us", (time.perf_counter() - t0) * 1e6, file=sys.stderr)
ms.sort()
print("step median ms", ms[len(ms) // 2], file=sys.stderr)
