"""Host-phase marks (TQP_HOST_PROF=1) and event latency of one query at SF10:
    TQP_HOST_PROF=1 python tools/q3_host.py q3"""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2209_04579_b200 import tqp
q = sys.argv[1] if len(sys.argv) > 1 else "q3"
ctx = tqp.Context(0)
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
ex = tqp.Executor(json.loads((ROOT / f"paper_2209_04579_b200/plans/{q}.opplan.json").read_text()), ctx=ctx)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
for _ in range(5): ex.execute(tables)
ctx.sync()
ms = []
for _ in range(20):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(stream); ex.execute(tables); b.record(stream); b.synchronize(); ms.append(a.elapsed_time(b))
ms.sort()
print(q, "latency median ms", ms[len(ms) // 2], file=sys.stderr)
