"""Median device latency per query (CUDA events on the library's stream
around each execute, results left on the device), SF10 by default.

    python tools/query_time.py [--sf 10] [--queries q3] [--iters 30]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2209_04579_b200 import tqp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--queries", default="q1,q6,q14,q3")
ap.add_argument("--iters", type=int, default=30)
a = ap.parse_args()
ctx = tqp.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
tables = {n: tqp.Table.generate(n, a.sf, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
for q in a.queries.split(","):
    ex = tqp.Executor(json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text()), ctx=ctx)
    for _ in range(3):
        ex.execute(tables)
    ctx.sync()
    ms = []
    for _ in range(a.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ex.execute(tables)
        e.record(stream)
        e.synchronize()
        ms.append(s.elapsed_time(e))
    print(f"{q} median {statistics.median(ms):.4f} ms  min {min(ms):.4f}  fallbacks {ex.fallbacks}", flush=True)
