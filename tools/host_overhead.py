"""Per-query host overhead: wall time of Executor.execute vs the device time
of its kernels (CUDA events recorded by the library), SF10 device tables."""
import json, os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2209_04579_b200 import tqp

ctx = tqp.Context(0)
sf = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
tables = {n: tqp.Table.generate(n, sf, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
for q in ("q6", "q1", "q14", "q3"):
    ex = tqp.Executor(json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text()), ctx=ctx)
    for _ in range(5):
        ex.execute(tables)
    ctx.sync()
    ex.set_timing(os.environ.get("TQP_HO_TIMING", "1") == "1")
    ex.reset_timings()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        ex.execute(tables)
    ctx.sync()
    wall = (time.perf_counter() - t0) / n * 1e3
    tm = ex.timings()
    kern = sum(v["total_ms"] for k, v in tm.items() if k.startswith("kernel:")) / n
    print(f"{q}: wall {wall:.3f} ms/exec, timed kernels {kern:.3f} ms, units {json.dumps({k: round(v['total_ms']/n, 4) for k, v in tm.items()})}")
