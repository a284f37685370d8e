"""qg (GROUP BY l_partkey) hash kernel time vs scale factor (table size vs
L2) — experiment aid: python tools/qg_l2_probe.py SF [SF ...]"""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
plan = json.loads((ROOT / "paper_2209_04579_b200/plans/qg.opplan.json").read_text())
for sf in [float(x) for x in sys.argv[1:]]:
    t = {"lineitem": tqp.Table.generate("lineitem", sf, 7, ctx=ctx)}
    ex = tqp.Executor(plan, ctx=ctx)
    ex.set_timing(True)
    for _ in range(3): ex.execute(t)
    ex.reset_timings()
    for _ in range(5): ex.execute(t)
    tm = ex.timings()
    k = {n: round(v["total_ms"] / v["calls"], 4) for n, v in tm.items()}
    rows = 6e6 * sf
    kt = [v for n, v in k.items() if n.startswith("kernel:") and "_tile<" in n]
    print(f"sf {sf}: {k}  ns/row {kt[0] * 1e6 / rows:.3f}" if kt else k, flush=True)
    del t, ex
