"""Does initialising torch's CUDA context first change the Q1 scan kernel?
(bench.py imports torch before the library; tools/run_queries.py does not)"""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
mode = sys.argv[1] if len(sys.argv) > 1 else "none"
if mode != "none":
    import torch
    torch.cuda.set_device(0)
    if mode == "stream":
        pass
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
if mode == "stream":
    s = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
ex = tqp.Executor(json.loads((ROOT / "paper_2209_04579_b200" / "plans" / "q1.opplan.json").read_text()), ctx=ctx)
for _ in range(3):
    ex.execute(tables)
