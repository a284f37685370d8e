"""Generic scan kernels at 60 M rows: prefix_sum_exclusive (int64) and
compact (int64 values, ~50 % mask); median of 10 with CUDA events on the
library stream, GB/s over read + write bytes:  python tools/scan_probe.py"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
n = 60_000_000
rng = np.random.default_rng(1)
x = tqp.Tensor.from_numpy(rng.integers(0, 1000, n, dtype=np.int64), ctx=ctx)
m = tqp.Tensor.from_numpy(rng.random(n) < 0.5, ctx=ctx)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
def t(f, nbytes, name):
    for _ in range(3): f()
    ctx.sync()
    v = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); r = f(); b.record(stream); b.synchronize(); v.append(a.elapsed_time(b))
    v.sort()
    ms = v[5]
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
t(lambda: tqp.prefix_sum_exclusive(x, ctx=ctx), 16 * n, "prefix_sum")
t(lambda: tqp.compact(x, m, ctx=ctx), 9 * n + 4 * n, "compact")
