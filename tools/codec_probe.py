"""Per-column upload time of the compressed host format vs the raw layout
(pinned host memory, SF10 tables; device time with CUDA events)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2209_04579_b200 import tqp
ctx = tqp.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
for n in ("lineitem", "orders"):
    t = tqp.Table.generate(n, float(sys.argv[1]) if len(sys.argv) > 1 else 10, 7, ctx=ctx)
    for cname, lt in t.columns():
        dev = t.column(cname)
        arr = dev.numpy(widen_strings=False)
        codec, payload = tqp.encode_column(arr, dev.dtype)
        pin = torch.from_numpy(payload).pin_memory()
        raw = torch.from_numpy(arr).pin_memory()
        res = []
        for kind in ("enc", "raw"):
            for _ in range(2):
                if kind == "enc":
                    x = tqp.Tensor.from_encoded(codec, pin, dev.dtype, arr.shape[0], arr.shape[1], ctx=ctx)
                else:
                    x = tqp.Tensor.from_numpy(raw.numpy(), dev.dtype, ctx=ctx)
            ctx.sync()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                if kind == "enc":
                    x = tqp.Tensor.from_encoded(codec, pin, dev.dtype, arr.shape[0], arr.shape[1], ctx=ctx)
                else:
                    x = tqp.Tensor.from_numpy(raw.numpy(), dev.dtype, ctx=ctx)
            e1.record(stream); e1.synchronize()
            res.append(e0.elapsed_time(e1) / 5)
        print(f"{n}.{cname:18s} {codec.name}{codec.width:<3d} {payload.nbytes/1e6:8.1f} MB enc {res[0]:7.3f} ms  raw {arr.nbytes/1e6:8.1f} MB {res[1]:7.3f} ms")
