"""Times the pieces of Table.load_csv on the lineitem SF1 CSV (tools/ probe)."""
import sys, time, subprocess
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2209_04579_b200 import tqp
path = Path("/tmp/tqp_bench_lineitem_sf1.csv")
if not path.exists():
    subprocess.run([str(ROOT / "oracle/_ref/csv_cases"), "lineitem", "1", str(path)], check=True)
schema = [("l_orderkey", "int64"), ("l_partkey", "int64"), ("l_quantity", "int64"), ("l_extendedprice", "float64"),
          ("l_discount", "float64"), ("l_tax", "float64"), ("l_returnflag", "utf8"), ("l_linestatus", "utf8"),
          ("l_shipdate", "date")]
ctx = tqp.Context(0)
data = path.read_bytes()
for name, fn in (("load_csv(file)", lambda: tqp.Table.load_csv(path, schema, ctx=ctx)),
                 ("from_csv_text(bytes in RAM)", lambda: tqp.Table.from_csv_text(data, schema, ctx=ctx))):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); fn(); ctx.sync(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name}: {sorted(ts)[2]:.1f} ms ({len(data)/1e9/(sorted(ts)[2]/1e3):.2f} GB/s)")
t0 = time.perf_counter(); b = path.read_bytes(); print(f"python read_bytes: {(time.perf_counter()-t0)*1e3:.1f} ms")
