"""SF100 on one B200: the four queries unsharded vs 8 order-aligned shards
merged through execute_partial/finish; integers, keys and
Q3's exact sums must be bit-identical, fp64 scan sums within 1e-9. Writes
profiles/r1c_sf100_check.json. (The reference executor needs > 190 GB of host
RAM at SF100, so parity there is by this property plus the SF1/SF10 goldens.)"""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2209_04579_b200 import tqp

sf = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
nsh = 8
ctx = tqp.Context(0)
plans = {q: json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text()) for q in ("q1", "q6", "q14", "q3")}
out = {"sf": sf, "shards": nsh, "queries": {}}
t0 = time.time()
full = {n: tqp.Table.generate(n, sf, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
out["lineitem_rows"] = full["lineitem"].rows
want = {}
for q, p in plans.items():
    ex = tqp.Executor(p, ctx=ctx)
    ex.execute(full)
    ctx.sync()
    t = time.perf_counter(); res = ex.execute(full).to_numpy(); ms = (time.perf_counter() - t) * 1e3
    want[q] = res
    out["queries"][q] = {"latency_ms_wall": ms, "rows": int(len(res[0][2]))}
del full
ctx.sync()
for q, p in plans.items():
    ex = tqp.Executor(p, ctx=ctx)
    parts = []
    for s in range(nsh):
        tabs = {n: tqp.Table.generate(n, sf, 7, shard=s if n in ("lineitem", "orders") else 0,
                                      nshards=nsh if n in ("lineitem", "orders") else 1, ctx=ctx)
                for n in ("lineitem", "orders", "customer", "part")}
        parts.append(ex.execute_partial(tabs))
        del tabs
        ctx.sync()
    got = ex.finish(parts).to_numpy()
    ok = True
    maxrel = 0.0
    for (n, t, g), (_, _, w) in zip(got, want[q]):
        if g.dtype == np.float64 and q != "q3":
            rel = float(np.max(np.abs(g - w) / np.maximum(1.0, np.abs(w)))) if g.size else 0.0
            maxrel = max(maxrel, rel)
            ok = ok and rel <= 1e-9
        else:
            ok = ok and np.array_equal(np.asarray(g).view(np.uint8), np.asarray(w).view(np.uint8))
    out["queries"][q].update({"sharded_equals_unsharded": ok, "max_rel_fp64_diff": maxrel})
    out["queries"][q]["result_head"] = {n: (np.asarray(w)[:3].tolist() if t != "utf8" else None) for n, t, w in want[q]}
out["wall_s"] = time.time() - t0
(ROOT / "profiles").mkdir(exist_ok=True)
(ROOT / "profiles" / "r1b_sf100_check.json").write_text(json.dumps(out, indent=1, default=str))
print(json.dumps({q: {k: v for k, v in d.items() if k != "result_head"} for q, d in out["queries"].items()}))
