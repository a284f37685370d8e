"""Runs TPC-H queries through the B200 executor (for ncu / nsight captures).

    python tools/run_queries.py --sf 10 --queries q1,q6 --iters 2 [--no-fuse]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2209_04579_b200 import tqp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10)
    ap.add_argument("--queries", default="q1,q6,q14,q3")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--no-fuse", action="store_true")
    a = ap.parse_args()
    ctx = tqp.default_context()
    tables = {n: tqp.Table.generate(n, a.sf, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
    for q in a.queries.split(","):
        plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text())
        ex = tqp.Executor(plan, fuse=not a.no_fuse, ctx=ctx)
        ex.set_timing(True)
        for _ in range(a.iters):
            res = ex.execute(tables)
        print(q, json.dumps(ex.timings()), [(n, arr.ravel()[:3].tolist()) for n, _, arr in res.to_numpy()][:3])


if __name__ == "__main__":
    main()
