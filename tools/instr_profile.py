"""Per-instruction device profile of a lowered plan (Executor.profile_execute:
a synchronisation after every instruction, the reference's ProfileTrace
shape), top instructions by time.

    python tools/instr_profile.py --sf 10 --query q1 [--fuse]
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
    ap.add_argument("--query", default="q1")
    ap.add_argument("--fuse", action="store_true")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    ctx = tqp.default_context()
    tables = {n: tqp.Table.generate(n, a.sf, 7, ctx=ctx) for n in ("lineitem", "orders", "customer", "part")}
    plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{a.query}.opplan.json").read_text())
    ex = tqp.Executor(plan, fuse=a.fuse, ctx=ctx)
    ex.execute(tables)
    _, trace = ex.profile_execute(tables)
    ev = trace if isinstance(trace, list) else trace.get("traceEvents", [])
    ev = [e for e in ev if isinstance(e, dict) and e.get("dur") is not None]
    tot = sum(e["dur"] for e in ev if e.get("cat", "") != "operator")
    print(f"{len(ev)} events")
    for e in sorted(ev, key=lambda e: -e["dur"])[: a.top]:
        print(f"{e['dur'] / 1e3:9.3f} ms  {e.get('cat', '')}  {e.get('name', '')}  {json.dumps(e.get('args', {}))[:120]}")


if __name__ == "__main__":
    main()
