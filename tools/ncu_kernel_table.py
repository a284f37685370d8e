"""Per-kernel table from an ncu --csv log with gpu__time_duration.sum and
dram__bytes_{read,write}.sum: launches, total time, DRAM GB and achieved GB/s
against MEASURED_PEAKS.json's HBM figure (when present).

    python tools/ncu_kernel_table.py launches.csv [--last-half]
--last-half keeps the second half of the launches (the warm execution when
the command ran the workload twice)."""
import csv
import json
import sys
from collections import OrderedDict
from pathlib import Path


def main(path, last_half=False):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ls = list(launches.values())
    if last_half:
        ls = ls[len(ls) // 2:]
    peak = None
    mp = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            peak = float(json.loads(mp.read_text()).get("hbm_gbs"))
        except Exception:
            peak = None
    peak = peak or 6556.0
    agg = OrderedDict()
    for d in ls:
        name = d["name"].split("(")[0].replace("void ", "").replace("tqp::<unnamed>::", "").replace("tqp::", "")[:48]
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / 1e9
    tot_t = sum(a[1] for a in agg.values())
    tot_b = sum(a[2] for a in agg.values())
    print(f"{'kernel':48} {'n':>4} {'us':>9} {'share':>6} {'GB':>7} {'GB/s':>7} {'of_peak':>7}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48} {n:4d} {t:9.1f} {t / tot_t:6.1%} {b:7.3f} {b / t * 1e6 if t else 0:7.0f} {b / t * 1e6 / peak if t else 0:7.2f}")
    print(f"{'total':48} {len(ls):4d} {tot_t:9.1f} {'':6} {tot_b:7.3f} {tot_b / tot_t * 1e6:7.0f} {tot_b / tot_t * 1e6 / peak:7.2f}")


if __name__ == "__main__":
    main(sys.argv[1], "--last-half" in sys.argv)
