"""Summarises an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'total_ms':>9} {'n':>4} {'avg_us':>10} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:top]:
        print(f"{sum(v)/1e6:9.3f} {len(v):4d} {sum(v)/len(v)/1e3:10.1f} {sum(v)/total:6.1%}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
