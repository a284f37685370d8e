"""Summarises an `ncu --set full` capture (.ncu-rep) into profiles/ JSON.

    python tools/ncu_summary.py REP.ncu-rep OUT.json [--traffic profiles/kernel_traffic.json] [--tag q1,q6,...]

`--tag` names the captured launches in order (e.g. the query each fused scan
kernel ran for) so bench.py can look their DRAM traffic up as "<tag>:<kernel>".
"""
import argparse
import csv
import io
import json
import re
import subprocess

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name: str) -> str:
    m = re.match(r"(?:void )?(?:[\w:]+::)?(\w+(?:<[^()]*>)?)", name)
    return m.group(1) if m else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    tags = [t for t in a.tag.split(",") if t]
    out = {"units": {m: units[hdr.index(m)] for m in METRICS if m in hdr}, "kernels": {}}
    traffic = {}
    for i, r in enumerate(data):
        name = short(r[ki])
        key = f"{tags[i]}:{name}" if i < len(tags) else f"{i}:{name}"
        rec = {m: r[hdr.index(m)] for m in METRICS if m in hdr}
        out["kernels"][key] = rec
        if "dram__bytes_read.sum" in hdr:
            rd = float(rec["dram__bytes_read.sum"].replace(",", "")) * SCALE.get(out["units"]["dram__bytes_read.sum"], 1)
            wr = float(rec["dram__bytes_write.sum"].replace(",", "")) * SCALE.get(out["units"]["dram__bytes_write.sum"], 1)
            traffic[key] = rd + wr
    json.dump(out, open(a.out, "w"), indent=1)
    if a.traffic:
        json.dump(traffic, open(a.traffic, "w"), indent=1)
    for k, v in out["kernels"].items():
        print(k, v.get("gpu__time_duration.sum"), "ms", traffic.get(k))


if __name__ == "__main__":
    main()
