"""Occupancy / issue / DRAM / warp-stall mix per kernel of an ncu --set full
capture (.ncu-rep), as committed under profiles/ (r*_kernel_stalls.txt).

    python tools/ncu_stalls.py REP.ncu-rep [--tag q1,q1,...]
"""
import argparse
import csv
import io
import subprocess

SHOW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic"]
PFX = "smsp__pcsamp_warps_issue_stalled_"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    tags = [t for t in a.tag.split(",") if t]
    stall = [i for i, h in enumerate(hdr) if h.startswith(PFX) and not h.endswith("not_issued")]
    for n, r in enumerate(data):
        name = r[hdr.index("Kernel Name")][:60]
        print(f"== {tags[n] + ' ' if n < len(tags) else ''}{name}")
        for m in SHOW:
            if m in hdr:
                print(f"  {m:55s} {r[hdr.index(m)]} {units[hdr.index(m)]}")
        tot = sum(float(r[i] or 0) for i in stall) or 1.0
        top = sorted(((float(r[i] or 0) / tot, hdr[i][len(PFX):]) for i in stall), reverse=True)[:6]
        print("  stalls: " + ", ".join(f"{k}={v:.0%}" for v, k in top))
        print()


if __name__ == "__main__":
    main()
