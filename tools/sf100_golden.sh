#!/usr/bin/env bash
# SF100 golden results from the UNMODIFIED reference executor (oracle/_ref/
# tqp_ref_runner, par backend, every host core), run on a GPU box's host
# (196 GB RAM, 16 cores; the build container has 62 GB). Test infrastructure:
# writes gpurun_out/tpch_results_sf100.json, committed as
# tests/golden/tpch_results_sf100.json (the device regenerates the tables
# bit-identically from include/tqp_gen.h, so only the results are kept).
#
#   gpurun --timeout 2400 -- bash tools/sf100_golden.sh
set -uo pipefail
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# a failed allocation must end the runner, not the box: cap the address space
ulimit -v 185000000
free -g > gpurun_out/sf100_golden_host.txt
nproc >> gpurun_out/sf100_golden_host.txt
start=$(date +%s)
./oracle/_ref/tqp_ref_runner run --sf 100 --queries q6,q14,q3,q1 --repeat 0 --warmup 0 \
    --results gpurun_out/tpch_results_sf100_raw.json > gpurun_out/sf100_golden_log.jsonl 2> gpurun_out/sf100_golden.err
rc=$?
echo "rc=$rc wall_s=$(( $(date +%s) - start ))" >> gpurun_out/sf100_golden_host.txt
[ $rc -eq 0 ] || exit $rc
python3 - <<'PY'
import json
r = json.load(open('gpurun_out/tpch_results_sf100_raw.json'))
doc = {"generator": "tools/sf100_golden.sh: tqp_ref_runner run --sf 100 (reference executor, par backend, "
                    "16 host cores of the GPU box)",
       "sf": 100.0, "seed": 7, "lineitem_rows": r["lineitem_rows"], "results": r["results"]}
json.dump(doc, open('gpurun_out/tpch_results_sf100.json', 'w'), indent=0)
PY
