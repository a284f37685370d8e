#!/usr/bin/env bash
# Regenerates tests/golden/ from the UNMODIFIED reference (run in the build
# container, where /root/reference exists). Test infrastructure only.
set -euo pipefail
cd "$(dirname "$0")"
make -j8 >/dev/null
G=../tests/golden
./_ref/golden_cases kernels $G/kernels.json
./_ref/golden_cases plans $G/plans.json _ref/queries
./_ref/csv_cases $G/csv.json
./_ref/tqp_ref_runner opplan --out ../paper_2209_04579_b200/plans
SF=0.005
./_ref/tqp_ref_runner tables --sf $SF --out /tmp/tqp_tables.json
./_ref/tqp_ref_runner run --sf $SF --repeat 0 --warmup 0 --results /tmp/tqp_results.json >/dev/null
python3 - "$SF" <<'PY'
import gzip, json, sys
sf = float(sys.argv[1])
t = json.load(open('/tmp/tqp_tables.json')); r = json.load(open('/tmp/tqp_results.json'))
doc = {"generator": "oracle/make_golden.sh: tqp_ref_runner tables/run (reference executor, par backend)",
       "sf": sf, "seed": 7, "tables": t, "results": r["results"]}
with gzip.open('../tests/golden/tpch_sf%s.json.gz' % sys.argv[1], 'wt') as f:
    json.dump(doc, f)
PY

# Full-size results (tables are regenerated bit-identically on the device by
# include/tqp_gen.h, so only the reference executor's results are committed).
for SF in 1 10; do
  ./_ref/tqp_ref_runner run --sf $SF --repeat 0 --warmup 0 --results /tmp/tqp_results_sf$SF.json >/dev/null
  python3 - "$SF" <<'PY'
import json, sys
sf = sys.argv[1]
r = json.load(open('/tmp/tqp_results_sf%s.json' % sf))
doc = {"generator": "oracle/make_golden.sh: tqp_ref_runner run (reference executor, par backend)",
       "sf": float(sf), "seed": 7, "lineitem_rows": r["lineitem_rows"], "results": r["results"]}
json.dump(doc, open('../tests/golden/tpch_results_sf%s.json' % sf, 'w'), indent=0)
PY
done

# qg (GROUP BY l_partkey, the hash-group workload): reference results at SF0.05 and SF1
for SF in 0.05 1; do
  ./_ref/tqp_ref_runner run --sf $SF --queries qg --repeat 0 --warmup 0 --results /tmp/tqp_qg_sf$SF.json >/dev/null
  python3 - "$SF" <<'PY'
import gzip, json, sys
sf = sys.argv[1]
r = json.load(open('/tmp/tqp_qg_sf%s.json' % sf))
doc = {"generator": "oracle/make_golden.sh: tqp_ref_runner run --queries qg (reference executor, par backend)",
       "sf": float(sf), "seed": 7, "lineitem_rows": r["lineitem_rows"], "results": r["results"]}
with gzip.open('../tests/golden/qg_results_sf%s.json.gz' % sf, 'wt') as f:
    json.dump(doc, f)
PY
done
