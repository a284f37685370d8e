timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/gputests.log
grep -E "FAIL|PASS sqlx|PASS q3.sql" -m 10 gpurun_out/gputests.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], {q: round(v['latency_ms'], 3) for q, v in d['queries'].items()})
print('roofline', d['roofline']['kernel'], round(d['roofline']['frac'], 3), 'e2e', d['e2e']['value'] if d.get('e2e') else None)
print('hash_group', {k: d['hash_group'][k] for k in ('latency_ms', 'hbm_frac', 'per_instruction_ms')})
print('per_instruction', d['per_instruction']['latency_ms'])
print('cpu', d['cpu_baseline']['value'] if d.get('cpu_baseline') else None, d['clocks'])
PY
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('dropin', json.dumps(d.get('dropin_e2e'))[:800])
PY
