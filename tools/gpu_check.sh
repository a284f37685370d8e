timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/gputests.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], {q: (round(v['latency_ms'],3), {k: round(u['total_ms']/u['calls'],3) for k,u in v['units'].items()}) for q,v in d['queries'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo done
