timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gputests.log
TQP_HOST_PROF=1 timeout 300 python tools/host_overhead.py > gpurun_out/host.log 2> gpurun_out/host_err.log; tail -4 gpurun_out/host.log
for tag in "exec" "unit"; do grep "host $tag" gpurun_out/host_err.log | tail -150 | awk '{$1=$2=$3=""; print}' | sort | uniq -c | sort -rn | head -6; done
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], {q: (round(v['latency_ms'],3), {k: round(u['total_ms']/u['calls'],3) for k,u in v['units'].items()}) for q,v in d['queries'].items()})"
