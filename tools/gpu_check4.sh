timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gputests.log
TQP_B200_LIB=tools/_prof/libtqp_b200.so timeout 200 python tools/run_queries.py --sf 10 --queries q3 --iters 3 2>&1 | grep topk | tail -8
for r in 1 2; do TQP_BUILD_ROWS=$r timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_build --csv --log-file gpurun_out/bsw.csv python tools/run_queries.py --sf 10 --queries q3 --iters 3 > /dev/null 2>&1
  echo rows=$r $(grep q_build gpurun_out/bsw.csv | tail -2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '); done
TQP_HOST_PROF=1 timeout 300 python tools/host_overhead.py > gpurun_out/host.log 2> gpurun_out/host_err.log; tail -4 gpurun_out/host.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], {q: (round(v['latency_ms'],3), {k: round(u['total_ms']/u['calls'],3) for k,u in v['units'].items()}) for q,v in d['queries'].items()})"
