#!/bin/bash
# End-of-round evidence on the final code (one GPU): GPU suite, the default
# bench line, the launch list of the bench command, SF100, the reference arm.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-csv > gpurun_out/ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -12 gpurun_out/launches_summary.txt
timeout 1200 python bench.py --sf 100 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-csv > gpurun_out/bench_sf100.log 2>&1; echo sf100_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
tail -c 600 gpurun_out/bench_ref.log
