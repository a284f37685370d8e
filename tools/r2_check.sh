set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 3000 gpurun_out/bench.log
