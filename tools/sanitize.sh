#!/bin/bash
# compute-sanitizer over the GPU parity suite at small sizes:
# memcheck on every small-SF GPU test module, racecheck + synccheck on the
# fused TPC-H path (TMA/mbarrier rings, lookback scans, top-k) and the
# generic kernels. Logs -> gpurun_out/sanitize_*.log
set -u
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 50"
SMALL="tests/test_kernels_gpu.py tests/test_executor_gpu.py tests/test_jit_gpu.py tests/test_sharded_gpu.py tests/test_csv.py tests/test_codec.py tests/test_dropin_gpu.py"
export TQP_SANITIZE=1
timeout 2400 $CS --tool memcheck --leak-check no python -m pytest $SMALL -m gpu -x -q -p no:cacheprovider > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck_rc=$?
tail -5 gpurun_out/sanitize_memcheck.log
for tool in racecheck synccheck; do
  timeout 1800 $CS --tool $tool python -m pytest tests/test_executor_gpu.py tests/test_kernels_gpu.py tests/test_jit_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1; echo ${tool}_rc=$?
  tail -5 gpurun_out/sanitize_$tool.log
done
