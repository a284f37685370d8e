export TQP_DEBUG_FALLBACK=1
timeout 900 python -m pytest tests/test_sharded_exec_gpu.py -m gpu -x -q > gpurun_out/shard_tests.log 2>&1; echo tests_rc=$?; tail -30 gpurun_out/shard_tests.log | cut -c1-300
