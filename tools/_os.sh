timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py tests/test_oracle.py -m gpu -x -q > gpurun_out/os_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/os_tests.log
timeout 900 python -m pytest tests/test_tpch_scale_gpu.py tests/test_random_plans_gpu.py tests/test_hash_group_gpu.py -m gpu -x -q > gpurun_out/os_tests2.log 2>&1; echo tests2_rc=$?; tail -3 gpurun_out/os_tests2.log
bash tools/r2_nofuse_ncu.sh 2>&1 | grep -E "rc=|onesweep|os_hist|total|k_scatter|k_hist"
