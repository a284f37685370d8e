# Q3 changes (top-k rewrite, unique-key builds): quick parity gate, Q3 latency
# per top-k blocks-per-SM and build rows-per-thread setting, launch list
timeout 240 python -m pytest tests/test_executor_gpu.py -k "tpch_sf0005 or golden" -x -q > gpurun_out/q3_quick.log 2>&1 || { echo quick_fail; tail -5 gpurun_out/q3_quick.log; exit 1; }
timeout 1200 python -m pytest tests/test_executor_gpu.py tests/test_tpch_scale_gpu.py tests/test_random_plans_gpu.py tests/test_hash_group_gpu.py tests/test_jit_gpu.py -m gpu -x -q > gpurun_out/q3_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/q3_tests.log
for b in 2 4 8; do echo "bps=$b"; TQP_TOPK_BPS=$b timeout 200 python tools/query_time.py --queries q3 --iters 30; done
for r in 1 2 4; do echo "build_rows=$r"; TQP_BUILD_ROWS=$r timeout 200 python tools/query_time.py --queries q3 --iters 30; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q3_launches.csv python tools/run_queries.py --sf 10 --queries q3 --iters 3 > /dev/null 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/q3_launches.csv
