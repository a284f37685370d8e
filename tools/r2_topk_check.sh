# top-k rewrite: parity (executor, TPC-H at scale, random plans) and the
# k_topk_groups launch time per walk-blocks-per-SM setting (ncu, Q3 SF10)
timeout 180 python -m pytest tests/test_executor_gpu.py -k "tpch_sf0005 or golden" -x -q > gpurun_out/topk_quick.log 2>&1 || { echo quick_fail; tail -5 gpurun_out/topk_quick.log; exit 1; }
timeout 1200 python -m pytest tests/test_executor_gpu.py tests/test_tpch_scale_gpu.py tests/test_random_plans_gpu.py tests/test_hash_group_gpu.py tests/test_jit_gpu.py -m gpu -x -q > gpurun_out/topk_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/topk_tests.log
for b in 2 4 6 8; do
  TQP_TOPK_BPS=$b timeout 300 ncu --clock-control none -k regex:"k_topk|q_build" --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --csv python tools/run_queries.py --sf 10 --queries q3 --iters 3 2>/dev/null | grep -E "k_topk|q_build" | awk -F'","' -v b=$b '{print "bps=" b, $5, $(NF-2), $(NF)}' | tail -6
done
python tools/run_queries.py --sf 10 --queries q3 --iters 20 2>&1 | cut -c1-600
