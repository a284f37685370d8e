timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_tpch_scale_gpu.py -m gpu -x -q -k "10-False or 1-False" 2>&1 | tail -2
python tools/q1_nofuse_wall.py lineitem,orders,customer,part 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nofuse_launches.csv python tools/run_queries.py --sf 10 --queries q1 --iters 2 --no-fuse > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/nofuse_launches.csv 2>&1 | head -24
