timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nofuse_launches.csv python tools/run_queries.py --sf 10 --queries q1 --iters 1 --no-fuse > gpurun_out/nofuse_run.log 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/nofuse_launches.csv 2>&1 | head -30
