# round-1 final ncu captures: --set full of one execution of each query (SF10)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"q_tile|q_build|k_build|k_topk|k_final" -o gpurun_out/r1d_full python tools/run_queries.py --sf 10 --queries q1,q6,q14,q3 --iters 1 > gpurun_out/r1d_full.log 2>&1; echo full_rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-csv > /dev/null 2>&1; echo launches_rc=$?
