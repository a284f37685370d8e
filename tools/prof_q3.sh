set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"q_build|k_topk" -c 6 -o gpurun_out/q3_full python tools/run_queries.py --sf 10 --queries q3 --iters 2 > gpurun_out/q3_full.log 2>&1
for bt in 0 1; do
TQP_BUILD_TILE=$bt timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q3_launch_bt$bt.csv python tools/run_queries.py --sf 10 --queries q3 --iters 4 > /dev/null 2>&1
TQP_BUILD_TILE=$bt python tools/run_queries.py --sf 10 --queries q3 --iters 20 > gpurun_out/q3_time_bt$bt.log 2>&1
done
