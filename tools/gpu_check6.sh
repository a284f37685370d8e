TQP_HOST_PROF=1 timeout 300 python tools/host_overhead.py > gpurun_out/host.log 2> gpurun_out/host_err.log; tail -4 gpurun_out/host.log
for tag in "exec" "unit"; do grep "host $tag" gpurun_out/host_err.log | tail -150 | awk '{$1=$2=$3=""; print}' | sort | uniq -c | sort -rn | head -8; done
