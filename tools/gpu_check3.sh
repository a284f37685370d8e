bash tools/build_sweep.sh
TQP_HOST_PROF=1 timeout 300 python tools/host_overhead.py > gpurun_out/host.log 2> gpurun_out/host_err.log; tail -4 gpurun_out/host.log
