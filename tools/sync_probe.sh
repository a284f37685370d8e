echo base; timeout 300 python tools/host_overhead.py 0.2
echo notiming; TQP_HO_TIMING=0 timeout 300 python tools/host_overhead.py 0.2
echo poll; TQP_SYNC_POLL=1 timeout 300 python tools/host_overhead.py 0.2
