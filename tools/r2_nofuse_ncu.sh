# per-instruction (fuse=False) Q1 and Q3 at SF10: every generic kernel's time
# and DRAM bytes (ncu, one execution after one warm-up), summarised per kernel
for q in q1 q3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/nofuse_$q.csv -k regex:'^(?!k_gen|k_str_maxlen|k_order_lines)' python tools/run_queries.py --sf 10 --queries $q --iters 2 --no-fuse > gpurun_out/nofuse_$q.log 2>&1
  echo "$q rc=$?"
  python tools/ncu_kernel_table.py gpurun_out/nofuse_$q.csv --last-half
done
