for v in new old; do
  if [ $v = new ]; then S=tools/run_queries.py; else S=_old/run_queries.py; fi
  ncu --clock-control none -k regex:q_tile --launch-skip 1 --launch-count 1 --section LaunchStats --section SpeedOfLight --metrics launch__registers_per_thread,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,gpu__time_duration.sum,dram__bytes_read.sum python $S --sf 10 --queries q1 --iters 3 2>&1 | grep -E "Registers|Shared Memory|gpu__time|dram__bytes|launch__|Duration|Threads" | head -20
  echo ====
  TQP_HOST_PROF=1 python $S --sf 10 --queries q1 --iters 4 2>&1 | grep "tqp host" | tail -2
done
