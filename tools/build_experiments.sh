# Q3 orders build: cost of each insert side effect (timing only; results invalid)
for x in NONE NOZERO NOTABLE NOBITMAP NODUP NOMATCH NOZERO,NOTABLE,NOBITMAP; do
  TQP_BUILD_EXPERIMENT=$x timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:q_build --csv --log-file gpurun_out/bx.csv python tools/run_queries.py --sf 10 --queries q3 --iters 2 > /dev/null 2>&1
  echo $x; grep q_build gpurun_out/bx.csv | tail -3 | awk -F'","' '{print $(NF-2), $NF}'
done
