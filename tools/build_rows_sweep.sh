# q_build rows-per-thread sweep (launch list of the Q3 build sides)
for r in 2 4 8; do
  TQP_BUILD_ROWS=$r timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_build --csv --log-file gpurun_out/brows_$r.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo rows=$r; grep q_build gpurun_out/brows_$r.csv | tail -3 | awk -F'","' '{print $NF}'
done
