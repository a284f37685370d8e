# Q1 small-group kernel variants: per-launch time (ncu launch list, SF10)
run() {
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_tile --csv --log-file gpurun_out/q1sw.csv python tools/run_queries.py --sf 10 --queries q1 --iters 3 > gpurun_out/q1sw.log 2>&1
  echo "$@" $(grep q_tile gpurun_out/q1sw.csv | tail -2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
}
run TQP_SMALL_REG=0
for c in "10 1280" "12 1536" "14 1792" "12 1152" "14 1344" "12 768" "10 960"; do set -- $c; run TQP_SMALL_REG=1 TQP_SMALL_CW=$1 TQP_SMALL_ROWS=$2; done
