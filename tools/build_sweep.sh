# Q3 build-side kernel shapes: per-launch times (ncu launch list, SF10)
run() {
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_build --csv --log-file gpurun_out/bsw.csv python tools/run_queries.py --sf 10 --queries q3 --iters 3 > /dev/null 2>&1
  echo "$@" $(grep q_build gpurun_out/bsw.csv | tail -2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
}
run TQP_BUILD_ROWS=4
run TQP_BUILD_ROWS=8
run TQP_BUILD_ROWS=2
run TQP_BUILD_TILE=1 TQP_BUILD_TILE_CW=16 TQP_BUILD_TILE_ROWS=2048
run TQP_BUILD_TILE=1 TQP_BUILD_TILE_CW=16 TQP_BUILD_TILE_ROWS=4096
run TQP_BUILD_TILE=1 TQP_BUILD_TILE_CW=24 TQP_BUILD_TILE_ROWS=3072
run TQP_BUILD_TILE=1 TQP_BUILD_TILE_CW=31 TQP_BUILD_TILE_ROWS=3968
run TQP_BUILD_TILE=1 TQP_BUILD_TILE_CW=8 TQP_BUILD_TILE_ROWS=2048
