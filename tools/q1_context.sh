for m in none torch; do for c in "14 1792" "13 1664" "10 1280" "12 1536"; do set -- $c
TQP_SMALL_CW=$1 TQP_SMALL_ROWS=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_tile --csv --log-file gpurun_out/a.csv python tools/q1_torch_probe.py $m > /dev/null 2>&1
echo $m $c $(grep q_tile gpurun_out/a.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
done; done
TQP_SMALL_REG=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_tile --csv --log-file gpurun_out/a.csv python tools/q1_torch_probe.py torch > /dev/null 2>&1
echo torch cells $(grep q_tile gpurun_out/a.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
