bash tools/gpu_check.sh
for m in none torch; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q_tile --csv --log-file gpurun_out/a.csv python tools/q1_torch_probe.py $m > /dev/null 2>&1
echo $m $(grep q_tile gpurun_out/a.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
done
