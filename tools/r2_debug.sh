# first failing random plan of a seed/profile, then that plan under compute-sanitizer
PROFILE=${PROFILE:-groups}; SEED=${SEED:-1}; N=${N:-60}
timeout 600 oracle/_ref/tqp_random_plans --profile $PROFILE --seed $SEED --plans $N > gpurun_out/dbg_full.log 2>&1
grep -m3 "FAIL" gpurun_out/dbg_full.log | cut -c1-300; tail -1 gpurun_out/dbg_full.log
first=$(grep -m1 -o "FAIL plan [0-9]*" gpurun_out/dbg_full.log | awk '{print $3}')
if [ -n "$first" ]; then
  timeout 600 compute-sanitizer --print-limit 10 oracle/_ref/tqp_random_plans --profile $PROFILE --seed $SEED --plans $N --only $first > gpurun_out/dbg_san.log 2>&1
  grep -v "^  " gpurun_out/dbg_san.log | head -60
fi
