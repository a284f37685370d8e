export TQP_DEBUG_FALLBACK=1
for seed in 1 2 3 4 5 6; do timeout 600 oracle/_ref/tqp_random_plans --profile groups --seed $seed --plans 60 --require-fused 1 > gpurun_out/hash_rp_$seed.log 2>&1; grep -m4 "FAIL" gpurun_out/hash_rp_$seed.log | cut -c1-300; tail -1 gpurun_out/hash_rp_$seed.log; done
cat gpurun_out/hash_rp_*.log | grep -o "tqp: .*" | sort | uniq -c
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/gputests.log; grep -m3 "FAIL plan" gpurun_out/gputests.log | cut -c1-300
