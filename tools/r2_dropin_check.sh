timeout 600 oracle/_ref/tqp_dropin_test --sf 0.01 --gpus 2 2>&1 | tail -12
timeout 900 oracle/_ref/tqp_dropin_bench --sf 1 --reps 5
