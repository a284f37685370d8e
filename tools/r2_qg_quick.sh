export TQP_DEBUG_FALLBACK=1
timeout 600 python -m pytest tests/test_hash_group_gpu.py -m gpu -x -q 2>&1 | tail -2
for seed in 1 2 3; do timeout 600 oracle/_ref/tqp_random_plans --profile groups --seed $seed --plans 60 --require-fused 1 2>&1 | tail -1; done
python tools/run_queries.py --sf 10 --queries qg --iters 6 2>&1 | tail -1 | cut -c1-400
TQP_HASH_NOPART=1 python tools/run_queries.py --sf 10 --queries qg --iters 6 2>&1 | tail -1 | cut -c1-400
timeout 600 ncu --clock-control none -k regex:"k_tile|k_hash_part" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct python tools/run_queries.py --sf 10 --queries qg --iters 1 2>&1 | grep -E "k_tile|k_hash|dram__|gpu__time|lts__" | head -12
