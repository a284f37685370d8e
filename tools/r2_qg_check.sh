# qg (hash-group) parity, random group plans, bench leg and ncu capture of its scan kernel
export TQP_DEBUG_FALLBACK=1
timeout 900 python -m pytest tests/test_hash_group_gpu.py tests/test_random_plans_gpu.py tests/test_sharded_gpu.py -m gpu -x -q > gpurun_out/qg_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/qg_tests.log
for seed in 2 3 5 6; do timeout 600 oracle/_ref/tqp_random_plans --profile groups --seed $seed --plans 60 --require-fused 1 > gpurun_out/hash_rp_$seed.log 2>&1; tail -1 gpurun_out/hash_rp_$seed.log; done
cat gpurun_out/hash_rp_*.log | grep -o "tqp: .*" | sort | uniq -c
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-csv > gpurun_out/qg_bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/qg_bench.log').read().strip().splitlines()[-1]); h=d['hash_group']; print(json.dumps({k: h[k] for k in h if k not in ('explain',)}, indent=0)[:3000]); print(d['ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_count|k_group|k_radix|k_compact" -o gpurun_out/r2_qg_full python tools/run_queries.py --sf 10 --queries qg --iters 1 > gpurun_out/r2_qg_full.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/r2_qg_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct > gpurun_out/r2_qg_raw.csv 2>&1; head -30 gpurun_out/r2_qg_raw.csv | cut -c1-300
