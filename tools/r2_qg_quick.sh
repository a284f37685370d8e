python tools/run_queries.py --sf 10 --queries qg --iters 6 2>&1 | tail -2 | cut -c1-600
TQP_NO_EVICT_FIRST=1 python tools/run_queries.py --sf 10 --queries qg --iters 6 2>&1 | tail -2 | cut -c1-600
timeout 300 python -m pytest tests/test_hash_group_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 600 ncu --clock-control none -k regex:"k_tile" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct python tools/run_queries.py --sf 10 --queries qg --iters 1 2>&1 | grep -E "k_tile|dram__|gpu__time|lts__" | head
