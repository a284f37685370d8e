# end-of-round ncu captures on the final code: --set full of one execution of
# each suite query and of qg (SF10), stall / DRAM summary per kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"q_tile|q_build|k_topk|k_final|k_nonzero_slots|k_group_rows" -o gpurun_out/r2m_full python tools/run_queries.py --sf 10 --queries q1,q6,q14,q3,qg --iters 1 > gpurun_out/r2m_full.log 2>&1; echo full_rc=$?
python tools/ncu_stalls.py gpurun_out/r2m_full.ncu-rep --tag q1,q1,q6,q6,q14,q14,q14,q3,q3,q3,q3,qg,qg,qg > gpurun_out/r2m_kernel_stalls.txt 2>&1; head -60 gpurun_out/r2m_kernel_stalls.txt
