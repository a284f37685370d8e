#!/bin/bash
# last-session evidence on the final hash-group kernels: random-plan sweep (default and
# all-NVRTC) and the random group-plan profile
set -u
mkdir -p gpurun_out
# (compute-sanitizer is closed on the GPU pool since this round's first sanitizer pass)
SEED0=700 bash tools/random_sweep.sh
export TQP_DEBUG_FALLBACK=1
for seed in $(seq 30 39); do timeout 600 oracle/_ref/tqp_random_plans --profile groups --seed $seed --plans 60 2>&1 | tail -1; done > gpurun_out/random_groups.txt
cat gpurun_out/random_groups.txt
