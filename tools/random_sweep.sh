# Broad random-plan parity sweep (beyond the seeds pinned in the tests):
# default dispatch and every fused unit on NVRTC kernels (TQP_JIT=1)
run() {  # seed jit
  out=$(TQP_JIT=$2 timeout 900 oracle/_ref/tqp_random_plans --seed $1 --plans 250 2>&1 | tail -3)
  echo "seed=$1 jit=$2 $(echo "$out" | grep -o '[0-9]* failure(s)')"
  echo "$out" | grep -q " 0 failure(s)" || echo "$out" > gpurun_out/rand_fail_$1_$2.txt
}
export -f run
( for s in $(seq ${SEED0:-300} $(( ${SEED0:-300} + 39 ))); do echo "$s 0"; echo "$s 1"; done ) | xargs -P 8 -n 2 bash -c 'run "$0" "$1"' | sort -t= -k2 -n > gpurun_out/random_sweep.txt
grep -c " 0 failure" gpurun_out/random_sweep.txt; grep -v " 0 failure" gpurun_out/random_sweep.txt | head
