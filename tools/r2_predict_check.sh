for s in 1 2; do timeout 600 oracle/_ref/tqp_predict_test --seed $s --rows 20000 2>&1 | tail -12; done
timeout 600 python -m pytest tests/test_dropin_gpu.py tests/test_kernels_gpu.py -m gpu -x -q 2>&1 | tail -3
