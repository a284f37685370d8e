"""PREDICT on the device: models the reference lowers to
tensor instructions (operator_plan.cpp:521-577; the Hummingbird GEMM tree of
ml_model.cpp:154-231) run on the B200 executor, MatMul on the FP64 tensor
cores (DMMA), fused and per instruction, against tensql::Executor: the
ml_test.cpp fixtures and random trees to depth 8 (oracle/tools/predict_test.cpp)."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = ROOT / "oracle" / "_ref" / "tqp_predict_test"


@pytest.mark.parametrize("seed", [1, 2])
def test_predict_matches_reference(seed):
    assert BIN.exists(), "build it with `make -C oracle` (needs /root/reference at build time)"
    r = subprocess.run([str(BIN), "--seed", str(seed), "--rows", "20000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout
