"""Drop-in proof on the GPU: the reference's SQL frontend, optimizer and
lowering (oracle/_ref, built from /root/reference by oracle/Makefile) feed the
integration adapter (integration/tensql_b200_executor.hpp), whose results must
equal tensql::Executor's on the same tables (oracle/tools/dropin_test.cpp)."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = ROOT / "oracle" / "_ref" / "tqp_dropin_test"


def test_reference_frontend_to_b200_executor():
    assert BIN.exists(), "build it with `make -C oracle` (needs /root/reference at build time)"
    r = subprocess.run([str(BIN), "--sf", "0.01", "--gpus", "2"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 18
