import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libtqp_b200.so on cuda:0)")


@pytest.fixture(scope="session")
def golden_kernels():
    return json.loads((GOLDEN / "kernels.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_plans():
    return json.loads((GOLDEN / "plans.json").read_text())["cases"]


@pytest.fixture(scope="session")
def ctx():
    from paper_2209_04579_b200 import tqp
    return tqp.default_context()


def load_tpch_golden():
    import gzip
    with gzip.open(GOLDEN / "tpch_sf0.005.json.gz", "rt") as f:
        return json.load(f)
