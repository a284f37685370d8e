"""SQL frontend extension: ORDER BY and n-way joins over
the unmodified reference frontend (integration/tensql_sql_ext.hpp), checked
by oracle/tools/sql_ext_test.cpp against the reference executor: TPC-H Q3
written in SQL (queries/q3.sql) returns exactly what the committed plan JSON
returns; ORDER BY on one- and two-table statements equals the reference plan
plus make_sort; statements the reference accepts plan identically; errors are
the reference's SqlError. CPU only (the B200 side runs in test_dropin_gpu.py)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "tqp_sql_ext_test"


def test_sql_extension_matches_reference_executor():
    if not BIN.exists():
        pytest.skip(f"{BIN} is not built (make -C oracle, needs the reference sources)")
    r = subprocess.run([str(BIN), "--sf", "0.05"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "OK: 0 failure(s)" in r.stdout
    assert r.stdout.count("PASS") >= 13
