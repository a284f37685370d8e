"""Random-plan parity: seeded random tables and random
well-typed plans over the reference's whole plan API (scan, filter with
AND/OR/NOT/BETWEEN/LIKE/compare, project with arithmetic and CASE, inner
join with unique or duplicate keys, grouped and scalar aggregates, mixed-
direction sorts, limits), lowered by the reference's own optimize +
plan_operators and run on the reference executor and on the B200 executor
(fused and per-instruction). oracle/tools/random_plans.cpp does the work;
results must match as tables_diff_ordered (fp64 within 1e-9, row order
included) and errors by their text."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "tqp_random_plans"


# seeds 12 / 17 / 123 reach plans that once failed (a build-group unit keyed
# by a non-unique build column, a constant build predicate, group output order)
@pytest.mark.parametrize("seed,plans", [(1, 150), (12, 300), (17, 300), (123, 300)])
def test_random_plans_match_reference(seed, plans):
    if not BIN.exists():
        pytest.fail(f"{BIN} is not built (make -C oracle)")
    r = subprocess.run([str(BIN), "--seed", str(seed), "--plans", str(plans)], capture_output=True, text=True,
                       timeout=900)
    tail = "\n".join(r.stdout.splitlines()[-40:])
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout, tail


@pytest.mark.parametrize("env", [{"TQP_JIT": "1"}, {"TQP_JIT": "1", "TQP_BUILD_TILE": "1"}])
def test_random_plans_nvrtc_kernels(env):
    """The same comparison with every fused unit on NVRTC kernels, and with
    build sides through the TMA-staged build kernel."""
    import os
    if not BIN.exists():
        pytest.fail(f"{BIN} is not built (make -C oracle)")
    r = subprocess.run([str(BIN), "--seed", "17", "--plans", "120"], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, **env))
    tail = "\n".join(r.stdout.splitlines()[-40:])
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout, tail


# --profile groups (oracle/tools/random_plans.cpp): group-by over int / date /
# short-string keys with 1 .. 10 M distinct values (dense, sparse, from the
# fact or the joined dim), joins with dense, non-dense (spread keys) and
# repeated (1:N) build keys, NaN / -0.0 values, ORDER BY + LIMIT with ties.
# Every plan must match the reference AND every fused unit must stay on the
# fused path (--require-fused: an exact-path fallback counts as a failure).
@pytest.mark.parametrize("seed", [1, 4])
def test_random_group_plans_stay_fused(seed):
    if not BIN.exists():
        pytest.fail(f"{BIN} is not built (make -C oracle)")
    r = subprocess.run([str(BIN), "--profile", "groups", "--seed", str(seed), "--plans", "60", "--require-fused", "1"],
                       capture_output=True, text=True, timeout=900)
    tail = "\n".join(r.stdout.splitlines()[-40:])
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert "0 fused fallback(s), 0 failure(s)" in r.stdout, tail
