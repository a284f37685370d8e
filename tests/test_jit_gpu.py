"""Run-time specialised pipeline kernels (csrc/jit.cu, NVRTC): the generated
straight-line kernel must reproduce the generic k_tile bit for bit (same
operation order, same per-thread row partition, same reduction trees), and
match the reference's golden results."""
import json
import os

import numpy as np
import pytest

import tqp_oracle as O
from conftest import ROOT, load_tpch_golden
from test_oracle import compare_tables

pytestmark = pytest.mark.gpu
PLANS = ROOT / "paper_2209_04579_b200" / "plans"
QUERIES = ("q1", "q6", "q14", "q3")


def run(tqp, q, tables, jit, wide=False, regacc=True):
    old = os.environ.get("TQP_JIT")
    old_w = os.environ.get("TQP_SMALL_WIDE")
    old_r = os.environ.get("TQP_SMALL_REG")
    os.environ["TQP_JIT"] = "1" if jit else "0"
    os.environ["TQP_SMALL_WIDE"] = "1" if wide else "0"
    os.environ["TQP_SMALL_REG"] = "1" if regacc else "0"
    try:
        ex = tqp.Executor(json.loads((PLANS / f"{q}.opplan.json").read_text()))
        ex.set_timing(True)
        res = ex.execute(tables).to_numpy()
        kernels = [k for k in ex.timings() if k.startswith("kernel:")]
        return res, kernels
    finally:
        if old is None:
            del os.environ["TQP_JIT"]
        else:
            os.environ["TQP_JIT"] = old
        if old_w is None:
            del os.environ["TQP_SMALL_WIDE"]
        else:
            os.environ["TQP_SMALL_WIDE"] = old_w
        if old_r is None:
            del os.environ["TQP_SMALL_REG"]
        else:
            os.environ["TQP_SMALL_REG"] = old_r


@pytest.mark.parametrize("q", QUERIES)
def test_jit_bit_identical_to_generic(ctx, q):
    from paper_2209_04579_b200 import tqp
    tables = {n: tqp.Table.generate(n, 0.05, 7) for n in ("lineitem", "orders", "customer", "part")}
    got, kj = run(tqp, q, tables, True)
    want, kg = run(tqp, q, tables, False)
    assert any(k.startswith("kernel:q_tile") for k in kj), kj
    assert not any(k.startswith("kernel:q_tile") for k in kg), kg
    if q in ("q14", "q3"):  # build sides specialised too
        assert any(k.startswith("kernel:q_build") for k in kj), kj
        assert any(k.startswith("kernel:k_build") for k in kg), kg
    assert [(n, t) for n, t, _ in got] == [(n, t) for n, t, _ in want]
    for (n, _, g), (_, _, w) in zip(got, want):
        np.testing.assert_array_equal(g.view(np.uint8), w.view(np.uint8), err_msg=f"{q}.{n}")


def test_jit_matches_reference_golden(ctx):
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    tables = {name: tqp.Table.from_columns([(c, typ, arr) for c, (typ, arr) in t.items()])
              for name, t in O.tables_from_json(gold["tables"]).items()}
    for q in QUERIES:
        got, _ = run(tqp, q, tables, True)
        compare_tables(got, gold["results"][q])


def test_jit_golden_plans(ctx, golden_plans):
    """Every golden plan (string predicates, LIKE anchors, joins, CASE, zero
    rows, error text) with every fused unit forced onto NVRTC kernels."""
    from paper_2209_04579_b200 import tqp
    from test_executor_gpu import as_numpy, device_tables
    old = os.environ.get("TQP_JIT")
    os.environ["TQP_JIT"] = "1"
    try:
        for case in golden_plans:
            tables = device_tables(tqp, case["tables"])
            ex = tqp.Executor(case["opplan"], fuse=True)
            if "error" in case:
                with pytest.raises(tqp.ExecError) as ei:
                    ex.execute(tables)
                assert str(ei.value) == case["error"], case["name"]
                continue
            compare_tables(as_numpy(ex.execute(tables)), case["result"])
    finally:
        if old is None:
            del os.environ["TQP_JIT"]
        else:
            os.environ["TQP_JIT"] = old


def _q1_close(got, want):
    assert [(n, t) for n, t, _ in got] == [(n, t) for n, t, _ in want]
    for (n, t, g), (_, _, w) in zip(got, want):
        np.testing.assert_array_equal(g.view(np.uint8), w.view(np.uint8), err_msg=n)


def _q1_within(got, want, rtol=1e-12):
    """Keys, integer sums and counts bit for bit; fp64 sums within rtol (a
    different row-to-thread split changes the fp64 association only)."""
    assert [(n, t) for n, t, _ in got] == [(n, t) for n, t, _ in want]
    for (n, t, g), (_, _, w) in zip(got, want):
        if g.dtype == np.float64:
            np.testing.assert_allclose(g, w, rtol=rtol, atol=0, err_msg=n)
        else:
            np.testing.assert_array_equal(g, w, err_msg=n)


def test_small_group_wide_kernel(ctx):
    """The 4-slot small-group kernels (the default for large Q1-shaped scans)
    against the 8-slot generic kernel: the shared-memory-cell variant is
    bit-identical (same tile shape, same per-thread row order); the register
    variant (taller tiles, more warps) matches within 1e-12 and is
    deterministic; with six keys per CTA both flag the overflow and the unit
    reruns on the 8-slot kernel."""
    from paper_2209_04579_b200 import tqp
    tables = {"lineitem": tqp.Table.generate("lineitem", 0.05, 7)}
    cells, kc = run(tqp, "q1", tables, True, wide=True, regacc=False)
    wide, kw = run(tqp, "q1", tables, True, wide=True)
    again, _ = run(tqp, "q1", tables, True, wide=True)
    generic, _ = run(tqp, "q1", tables, False)
    assert any(k.startswith("kernel:q_tile") for k in kw)
    assert any(k.startswith("kernel:q_tile") for k in kc)
    _q1_close(cells, generic)
    _q1_close(wide, again)
    _q1_within(wide, generic)
    # six (returnflag, linestatus) keys: more than the wide kernel's 4 slots
    host = tables["lineitem"].to_numpy()
    rng = np.random.default_rng(3)
    flags = np.array([ord(c) for c in "ABC"], dtype=np.int32)[rng.integers(0, 3, host["l_returnflag"].shape[0])]
    cols = []
    for name, lt in tables["lineitem"].columns():
        a = host[name]
        if name == "l_returnflag":
            a = flags.reshape(-1, 1).astype(a.dtype)
        cols.append((name, lt, a))
    six = {"lineitem": tqp.Table.from_columns(cols)}
    wide6, kw6 = run(tqp, "q1", six, True, wide=True)
    cells6, _ = run(tqp, "q1", six, True, wide=True, regacc=False)
    generic6, _ = run(tqp, "q1", six, False)
    assert len(wide6[0][2]) == 6
    assert any(k.startswith("kernel:q_tile") for k in kw6)
    _q1_close(wide6, generic6)
    _q1_close(cells6, generic6)
