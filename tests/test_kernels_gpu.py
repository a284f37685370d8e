"""Parity of every CUDA kernel (through the C ABI) against the reference's own
outputs (tests/golden/kernels.json) and the numpy oracle on larger inputs."""
import numpy as np
import pytest

import tqp_oracle as O
from test_oracle import assert_tensor_equal

pytestmark = pytest.mark.gpu


def run_case(tqp, case, strings_as_str8=False):
    a = case["args"]
    raw = [O.tensor_from_json(x) for x in a["tensors"]]
    k = case["kernel"]
    if k == "substring_match" and strings_as_str8:
        t = [tqp.Tensor.from_numpy(raw[0], utf8=True)]
    else:
        t = [tqp.Tensor.from_numpy(x) for x in raw]
    if k == "compare":
        return tqp.compare(t[0], t[1], a["op"])
    if k == "arith":
        return tqp.arith(t[0], t[1], a["op"])
    if k == "logical":
        return tqp.logical(t[0], t[1], a["op"])
    if k == "not":
        return tqp.logical_not(t[0])
    if k == "select_where":
        return tqp.select_where(*t)
    if k == "prefix_sum_exclusive":
        return tqp.prefix_sum_exclusive(t[0])
    if k == "compact":
        return tqp.compact(t[0], t[1])
    if k == "argsort_stable":
        return tqp.argsort_stable(t[0])
    if k == "gather":
        return tqp.gather(t[0], t[1])
    if k == "searchsorted":
        return tqp.searchsorted(t[0], t[1], a["side"])
    if k == "expand_segments":
        return tqp.expand_segments(t[0], t[1])
    if k == "segment_starts":
        return tqp.segment_starts(t[0])
    if k == "segmented_reduce":
        return tqp.segmented_reduce(t[0], t[1], a["num"], a["op"])
    if k == "matmul":
        return tqp.matmul(t[0], t[1])
    if k == "substring_match":
        return tqp.substring_match(t[0], a["pattern"], a["anchor"])
    raise AssertionError(k)


@pytest.mark.parametrize("str8", [False, True])
def test_kernels_match_reference_golden(ctx, golden_kernels, str8):
    from paper_2209_04579_b200 import tqp
    for case in golden_kernels:
        if str8 and case["kernel"] != "substring_match":
            continue
        if "error" in case:
            with pytest.raises(tqp.KernelError) as ei:
                run_case(tqp, case, str8)
            assert str(ei.value) == case["error"], case["kernel"]
            continue
        got = run_case(tqp, case, str8).numpy()
        want = O.tensor_from_json(case["out"])
        fsum = case["kernel"] == "segmented_reduce" and case["args"]["op"] == 0
        scale = float(np.abs(O.tensor_from_json(case["args"]["tensors"][0])).sum()) if fsum else 0.0
        assert_tensor_equal(got, want, fsum, scale)


def test_radix_argsort_large(ctx):
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(5)
    for keys in (rng.integers(-1000, 1000, 1_000_003), rng.integers(-(2**62), 2**62, 300_001),
                 rng.normal(size=500_000).round(2), np.repeat(np.arange(7), 50_000)):
        got = tqp.argsort_stable(keys.reshape(-1, 1)).numpy().ravel()
        want = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(got, want)


def test_sort_perm_rows_strings_desc(ctx):
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(9)
    words = ["pear", "fig", "apple", "", "peach", "figs"]
    strs = [words[i] for i in rng.integers(0, len(words), 20_000)]
    chars = tqp.encode_string_rows(strs)
    perm = np.arange(len(strs), dtype=np.int64).reshape(-1, 1)
    for asc in (True, False):
        got = tqp.sort_perm_rows(tqp.Tensor.from_numpy(chars, utf8=True), perm, asc).numpy()
        want = O.sort_perm_rows(chars, perm, asc)
        np.testing.assert_array_equal(got, want)


def test_compact_prefix_sum_large(ctx):
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(3)
    n = 3_000_017
    vals = rng.normal(size=n)
    mask = (rng.random(n) < 0.3).astype(np.uint8)
    np.testing.assert_array_equal(tqp.compact(vals, mask).numpy().ravel(), vals[mask != 0])
    x = rng.integers(0, 100, n)
    want = np.concatenate([[0], np.cumsum(x)[:-1]])
    np.testing.assert_array_equal(tqp.prefix_sum_exclusive(x.reshape(-1, 1)).numpy().ravel(), want)


def test_segmented_reduce_long_segments(ctx):
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(11)
    n = 2_000_000
    ids = np.sort(rng.choice([0, 0, 0, 1, 3, 3, 5], n)).astype(np.int64)
    iv = rng.integers(-1000, 1000, n)
    fv = rng.normal(size=n)
    got = tqp.segmented_reduce(iv.reshape(-1, 1), ids.reshape(-1, 1), 6, "sum").numpy().ravel()
    want = np.array([iv[ids == s].sum() for s in range(6)])
    np.testing.assert_array_equal(got, want)
    got = tqp.segmented_reduce(fv.reshape(-1, 1), ids.reshape(-1, 1), 6, "sum").numpy().ravel()
    for s in range(6):
        seg = fv[ids == s]
        assert O.approx_rel(got[s], float(np.cumsum(seg)[-1]) if seg.size else 0.0, 1e-9, float(np.abs(seg).sum()))
    for op, f in (("min", np.min), ("max", np.max)):
        ids2 = np.sort(rng.integers(0, 4, n)).astype(np.int64)
        got = tqp.segmented_reduce(fv.reshape(-1, 1), ids2.reshape(-1, 1), 4, op).numpy().ravel()
        np.testing.assert_array_equal(got, [f(fv[ids2 == s]) for s in range(4)])
    # determinism: bit-identical across runs
    a = tqp.segmented_reduce(fv.reshape(-1, 1), ids.reshape(-1, 1), 6, "sum").numpy()
    b = tqp.segmented_reduce(fv.reshape(-1, 1), ids.reshape(-1, 1), 6, "sum").numpy()
    assert a.tobytes() == b.tobytes()


def test_segmented_reduce_long_int64_bounds(ctx):
    """Long int64 segments take bounded chunk sums (wrapping sum, +-max|v| x
    rows prefix bounds); where the bounds leave int64 the segment is redone
    in the ordered monoid: no false overflow, and a real one is still the
    reference's error (kernels.cpp segmented_reduce)."""
    from paper_2209_04579_b200 import tqp
    n = 2_000_000
    big = (1 << 46) - 1  # chunks stay bounded (x 64 K rows < 2^62), segments do not
    ids = np.zeros(n, dtype=np.int64)
    ids[n // 2:] = 1
    alt = np.where(np.arange(n) % 2 == 0, big, -big).astype(np.int64)
    alt[7] = 5
    got = tqp.segmented_reduce(alt.reshape(-1, 1), ids.reshape(-1, 1), 2, "sum").numpy().ravel()
    want = [int(alt[: n // 2].astype(object).sum()), int(alt[n // 2:].astype(object).sum())]
    np.testing.assert_array_equal(got, want)
    # chunks past the bound (values near 2^61): the ordered path per chunk
    huge = np.where(np.arange(n) % 2 == 0, 1 << 61, -(1 << 61)).astype(np.int64)
    got = tqp.segmented_reduce(huge.reshape(-1, 1), ids.reshape(-1, 1), 2, "sum").numpy().ravel()
    np.testing.assert_array_equal(got, [0, 0])
    # a real overflow in segment 1 only
    up = np.full(n, big, dtype=np.int64)
    up[: n // 2] = 1
    with pytest.raises(tqp.KernelError, match="overflow in segment 1"):
        tqp.segmented_reduce(up.reshape(-1, 1), ids.reshape(-1, 1), 2, "sum")


def test_string_compare_and_plumbing(ctx):
    from paper_2209_04579_b200 import tqp
    strs = ["BUILDING", "AUTOMOBILE", "", "BUILD", "BUILDINGS"]
    chars = tqp.encode_string_rows(strs)
    lit = tqp.encode_string_rows(["BUILDING"])
    for op in O.CMP:
        got = tqp.string_compare(tqp.Tensor.from_numpy(chars, utf8=True), tqp.Tensor.from_numpy(lit, utf8=True), op)
        np.testing.assert_array_equal(got.numpy(), O.string_compare(chars, lit, op))
    np.testing.assert_array_equal(tqp.cast(np.array([[0], [3]], dtype=np.int64), "bool").numpy(), [[0], [1]])
    np.testing.assert_array_equal(tqp.broadcast_rows(np.array([[2.5]]), 3).numpy(), [[2.5]] * 3)
    np.testing.assert_array_equal(tqp.last_or_zero(np.array([[4], [9]], dtype=np.int64)).numpy(), [[9]])
    np.testing.assert_array_equal(tqp.last_or_zero(np.zeros((0, 1), dtype=np.int64)).numpy(), [[0]])
    w = tqp.pad_width_like(tqp.Tensor.from_numpy(lit, utf8=True), tqp.Tensor.from_numpy(chars, utf8=True))
    assert w.cols == chars.shape[1]
    np.testing.assert_array_equal(tqp.iota(5).numpy().ravel(), np.arange(5))


def test_searchsorted_large(ctx):
    """Pivot-staged search with galloping (scan.cu k_searchsorted): sorted
    probes (the gallop path), random probes (the pivot path), duplicates,
    probes below / above every key, both sides, int64 and float64."""
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(21)
    keys = np.sort(rng.integers(-10**6, 10**6, 1_000_003))
    for probes in (np.sort(rng.integers(-2 * 10**6, 2 * 10**6, 3_000_001)),
                   rng.integers(-2 * 10**6, 2 * 10**6, 700_001),
                   np.repeat(keys[::997], 3)):
        for side in ("left", "right"):
            got = tqp.searchsorted(keys.reshape(-1, 1), probes.reshape(-1, 1), side).numpy().ravel()
            np.testing.assert_array_equal(got, np.searchsorted(keys, probes, side=side), err_msg=side)
    fk = np.sort(rng.normal(size=200_000).round(3))
    fp = rng.normal(size=300_000).round(3)
    for side in ("left", "right"):
        got = tqp.searchsorted(fk.reshape(-1, 1), fp.reshape(-1, 1), side).numpy().ravel()
        np.testing.assert_array_equal(got, np.searchsorted(fk, fp, side=side))


def test_segment_starts_one_column(ctx):
    """16-flags-per-store one-column segment starts (kernels.cu
    k_segment_starts1): byte and int64 keys, lengths off the 16 multiple."""
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(22)
    for n in (1, 15, 16, 17, 1_000_003):
        k64 = np.sort(rng.integers(0, max(1, n // 7), n))
        want = np.concatenate([[True], k64[1:] != k64[:-1]])
        np.testing.assert_array_equal(tqp.segment_starts(k64.reshape(-1, 1)).numpy().ravel().astype(bool), want)
        k8 = np.sort(rng.integers(0, 3, n)).astype(np.uint8) + ord("A")
        chars = k8.reshape(-1, 1)
        want8 = np.concatenate([[True], k8[1:] != k8[:-1]])
        got8 = tqp.segment_starts(tqp.Tensor.from_numpy(chars, utf8=True)).numpy().ravel().astype(bool)
        np.testing.assert_array_equal(got8, want8)
