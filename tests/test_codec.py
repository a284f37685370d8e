"""Compressed columnar host format (tqp_codec_encode / tqp_tensor_from_encoded,
SURVEY.md 8(f)1): the encoder picks a lossless codec per column; a numpy
decoder here (CPU) and the device decoder (GPU) must both give back the
column bit for bit."""
import numpy as np
import pytest

from conftest import ROOT  # noqa: F401  (sys.path)


def np_decode(codec, payload, dtype, rows, cols=1):
    from paper_2209_04579_b200 import tqp
    if codec.name == "raw":
        return payload.view(tqp.NP_OF[dtype]).reshape(rows, -1) if rows else payload.view(tqp.NP_OF[dtype])
    off = 8 * codec.dict_n if codec.name == "dict" else (((codec.dict_n * cols + 7) // 8) * 8 if codec.name == "rowdict" else 0)
    words = payload[off:].view(np.uint32).astype(np.uint64)
    w = codec.width
    bit = np.arange(rows, dtype=np.uint64) * np.uint64(w)
    wi = (bit >> np.uint64(5)).astype(np.int64)
    two = words[wi] | (words[wi + 1] << np.uint64(32))
    u = (two >> (bit & np.uint64(31))) & np.uint64((1 << w) - 1)
    if codec.name == "rowdict":
        d = payload[:codec.dict_n * cols].reshape(codec.dict_n, cols)
        return d[u.astype(np.int64)]
    if codec.name == "dict":
        d = payload[:off].view(np.uint64)
        return d[u.astype(np.int64)].view(np.float64).reshape(-1, 1)
    if codec.name == "for":
        v = np.uint64(codec.base & 0xFFFFFFFFFFFFFFFF) + np.uint64(codec.scale) * u
        return (v.view(np.int64) if dtype == 2 else v.astype(np.uint8)).reshape(-1, 1)
    if codec.name == "delta":
        v = np.uint64(codec.base & 0xFFFFFFFFFFFFFFFF) + np.cumsum(np.uint64(codec.scale) * u, dtype=np.uint64)
        return v.view(np.int64).reshape(-1, 1)
    return ((codec.base + u.astype(np.int64)).astype(np.float64) / np.float64(codec.scale)).reshape(-1, 1)


def cases():
    rng = np.random.default_rng(11)
    day = 86_400 * 10**9
    n = 200_003
    yield "dates", 2, (rng.integers(8035, 10561, n) * day), "for", 12
    yield "qty", 2, rng.integers(1, 51, n), "for", 6
    yield "keys", 2, rng.integers(1, 2_000_001, n), "for", 21
    yield "negative", 2, rng.integers(-(2**40), -(2**40) + 70_000, n), "for", 17
    yield "const", 2, np.full(n, -7, dtype=np.int64), "for", 1
    yield "sorted_runs", 2, np.repeat(np.arange(1, n // 4 + 2), 4)[:n], "delta", 1  # lineitem's l_orderkey
    yield "dense_seq", 2, np.arange(5, n + 5), "delta", 1
    yield "sorted_gaps", 2, np.cumsum(rng.integers(0, 4, n)) * 8 - 2**62, "delta", 2
    yield "one_row", 2, np.array([123456789], dtype=np.int64), "raw", 0  # packed would not be smaller
    yield "wide32", 2, rng.integers(0, 2**32, n), "for", 32
    yield "flags", 4, np.array([65, 78, 82], dtype=np.uint8)[rng.integers(0, 3, n)], "rowdict", 2
    yield "bytes_many", 4, (np.arange(n) % 251).astype(np.uint8), "raw", 0  # 8-bit codes would not be smaller
    yield "extremes", 2, np.array([-(2**63), 2**63 - 1, 0], dtype=np.int64), "raw", 0
    yield "discount", 3, rng.integers(0, 11, n) / 100.0, "dict", 4
    yield "price", 3, np.round(rng.uniform(900, 105000, n), 2), "dec", 24
    yield "price_neg", 3, -np.round(rng.uniform(0.01, 300, n), 2), "dec", 15
    yield "integral_f64", 3, rng.integers(-100, 100, n).astype(np.float64) * 3.0, "dict", 8
    yield "random_f64", 3, rng.standard_normal(n), "raw", 0
    zneg = np.round(rng.uniform(1, 20, n), 2)
    zneg[5] = -0.0
    yield "neg_zero_many", 3, zneg, "raw", 0  # -0.0 breaks DEC; > 256 values rule DICT out
    nan = rng.integers(0, 5, n).astype(np.float64)
    nan[7] = np.nan
    yield "nan_dict", 3, nan, "dict", 3  # DICT keeps bit patterns, NaN included
    yield "empty", 2, np.zeros(0, dtype=np.int64), "raw", 0


@pytest.mark.parametrize("name,dtype,arr,want,width", list(cases()), ids=[c[0] for c in cases()])
def test_encoder_lossless(name, dtype, arr, want, width):
    from paper_2209_04579_b200 import tqp
    arr = np.ascontiguousarray(arr, dtype=tqp.NP_OF[dtype])
    codec, payload = tqp.encode_column(arr, dtype)
    assert codec.name == want, (name, codec.name)
    if want in ("for", "dec", "dict", "delta", "rowdict"):
        assert codec.width == width, (name, codec.width)
    if want != "raw":
        assert payload.nbytes < arr.nbytes
    back = np_decode(codec, payload, dtype, len(arr))
    np.testing.assert_array_equal(back.reshape(-1).view(np.uint64 if arr.dtype.itemsize == 8 else arr.dtype),
                                  arr.view(np.uint64 if arr.dtype.itemsize == 8 else arr.dtype))


@pytest.mark.gpu
def test_device_decode_bit_identical(ctx):
    from paper_2209_04579_b200 import tqp
    for name, dtype, arr, _, _ in cases():
        arr = np.ascontiguousarray(arr, dtype=tqp.NP_OF[dtype])
        codec, payload = tqp.encode_column(arr, dtype)
        t = tqp.Tensor.from_encoded(codec, payload, dtype, len(arr), 1)
        got = t.numpy(widen_strings=False).reshape(-1)
        view = np.uint64 if arr.dtype.itemsize == 8 else arr.dtype
        np.testing.assert_array_equal(got.view(view), arr.view(view), err_msg=name)


@pytest.mark.gpu
def test_tpch_from_encoded_columns(ctx):
    """The four queries over tables uploaded in the compressed format match
    the golden results (and the columns decode to the generator's bits)."""
    import json
    from conftest import load_tpch_golden
    from test_oracle import compare_tables
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    tables = {}
    for n in ("lineitem", "orders", "customer", "part"):
        src = tqp.Table.generate(n, gold["sf"], gold["seed"])
        tab = tqp.Table.create(ctx)
        for cname, lt in src.columns():
            dev = src.column(cname)
            host = dev.numpy(widen_strings=False)
            codec, payload = tqp.encode_column(host, dev.dtype)
            t = tqp.Tensor.from_encoded(codec, payload, dev.dtype, host.shape[0], host.shape[1])
            np.testing.assert_array_equal(t.numpy(widen_strings=False), host, err_msg=f"{n}.{cname}")
            tab.add_column(cname, lt, t)
        tables[n] = tab
    for q in ("q1", "q6", "q14", "q3"):
        plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text())
        compare_tables(tqp.Executor(plan).execute(tables).to_numpy(), gold["results"][q])


def test_row_dictionary_multibyte():
    """ROWDICT over multi-byte string rows (p_type / c_mktsegment shaped):
    <= 256 distinct rows -> dictionary + codes; more -> RAW."""
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(5)
    words = [w.encode() for w in ("STANDARD", "SMALL", "MEDIUM", "LARGE", "ECONOMY", "PROMO")]
    rows = np.zeros((100_000, 25), dtype=np.uint8)
    pick = rng.integers(0, len(words), (rows.shape[0], 3))
    for i in range(rows.shape[0]):
        s = b" ".join(words[j] for j in pick[i])[:25]
        rows[i, :len(s)] = np.frombuffer(s, dtype=np.uint8)
    codec, payload = tqp.encode_column(rows, tqp.STR8)
    assert codec.name == "rowdict" and codec.dict_n <= 216
    np.testing.assert_array_equal(np_decode(codec, payload, tqp.STR8, rows.shape[0], 25), rows)
    noisy = rng.integers(0, 256, (5000, 10)).astype(np.uint8)
    codec, payload = tqp.encode_column(noisy, tqp.STR8)
    assert codec.name == "raw"
    np.testing.assert_array_equal(payload.reshape(noisy.shape), noisy)


@pytest.mark.gpu
def test_row_dictionary_device(ctx):
    from paper_2209_04579_b200 import tqp
    rng = np.random.default_rng(6)
    rows = np.array([list(b"BUILDING\0\0"), list(b"MACHINERY\0"), list(b"AUTOMOBILE")], dtype=np.uint8)[
        rng.integers(0, 3, 70_001)]
    codec, payload = tqp.encode_column(rows, tqp.STR8)
    assert codec.name == "rowdict"
    t = tqp.Tensor.from_encoded(codec, payload, tqp.STR8, rows.shape[0], rows.shape[1])
    np.testing.assert_array_equal(t.numpy(widen_strings=False), rows)


def test_codec_argument_errors():
    """Bad shapes, a too-small output buffer and a mismatched payload fail
    with a status instead of writing out of bounds."""
    from paper_2209_04579_b200 import tqp
    import ctypes as C
    a = np.arange(1000, dtype=np.int64)
    out = np.empty(16, dtype=np.uint8)
    codec, st = tqp.Codec(), tqp.Status()
    n = tqp.lib.tqp_codec_encode(tqp.I64, 1000, 1, a.ctypes.data, out.ctypes.data, out.nbytes, C.byref(codec),
                                 C.byref(st))
    assert n == -1 and st.code != 0  # RAW would need 8000 bytes; packed codes need more than 16
    n = tqp.lib.tqp_codec_encode(tqp.I64, -1, 1, a.ctypes.data, out.ctypes.data, out.nbytes, C.byref(codec),
                                 C.byref(st))
    assert n == -1 and b"shape" in st.msg
    assert tqp.lib.tqp_codec_bound(tqp.I64, 10, 0) == -1


@pytest.mark.gpu
def test_async_encoded_upload_pipeline(ctx):
    """sync=False uploads (copy stream + decode stream, the context stream
    waiting at first use): tables uploaded while the previous set's queries
    are queued give the golden results, kernels called straight on a
    still-decoding tensor see the decoded values, and tensors dropped before
    any use free cleanly (DevBuf waits for the decode)."""
    import json
    import torch
    from conftest import load_tpch_golden
    from test_oracle import compare_tables
    from paper_2209_04579_b200 import tqp
    gold = load_tpch_golden()
    host = {}
    for n in ("lineitem", "orders", "customer", "part"):
        src = tqp.Table.generate(n, gold["sf"], gold["seed"])
        cols = []
        for cname, lt in src.columns():
            dev = src.column(cname)
            arr = dev.numpy(widen_strings=False)
            codec, payload = tqp.encode_column(arr, dev.dtype)
            cols.append((cname, lt, dev.dtype, arr, codec, torch.from_numpy(payload).pin_memory()))
        host[n] = cols

    def upload():
        out = {}
        for n, cols in host.items():
            tab = tqp.Table.create(ctx)
            for cname, lt, dt, arr, codec, pin in cols:
                tab.add_column(cname, lt, tqp.Tensor.from_encoded(codec, pin, dt, arr.shape[0], arr.shape[1],
                                                                   ctx=ctx, sync=False))
            out[n] = tab
        return out

    plans = {q: json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text())
             for q in ("q1", "q6", "q14", "q3")}
    execs = {q: tqp.Executor(p, ctx=ctx) for q, p in plans.items()}
    tabs = upload()
    for step in range(3):
        nxt = upload()  # issued before this step's queries
        for q, ex in execs.items():
            compare_tables(ex.execute(tabs).to_numpy(), gold["results"][q])
        tabs = nxt
    # a kernel on a tensor whose decode may still be running
    cname, lt, dt, arr, codec, pin = host["lineitem"][0]
    for _ in range(4):
        t = tqp.Tensor.from_encoded(codec, pin, dt, arr.shape[0], arr.shape[1], ctx=ctx, sync=False)
        np.testing.assert_array_equal(tqp.compare(t, t, "eq", ctx=ctx).numpy().reshape(-1), np.ones(arr.shape[0], bool))
    # dropped unused
    for _ in range(8):
        tqp.Tensor.from_encoded(codec, pin, dt, arr.shape[0], arr.shape[1], ctx=ctx, sync=False)
    ctx.sync()
