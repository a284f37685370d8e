"""CSV loader: tensql::parse_csv_text / load_csv
(columnar.cpp:453-527) with the parsing on the GPU.

* CPU: the device field parsers (csrc/fparse.cuh, compiled for the host) are
  held to std::from_chars and the reference's encode_date on random and edge
  fields (oracle/_ref/fparse_check).
* GPU: every golden case (tests/golden/csv.json, parsed by the unmodified
  reference in oracle/tools/csv_cases.cpp) gives the same table, bit for bit,
  or the same error text; a TPC-H lineitem CSV parses to exactly the device
  generator's columns; load_csv reads a file."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
import tqp_oracle as O

FPARSE = ROOT / "oracle" / "_ref" / "fparse_check"


def test_field_parsers_match_reference_parsers():
    if not FPARSE.exists():
        pytest.skip("oracle/_ref/fparse_check not built (needs /root/reference)")
    r = subprocess.run([str(FPARSE), "200000", "5"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 mismatch(es)" in r.stdout


def golden():
    return json.loads((GOLDEN / "csv.json").read_text())["cases"]


def test_golden_csv_fixture_shape():
    cases = golden()
    assert len(cases) > 90
    assert sum("error" in c for c in cases) > 50


def same_table(got, want):
    cols = want["columns"]
    assert [(n, t) for n, t, _ in got] == [(c["name"], c["type"]) for c in cols]
    for (name, typ, arr), c in zip(got, cols):
        w = O.tensor_from_json(c["tensor"])
        if typ == "utf8":
            dec = lambda a: [bytes(int(x) for x in r).split(b"\0", 1)[0] for r in a]
            assert arr.shape[0] == w.shape[0], name
            assert dec(arr) == dec(w), name
            assert arr.shape[1] == w.shape[1], (name, arr.shape, w.shape)  # width = longest value
        elif w.dtype == np.float64:
            g = arr.reshape(-1)
            ww = w.reshape(-1)
            nan = np.isnan(ww)
            assert np.array_equal(np.isnan(g), nan), name
            assert np.array_equal(g[~nan].view(np.uint64), ww[~nan].view(np.uint64)), name
        else:
            np.testing.assert_array_equal(arr.reshape(w.shape), w, err_msg=name)


@pytest.mark.gpu
def test_csv_golden_cases(ctx):
    from paper_2209_04579_b200 import tqp
    for c in golden():
        text = bytes.fromhex(c["text_hex"])
        schema = [tuple(x) for x in c["schema"]]
        if "error" in c:
            with pytest.raises(tqp.TqpError) as ei:
                tqp.Table.from_csv_text(text, schema, c["delimiter"], origin="t.csv")
            assert str(ei.value) == c["error"], c["name"]
            if schema:
                assert isinstance(ei.value, tqp.EncodingError), c["name"]
            continue
        t = tqp.Table.from_csv_text(text, schema, c["delimiter"], origin="t.csv")
        assert t.rows == c["result"]["rows"], c["name"]
        host = t.to_numpy()
        same_table([(n, typ, host[n]) for n, typ in t.columns()], c["result"])


def lineitem_csv(tab):
    """lineitem as CSV text the way a TPC-H dump writes it: money with two
    decimals, rates as 0.0x, dates ISO."""
    cols = tab.columns()
    host = tab.to_numpy()
    out = [",".join(n for n, _ in cols)]
    parts = []
    for n, lt in cols:
        a = host[n]
        if lt == "int64":
            parts.append(a[:, 0].astype(str))
        elif lt == "float64":
            cents = np.rint(a[:, 0] * 100).astype(np.int64)
            parts.append(np.char.add(np.char.add((cents // 100).astype(str), "."),
                                     np.char.zfill((cents % 100).astype(str), 2)))
        elif lt == "date":
            parts.append(np.datetime_as_string(a[:, 0].astype("datetime64[ns]"), unit="D"))
        else:
            parts.append(np.array([bytes(np.asarray(r).astype(np.uint8)).split(b"\0", 1)[0].decode() for r in a]))
    rows = parts[0]
    for p in parts[1:]:
        rows = np.char.add(np.char.add(rows, ","), p)
    return "\n".join(out + list(rows)) + "\n"


@pytest.mark.gpu
def test_csv_lineitem_equals_generator(ctx, tmp_path):
    from paper_2209_04579_b200 import tqp
    gen = tqp.Table.generate("lineitem", 0.02, 7)
    text = lineitem_csv(gen)
    schema = gen.columns()
    parsed = tqp.Table.from_csv_text(text, schema)
    assert parsed.rows == gen.rows
    a, b = gen.to_numpy(), parsed.to_numpy()
    for n, lt in schema:
        if lt == "float64":
            assert np.array_equal(a[n].view(np.uint64), b[n].view(np.uint64)), n
        else:
            np.testing.assert_array_equal(a[n], b[n], err_msg=n)
    f = tmp_path / "lineitem.csv"
    f.write_text(text)
    loaded = tqp.Table.load_csv(f, schema)
    c = loaded.to_numpy()
    for n, _ in schema:
        np.testing.assert_array_equal(np.asarray(a[n]).view(np.uint8), np.asarray(c[n]).view(np.uint8), err_msg=n)
    with pytest.raises(tqp.EncodingError, match="cannot open"):
        tqp.Table.load_csv(tmp_path / "missing.csv", schema)
