"""CPU oracle: a numpy restatement of the reference's kernel set, plumbing ops
and executor (tensql, /root/reference/proj). TEST INFRASTRUCTURE ONLY — only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker. The product path
(paper_2209_04579_b200/) never imports it.

Pinning: tests/test_oracle.py checks every function here against
tests/golden/{kernels,plans}.json, which oracle/tools/golden_cases.cpp
produced by running the UNMODIFIED reference library (built from
/root/reference/proj/src by oracle/Makefile) on the same inputs.

Tensors are numpy 2-D arrays (rows, cols) with the reference dtypes:
uint8 (Bool), int32 (Int32 / Utf8 bytes), int64, float64.
"""
from __future__ import annotations

import json
from typing import Dict, List, Mapping, Optional, Sequence, Tuple

import numpy as np

INT64_MIN, INT64_MAX = -(1 << 63), (1 << 63) - 1
DT = {"bool": np.uint8, "int32": np.int32, "int64": np.int64, "float64": np.float64}
DT_NAME = {np.dtype(np.uint8): "bool", np.dtype(np.int32): "int32", np.dtype(np.int64): "int64",
           np.dtype(np.float64): "float64"}
CMP = ["eq", "ne", "lt", "le", "gt", "ge"]
ARITH = ["add", "sub", "mul", "div"]
PHYS = {"int64": np.int64, "float64": np.float64, "date": np.int64, "utf8": np.int32, "bool": np.uint8}


class KernelError(RuntimeError):
    """tensql::KernelError (tensor.hpp:20-23)."""


class ExecError(RuntimeError):
    """tensql::ExecError (interpreter.hpp:11-14)."""


class EncodingError(RuntimeError):
    """tensql::EncodingError (columnar.hpp:23-26)."""


def _name(a: np.ndarray) -> str:
    return DT_NAME[a.dtype]


def _shape(a) -> str:
    return f"{a.shape[0]}x{a.shape[1]}"


def tensor_from_json(j: Mapping) -> np.ndarray:
    """oracle/tools/dump.hpp tensor_to_json inverse."""
    data = [float(v) if isinstance(v, str) else v for v in j["data"]]
    return np.array(data, dtype=DT[j["dtype"]]).reshape(j["rows"], j["cols"])


# ---- broadcasting (kernels.cpp:46-106) ----------------------------------------
def _bcastable(s, rows, cols):
    if s.shape == (rows, cols):
        return True
    return s.shape[0] == 1 and (s.shape[1] == 1 or s.shape[1] == cols)


def _broadcast(kernel, a, b):
    """broadcast_shape (kernels.cpp:59-82) -> operands expanded to the shape."""
    if a.shape == b.shape or _bcastable(b, *a.shape):
        rows, cols = a.shape
    elif _bcastable(a, *b.shape):
        rows, cols = b.shape
    else:
        raise KernelError(f"{kernel}: shape mismatch ({_shape(a)} vs {_shape(b)})")

    def expand(t):
        scalar = t.shape == (1, 1) and (rows, cols) != (1, 1)
        row = t.shape != (1, 1) and t.shape[0] == 1 and rows > 1 and t.shape[1] == cols
        if not scalar and not row and t.shape != (rows, cols):
            raise KernelError(f"{kernel}: shape mismatch")
        return np.broadcast_to(t.reshape(1, -1) if row else t, (rows, cols))

    return expand(a), expand(b), rows, cols


def _same_dtype(kernel, a, b):
    if a.dtype != b.dtype:
        raise KernelError(f"{kernel}: dtype mismatch ({_name(a)} vs {_name(b)})")


def _require_dtype(kernel, t, want):
    if t.dtype != np.dtype(DT[want]):
        raise KernelError(f"{kernel}: expected {want}, got {_name(t)}")


def _require_vector(kernel, t):
    if t.shape[1] != 1:
        raise KernelError(f"{kernel}: expected a vector (m=1)")


# ---- kernels -----------------------------------------------------------------
def compare(a, b, op: str):
    """kernels.cpp:190-209."""
    _same_dtype("compare", a, b)
    x, y, _, _ = _broadcast("compare", a, b)
    f = {"eq": np.equal, "ne": np.not_equal, "lt": np.less, "le": np.less_equal, "gt": np.greater,
         "ge": np.greater_equal}[op]
    return f(x, y).astype(np.uint8)


def arith(a, b, op: str):
    """kernels.cpp:211-283 (checked integer ops, fp64 div-by-zero)."""
    _same_dtype("arith", a, b)
    if a.dtype == np.uint8:
        raise KernelError("arith: bool operands not supported")
    if op == "div" and a.dtype != np.float64:
        raise KernelError("arith: div requires float64 operands")
    x, y, rows, cols = _broadcast("arith", a, b)
    if a.dtype == np.float64:
        with np.errstate(all="ignore"):
            if op == "div":
                zero = np.flatnonzero((y == 0.0).ravel())
                if zero.size:
                    raise KernelError(f"arith: division by zero at row {zero[0] // cols}")
                return x / y
            return {"add": np.add, "sub": np.subtract, "mul": np.multiply}[op](x, y)
    # exact integer arithmetic through Python ints / object arrays
    lo, hi = (INT64_MIN, INT64_MAX) if a.dtype == np.int64 else (-(1 << 31), (1 << 31) - 1)
    xo, yo = x.astype(object), y.astype(object)
    r = {"add": lambda p, q: p + q, "sub": lambda p, q: p - q, "mul": lambda p, q: p * q}[op](xo, yo)
    flat = r.ravel()
    for i, v in enumerate(flat):
        if v < lo or v > hi:
            raise KernelError(f"arith: integer overflow at row {i // cols}")
    return r.astype(a.dtype)


def logical(a, b, op: str):
    """kernels.cpp:285-296."""
    _require_dtype("logical", a, "bool")
    _require_dtype("logical", b, "bool")
    x, y, _, _ = _broadcast("logical", a, b)
    return ((x != 0) & (y != 0) if op == "and" else (x != 0) | (y != 0)).astype(np.uint8)


def logical_not(v):
    """kernels.cpp:298-308."""
    _require_dtype("not", v, "bool")
    return (v == 0).astype(np.uint8)


def select_where(cond, a, b):
    """kernels.cpp:310-347 (full 2-D broadcasting)."""
    _require_dtype("select_where", cond, "bool")
    _same_dtype("select_where", a, b)
    rows = max(cond.shape[0], a.shape[0], b.shape[0])
    cols = max(cond.shape[1], a.shape[1], b.shape[1])
    for x in (cond, a, b):
        if (x.shape[0] not in (1, rows)) or (x.shape[1] not in (1, cols)):
            raise KernelError(f"select_where: shape {_shape(x)} does not broadcast to {rows}x{cols}")
    c = np.broadcast_to(cond, (rows, cols)) != 0
    return np.where(c, np.broadcast_to(a, (rows, cols)), np.broadcast_to(b, (rows, cols))).astype(a.dtype)


def prefix_sum_exclusive(x):
    """kernels.cpp:349-362 (sequential, overflow-checked)."""
    _require_vector("prefix_sum_exclusive", x)
    _require_dtype("prefix_sum_exclusive", x, "int64")
    v = x.ravel().astype(object)
    out = np.zeros(len(v), dtype=np.int64)
    acc = 0
    for i, e in enumerate(v):
        out[i] = acc
        acc += e
        if acc < INT64_MIN or acc > INT64_MAX:
            raise KernelError(f"prefix_sum_exclusive: overflow at row {i}")
    return out.reshape(-1, 1)


def compact(values, mask):
    """kernels.cpp:364-409: rows where mask, order preserved."""
    _require_dtype("compact", mask, "bool")
    _require_vector("compact", mask)
    if mask.shape[0] != values.shape[0]:
        raise KernelError(f"compact: mask length {mask.shape[0]} does not match rows {values.shape[0]}")
    return values[mask.ravel() != 0].reshape(-1, values.shape[1])


def _sort_key(v):
    # stable_sort with `<`: -0.0 == 0.0 compare equal (kernels.cpp:419-421)
    if v.dtype == np.float64:
        return np.where(v == 0.0, 0.0, v)
    return v


def argsort_stable(keys):
    """kernels.cpp:411-424."""
    _require_vector("argsort_stable", keys)
    k = keys.ravel()
    if k.dtype == np.float64 and np.isnan(k).any():
        raise KernelError("argsort_stable: NaN in keys")
    return np.argsort(_sort_key(k), kind="stable").astype(np.int64).reshape(-1, 1)


def gather(values, idx):
    """kernels.cpp:426-455."""
    _require_dtype("gather", idx, "int64")
    _require_vector("gather", idx)
    n = values.shape[0]
    iv = idx.ravel()
    bad = np.flatnonzero((iv < 0) | (iv >= n))
    if bad.size:
        p = int(bad[0])
        raise KernelError(f"gather: index {iv[p]} at position {p} out of bounds [0,{n})")
    return values[iv].reshape(len(iv), values.shape[1])


def searchsorted(sorted_, probes, side: str):
    """kernels.cpp:457-484."""
    _same_dtype("searchsorted", sorted_, probes)
    _require_vector("searchsorted", sorted_)
    _require_vector("searchsorted", probes)
    s, p = sorted_.ravel(), probes.ravel()
    if s.dtype == np.float64 and (np.isnan(s).any() or np.isnan(p).any()):
        raise KernelError("searchsorted: NaN in keys")
    dec = np.flatnonzero(s[1:] < s[:-1])
    if dec.size:
        raise KernelError(f"searchsorted: input not non-decreasing at row {dec[0] + 1}")
    return np.searchsorted(s, p, side=side).astype(np.int64).reshape(-1, 1)


def expand_segments(starts, counts):
    """kernels.cpp:486-516."""
    for t in (starts, counts):
        _require_dtype("expand_segments", t, "int64")
    for t in (starts, counts):
        _require_vector("expand_segments", t)
    if starts.shape[0] != counts.shape[0]:
        raise KernelError("expand_segments: starts/counts length mismatch")
    c = counts.ravel()
    neg = np.flatnonzero(c < 0)
    if neg.size:
        raise KernelError(f"expand_segments: negative count at row {neg[0]}")
    parts = [np.arange(s, s + k, dtype=np.int64) for s, k in zip(starts.ravel(), c)]
    out = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    return out.reshape(-1, 1)


def segment_starts(sorted_keys):
    """kernels.cpp:518-543 (full-width row comparison)."""
    n = sorted_keys.shape[0]
    out = np.zeros((n, 1), dtype=np.uint8)
    if n:
        out[0] = 1
        out[1:, 0] = (sorted_keys[1:] != sorted_keys[:-1]).any(axis=1)
    return out


def _segment_runs(ids, num):
    """segment_runs (kernels.cpp:552-580)."""
    v = ids.ravel()
    prev = -1
    for i, s in enumerate(v):
        if s < prev:
            raise KernelError(f"segmented_reduce: segment_ids decrease at row {i}")
        if s < 0 or s >= num:
            raise KernelError(f"segmented_reduce: segment id {s} out of range [0,{num}) at row {i}")
        prev = s
    lo = np.searchsorted(v, np.arange(num), side="left")
    hi = np.searchsorted(v, np.arange(num), side="right")
    return lo, hi


def segmented_reduce(values, ids, num: int, op: str):
    """kernels.cpp:584-672. Float64 SUM follows the `ref` backend's
    sequential order (backend.cpp:18-22; np.cumsum accumulates in order)."""
    _require_vector("segmented_reduce", values)
    _require_dtype("segmented_reduce", ids, "int64")
    _require_vector("segmented_reduce", ids)
    if values.shape[0] != ids.shape[0]:
        raise KernelError("segmented_reduce: values/segment_ids length mismatch")
    if num < 0:
        raise KernelError("segmented_reduce: negative segment count")
    lo, hi = _segment_runs(ids, num)
    if op == "count":
        return (hi - lo).astype(np.int64).reshape(-1, 1)
    if values.dtype == np.uint8:
        raise KernelError("segmented_reduce: bool values not supported")
    v = values.ravel()
    if op in ("min", "max"):
        for s in range(num):
            if lo[s] == hi[s]:
                raise KernelError(f"segmented_reduce: empty segment {s} for {op}")
        out = np.empty(num, dtype=values.dtype)
        for s in range(num):
            seg = v[lo[s]:hi[s]]
            acc = seg[0]
            for x in seg[1:]:
                if values.dtype == np.float64 and (np.isnan(x) or np.isnan(acc)):
                    acc = np.nan
                    continue
                acc = (x if x < acc else acc) if op == "min" else (x if x > acc else acc)
            out[s] = acc
        return out.reshape(-1, 1)
    if values.dtype == np.float64:
        out = np.zeros(num, dtype=np.float64)
        for s in range(num):
            if hi[s] > lo[s]:
                out[s] = np.cumsum(v[lo[s]:hi[s]])[-1]
        return out.reshape(-1, 1)
    lim = (INT64_MIN, INT64_MAX) if values.dtype == np.int64 else (-(1 << 31), (1 << 31) - 1)
    out = np.zeros(num, dtype=values.dtype)
    for s in range(num):
        acc = 0
        for x in v[lo[s]:hi[s]].tolist():
            acc += x
            if acc < lim[0] or acc > lim[1]:
                raise KernelError(f"segmented_reduce: sum overflow in segment {s}")
        out[s] = acc
    return out.reshape(-1, 1)


def matmul(a, b):
    """kernels.cpp:674-690."""
    _require_dtype("matmul", a, "float64")
    _require_dtype("matmul", b, "float64")
    if a.shape[1] != b.shape[0]:
        raise KernelError(f"matmul: inner dimensions differ ({a.shape[1]} vs {b.shape[0]})")
    return a @ b


def substring_match(chars, pattern: str, anchor: str):
    """kernels.cpp:692-728 over zero-padded byte rows."""
    _require_dtype("substring_match", chars, "int32")
    pat = list(pattern.encode("utf-8"))
    pl = len(pat)
    out = np.zeros((chars.shape[0], 1), dtype=np.uint8)
    for i, row in enumerate(chars):
        r = row.tolist()
        ln = 0
        while ln < len(r) and r[ln] != 0:
            ln += 1
        s = r[:ln]
        ok = False
        if pl <= ln:
            if anchor == "start":
                ok = s[:pl] == pat
            elif anchor == "end":
                ok = s[ln - pl:] == pat
            elif anchor == "any":
                ok = any(s[o:o + pl] == pat for o in range(ln - pl + 1))
            else:
                ok = ln == pl and s == pat
        out[i] = ok
    return out


# ---- plumbing ops (executor.cpp:25-278) ---------------------------------------
def string_compare(a, b, op: str):
    """string_compare_rows (executor.cpp:72-108): narrower side zero-extended."""
    rows = max(a.shape[0], b.shape[0])
    m = max(a.shape[1], b.shape[1])
    A = np.zeros((a.shape[0], m), dtype=np.int64)
    B = np.zeros((b.shape[0], m), dtype=np.int64)
    A[:, :a.shape[1]] = a
    B[:, :b.shape[1]] = b
    A = np.broadcast_to(A, (rows, m))
    B = np.broadcast_to(B, (rows, m))
    out = np.zeros((rows, 1), dtype=np.uint8)
    for i in range(rows):
        x, y = A[i].tolist(), B[i].tolist()
        c = (x > y) - (x < y)
        out[i] = {"eq": c == 0, "ne": c != 0, "lt": c < 0, "le": c <= 0, "gt": c > 0, "ge": c >= 0}[op]
    return out


def sort_perm_rows(key, perm, asc: bool):
    """sort_perm_rows (executor.cpp:44-68): one stable pass per byte column,
    last first; descending = reverse, stable argsort, flip."""
    p = perm
    for j in range(key.shape[1] - 1, -1, -1):
        col = key[:, j:j + 1]
        k = gather(col, p)
        if asc:
            p2 = argsort_stable(k)
        else:
            n = k.shape[0]
            ps = argsort_stable(k[::-1].copy()).ravel()
            p2 = (n - 1 - ps[::-1]).reshape(-1, 1)
        p = gather(p, p2)
    return p


def cast(t, to: str):
    """cast_tensor (executor.cpp:113-146)."""
    if _name(t) == to:
        return t
    if to == "bool":
        return (t != 0).astype(np.uint8)
    return t.astype(DT[to])


def pad_width_like(t, like):
    """PadWidthLike (executor.cpp:262-273)."""
    target = max(t.shape[1], like.shape[1])
    if t.shape[1] == target:
        return t
    out = np.zeros((t.shape[0], target), dtype=t.dtype)
    out[:, :t.shape[1]] = t
    return out


# ---- executor over a lowered OperatorPlan (executor.cpp:314-429) ----------------
def _instr(ins, slot, tables):
    op = ins["op"]
    a = lambda i: slot(ins["inputs"][i])  # noqa: E731
    if op == "compare":
        return compare(a(0), a(1), ins["cmp"])
    if op == "arith":
        return arith(a(0), a(1), ins["arith"])
    if op == "logical":
        return logical(a(0), a(1), ins["logic"])
    if op == "not":
        return logical_not(a(0))
    if op == "select_where":
        return select_where(a(0), a(1), a(2))
    if op == "prefix_sum_exclusive":
        return prefix_sum_exclusive(a(0))
    if op == "compact":
        return compact(a(0), a(1))
    if op == "argsort_stable":
        return argsort_stable(a(0))
    if op == "gather":
        return gather(a(0), a(1))
    if op == "searchsorted":
        return searchsorted(a(0), a(1), ins["side"])
    if op == "expand_segments":
        return expand_segments(a(0), a(1))
    if op == "segment_starts":
        return segment_starts(a(0))
    if op == "segmented_reduce":
        num = ins["param"]
        if num < 0:
            num = max(0, int(a(2).ravel()[0]))
        return segmented_reduce(a(0), a(1), num, ins["reduce"])
    if op == "matmul":
        return matmul(a(0), a(1))
    if op == "substring_match":
        return substring_match(a(0), ins["pattern"], ins["anchor"])
    if op == "load_column":
        t = None
        for name, tab in tables.items():
            if name.lower() == ins["table"].lower():
                t = tab
        if t is None:
            raise ExecError(f"no input table named '{ins['table']}'")
        for cname, (_, arr) in t.items():
            if cname.lower() == ins["column"].lower():
                return arr
        raise EncodingError(f"table: no column named '{ins['column']}'")
    if op == "const":
        return tensor_from_json(ins["constant"])
    if op == "iota_rows":
        n = a(0).shape[0]
        if ins["param"] >= 0:
            n = min(n, ins["param"])
        return np.arange(n, dtype=np.int64).reshape(-1, 1)
    if op == "iota_len":
        n = int(a(0).ravel()[0])
        if n < 0:
            raise ExecError("iota: negative length")
        return np.arange(n, dtype=np.int64).reshape(-1, 1)
    if op == "cast":
        return cast(a(0), ins["cast_to"])
    if op == "exp":
        return np.exp(a(0))
    if op == "last_or_zero":
        v = a(0).ravel()
        return np.array([[v[-1] if v.size else 0]], dtype=np.int64)
    if op == "pack_cols":
        return np.hstack([a(i) for i in range(len(ins["inputs"]))])
    if op == "broadcast_scalar":
        v = a(0)
        if v.shape[0] != 1:
            raise ExecError("broadcast: value must have one row")
        return np.repeat(v, a(1).shape[0], axis=0)
    if op == "pad_width_like":
        return pad_width_like(a(0), a(1))
    if op == "sort_perm_rows":
        return sort_perm_rows(a(0), a(1), ins["param"] == 1)
    if op == "string_compare":
        return string_compare(a(0), a(1), ins["cmp"])
    raise ExecError("unknown instruction")


TableSet = Mapping[str, Mapping[str, Tuple[str, np.ndarray]]]  # table -> col -> (logical, array)


def execute(opplan: Mapping, tables: TableSet) -> List[Tuple[str, str, np.ndarray]]:
    """Executor::run (executor.cpp:354-429) over numpy tensors."""
    for it in opplan["input_tables"]:
        t = next((tab for name, tab in tables.items() if name.lower() == it["name"].lower()), None)
        if t is None:
            raise ExecError(f"no input table named '{it['name']}'")
        for c in it["schema"]:
            col = next((v for k, v in t.items() if k.lower() == c["name"].lower()), None)
            if col is None:
                raise ExecError(f"input table '{it['name']}' is missing column '{c['name']}'")
            if col[0] != c["type"]:
                raise ExecError(f"input table '{it['name']}': column '{c['name']}' is {col[0]}, "
                                f"the plan expects {c['type']}")
    slots: Dict[int, np.ndarray] = {}
    for step in opplan["steps"]:
        for ins in step["instrs"]:
            try:
                slots[ins["output"]] = _instr(ins, lambda s: slots[s], tables)
            except (KernelError, EncodingError) as e:
                raise ExecError(f"{step['id']}: {e}") from None
    return [(o["name"], o["type"], slots[o["slot"]]) for o in opplan["outputs"]]


def tables_from_json(tj: Mapping) -> Dict[str, Dict[str, Tuple[str, np.ndarray]]]:
    """oracle/tools/dump.hpp table_to_json inverse."""
    out = {}
    for name, t in tj.items():
        out[name] = {c["name"]: (c["type"], tensor_from_json(c["tensor"])) for c in t["columns"]}
    return out


def approx_rel(a: float, b: float, tol: float = 1e-9, scale: float = 0.0) -> bool:
    """tests/support/test_util.hpp:62-68."""
    m = max(1.0, abs(a), abs(b), scale)
    return abs(a - b) <= tol * m
