"""Host-side mirror of the reference's execution API over the C ABI.

The reference (tensql, C++) exposes the kernel set as free functions
(include/tensql/kernels.hpp:28-78), device-free value carriers (Tensor,
tensor.hpp:49-122; EncodedTable, columnar.hpp:41-54) and an Executor over a
lowered OperatorPlan (executor.hpp:43-59). This module binds
libtqp_b200.so (include/tqp_b200.h) with ctypes and keeps those names,
argument meanings and error classes, so tests read like the reference's own.

There is no CPU fallback: importing this module without the built library
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path
from typing import Dict, Iterable, List, Mapping, Optional, Sequence, Tuple, Union

import numpy as np

_PKG = Path(__file__).resolve().parent
_LIB_PATH = Path(os.environ.get("TQP_B200_LIB", _PKG / "libtqp_b200.so"))

# ---- enums (values mirror kernels.hpp:11-16, tensor.hpp:13, columnar.hpp:13)
BOOL, I32, I64, F64, STR8 = 0, 1, 2, 3, 4
DTYPE_NAMES = {"bool": BOOL, "int32": I32, "int64": I64, "float64": F64}
NP_OF = {BOOL: np.uint8, I32: np.int32, I64: np.int64, F64: np.float64, STR8: np.uint8}
LT_INT64, LT_FLOAT64, LT_DATE, LT_UTF8, LT_BOOL = 0, 1, 2, 3, 4
LOGICAL_NAMES = {"int64": LT_INT64, "float64": LT_FLOAT64, "date": LT_DATE, "utf8": LT_UTF8, "bool": LT_BOOL}
LOGICAL_BY_ID = {v: k for k, v in LOGICAL_NAMES.items()}
COMPARE = {"eq": 0, "ne": 1, "lt": 2, "le": 3, "gt": 4, "ge": 5}
ARITH = {"add": 0, "sub": 1, "mul": 2, "div": 3}
LOGICAL = {"and": 0, "or": 1}
SIDE = {"left": 0, "right": 1}
REDUCE = {"sum": 0, "count": 1, "min": 2, "max": 3}
ANCHOR = {"start": 0, "end": 1, "any": 2, "exact": 3}

EXEC_FUSE, EXEC_NO_FUSE = 1, 0


class TqpError(RuntimeError):
    """Base of the mapped error classes; .bad_row is the first offending row."""

    def __init__(self, msg: str, bad_row: int = -1):
        super().__init__(msg)
        self.bad_row = bad_row


class KernelError(TqpError):
    """tensql::KernelError (tensor.hpp:20-23)."""


class ExecError(TqpError):
    """tensql::ExecError (interpreter.hpp:11-14)."""


class PlanError(TqpError):
    """tensql::PlanError (expr.hpp:14-17)."""


class EncodingError(TqpError):
    """tensql::EncodingError (columnar.hpp:23-26)."""


class CudaError(TqpError):
    pass


_ERR = {1: KernelError, 2: ExecError, 3: PlanError, 4: EncodingError, 5: CudaError, 6: TqpError}


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("bad_row", C.c_int64), ("msg", C.c_char * 1024)]


class Codec(C.Structure):
    """tqp_codec: the per-column codec of the compressed host format."""
    _fields_ = [("codec", C.c_int32), ("width", C.c_int32), ("base", C.c_int64), ("scale", C.c_int64),
                ("dict_n", C.c_int32), ("reserved", C.c_int32)]

    NAMES = {0: "raw", 1: "for", 2: "dict", 3: "dec", 4: "delta", 5: "rowdict"}

    @property
    def name(self) -> str:
        return self.NAMES.get(self.codec, "?")


class InstrDesc(C.Structure):
    _fields_ = [
        ("op", C.c_char_p), ("inputs", C.POINTER(C.c_int)), ("num_inputs", C.c_int), ("output", C.c_int),
        ("cmp", C.c_int), ("arith", C.c_int), ("logic", C.c_int), ("side", C.c_int), ("reduce", C.c_int),
        ("anchor", C.c_int), ("cast_to", C.c_int), ("pattern", C.c_char_p), ("pattern_len", C.c_int64),
        ("table", C.c_char_p), ("column", C.c_char_p), ("param", C.c_int64),
        ("const_dtype", C.c_int), ("const_rows", C.c_int64), ("const_cols", C.c_int64),
        ("const_data", C.c_void_p),
    ]


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2209_04579_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH))
    P, I, I64_, D, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64
    S = C.POINTER(Status)
    sig = {
        "tqp_abi_version": (I, []),
        "tqp_init": (P, [I, S]), "tqp_shutdown": (None, [P]), "tqp_sync": (I, [P, S]),
        "tqp_stream": (P, [P]), "tqp_backend_name": (C.c_char_p, [P]), "tqp_device": (I, [P]),
        "tqp_launch_count": (I64_, [P]), "tqp_dtype_size": (C.c_size_t, [I]), "tqp_jit_nvrtc_version": (I, []),
        "tqp_tensor_from_host": (P, [P, I, I64_, I64_, P, S]),
        "tqp_codec_bound": (I64_, [I, I64_, I64_]),
        "tqp_codec_encode": (I64_, [I, I64_, I64_, P, P, I64_, P, S]),
        "tqp_tensor_from_encoded": (P, [P, I, I64_, I64_, P, P, I64_, S]),
        "tqp_tensor_wait": (I, [P, S]),
        "tqp_executor_execute_async": (P, [P, C.POINTER(C.c_char_p), C.POINTER(P), I, S]),
        "tqp_pending_wait": (P, [P, S]),
        "tqp_pending_free": (None, [P]),
        "tqp_tensor_from_host_utf8_i32": (P, [P, I64_, I64_, P, S]),
        "tqp_tensor_from_device": (P, [P, I, I64_, I64_, P, S]),
        "tqp_tensor_dtype": (I, [P]), "tqp_tensor_rows": (I64_, [P]), "tqp_tensor_cols": (I64_, [P]),
        "tqp_tensor_data": (P, [P]), "tqp_tensor_to_host": (I, [P, P, P, S]),
        "tqp_tensor_to_host_utf8_i32": (I, [P, P, P, S]), "tqp_tensor_retain": (P, [P]),
        "tqp_tensor_free": (None, [P]),
        "tqp_compare": (P, [P, P, P, I, S]), "tqp_arith": (P, [P, P, P, I, S]),
        "tqp_logical": (P, [P, P, P, I, S]), "tqp_logical_not": (P, [P, P, S]),
        "tqp_select_where": (P, [P, P, P, P, S]), "tqp_prefix_sum_exclusive": (P, [P, P, S]),
        "tqp_compact": (P, [P, P, P, S]), "tqp_argsort_stable": (P, [P, P, S]),
        "tqp_gather": (P, [P, P, P, S]), "tqp_searchsorted": (P, [P, P, P, I, S]),
        "tqp_expand_segments": (P, [P, P, P, S]), "tqp_segment_starts": (P, [P, P, S]),
        "tqp_segmented_reduce": (P, [P, P, P, I64_, I, S]), "tqp_matmul": (P, [P, P, P, S]),
        "tqp_substring_match": (P, [P, P, C.c_char_p, I64_, I, S]),
        "tqp_iota": (P, [P, I64_, S]), "tqp_cast": (P, [P, P, I, S]), "tqp_exp_f64": (P, [P, P, S]),
        "tqp_last_or_zero": (P, [P, P, S]), "tqp_pack_cols": (P, [P, C.POINTER(P), I, S]),
        "tqp_broadcast_rows": (P, [P, P, I64_, S]), "tqp_pad_width_like": (P, [P, P, P, S]),
        "tqp_sort_perm_rows": (P, [P, P, P, I, S]), "tqp_string_compare": (P, [P, P, P, I, S]),
        "tqp_table_create": (P, [P, S]), "tqp_table_add_column": (I, [P, C.c_char_p, I, P, S]),
        "tqp_table_rows": (I64_, [P]), "tqp_table_num_columns": (I, [P]),
        "tqp_table_column_name": (C.c_char_p, [P, I]), "tqp_table_column_type": (I, [P, I]),
        "tqp_table_column": (P, [P, I]), "tqp_table_free": (None, [P]),
        "tqp_gen_table": (P, [P, C.c_char_p, D, U64, I, I, S]),
        "tqp_csv_parse": (P, [P, C.c_char_p, C.c_int64, C.POINTER(C.c_char_p), C.POINTER(C.c_int), I, C.c_char,
                              C.c_char_p, S]),
        "tqp_csv_load": (P, [P, C.c_char_p, C.POINTER(C.c_char_p), C.POINTER(C.c_int), I, C.c_char, S]),
        "tqp_plan_create": (P, [I, S]), "tqp_plan_begin_step": (I, [P, C.c_char_p, C.c_char_p, S]),
        "tqp_plan_add_instr": (I, [P, C.POINTER(InstrDesc), S]),
        "tqp_plan_set_step_outputs": (I, [P, C.POINTER(C.c_int), I, S]),
        "tqp_plan_add_output": (I, [P, C.c_char_p, I, I, S]),
        "tqp_plan_add_input_column": (I, [P, C.c_char_p, C.c_char_p, I, S]),
        "tqp_plan_free": (None, [P]), "tqp_plan_fusion_explain": (C.c_char_p, [P]),
        "tqp_executor_create": (P, [P, P, C.c_uint, S]),
        "tqp_executor_execute": (P, [P, C.POINTER(C.c_char_p), C.POINTER(P), I, S]),
        "tqp_executor_profile": (P, [P, C.POINTER(C.c_char_p), C.POINTER(P), I, C.POINTER(C.c_void_p), S]),
        "tqp_executor_explain": (C.c_char_p, [P]), "tqp_executor_free": (None, [P]),
        "tqp_executor_fallbacks": (I64_, [P]),
        "tqp_executor_set_timing": (None, [P, I]), "tqp_executor_timings": (C.c_char_p, [P]),
        "tqp_executor_reset_timings": (None, [P]),
        "tqp_executor_shardable": (I, [P, C.POINTER(C.c_char_p)]),
        "tqp_executor_execute_partial": (P, [P, C.POINTER(C.c_char_p), C.POINTER(P), I, S]),
        "tqp_executor_finish": (P, [P, C.POINTER(P), C.POINTER(I64_), I, S]),
        "tqp_free_str": (None, [P]),
        "tqp_comm_nccl_unique_id": (I, [P, S]), "tqp_comm_init_nccl": (P, [P, P, I, I, S]),
        "tqp_comm_init_local": (I, [I, C.POINTER(P), S]), "tqp_comm_rank": (I, [P]), "tqp_comm_size": (I, [P]),
        "tqp_comm_kind": (C.c_char_p, [P]), "tqp_comm_free": (None, [P]),
        "tqp_executor_execute_sharded": (P, [P, P, C.POINTER(C.c_char_p), C.POINTER(P), C.POINTER(I), I, S]),
        "tqp_executor_shard_stats": (C.c_char_p, [P]),
        "tqp_result_rows": (I64_, [P]), "tqp_result_num_columns": (I, [P]),
        "tqp_result_column_name": (C.c_char_p, [P, I]), "tqp_result_column_type": (I, [P, I]),
        "tqp_result_column": (P, [P, I]), "tqp_result_free": (None, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
ABI_SYMBOLS = None  # filled lazily by tests from include/tqp_b200.h


def _check(st: Status, ok: bool):
    if not ok or st.code != 0:
        cls = _ERR.get(st.code, TqpError)
        raise cls(st.msg.decode("utf-8", "replace"), st.bad_row)


class Context:
    """One device + CUDA stream (replaces KernelBackend, backend.hpp:22-70)."""

    def __init__(self, device: int = 0):
        st = Status()
        self.h = lib.tqp_init(device, C.byref(st))
        _check(st, bool(self.h))
        self.device = device

    def sync(self):
        st = Status()
        _check(st, lib.tqp_sync(self.h, C.byref(st)) == 0)

    @property
    def stream(self) -> int:
        return lib.tqp_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return lib.tqp_launch_count(self.h)

    def name(self) -> str:
        return lib.tqp_backend_name(self.h).decode()

    def close(self):
        if getattr(self, "h", None):
            lib.tqp_shutdown(self.h)
            self.h = None


_default: Optional[Context] = None


def encode_column(a: np.ndarray, dtype: int) -> Tuple["Codec", np.ndarray]:
    """Compressed host format of one column (device dtype layout): the codec
    and its payload bytes (tqp_codec_encode; lossless, verified per value)."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    a = np.ascontiguousarray(a, dtype=NP_OF[dtype] if dtype != STR8 else np.uint8)
    rows, cols = a.shape
    out = np.empty(max(1, lib.tqp_codec_bound(dtype, rows, cols)), dtype=np.uint8)
    codec, st = Codec(), Status()
    n = lib.tqp_codec_encode(dtype, rows, cols, a.ctypes.data, out.ctypes.data, out.nbytes, C.byref(codec), C.byref(st))
    _check(st, n >= 0)
    return codec, out[:n].copy()


def nvrtc_version() -> int:
    """NVRTC the run-time specialised kernels compile with (12090 = 12.9)."""
    return int(lib.tqp_jit_nvrtc_version())


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default


class Tensor:
    """Immutable device tensor (tensql::Tensor on HBM)."""

    __slots__ = ("h", "ctx")

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_tensor_free(self.h)
            self.h = None

    @staticmethod
    def from_numpy(a, dtype: Optional[int] = None, ctx: Optional[Context] = None, utf8: bool = False) -> "Tensor":
        ctx = ctx or default_context()
        a = np.asarray(a)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        if a.ndim != 2:
            raise ValueError("tensors are 2-D (rows, cols)")
        if dtype is None:
            dtype = {np.dtype(np.uint8): BOOL, np.dtype(np.bool_): BOOL, np.dtype(np.int32): I32,
                     np.dtype(np.int64): I64, np.dtype(np.float64): F64}[a.dtype]
        st = Status()
        if utf8:
            a = np.ascontiguousarray(a, dtype=np.int32)
            h = lib.tqp_tensor_from_host_utf8_i32(ctx.h, a.shape[0], a.shape[1], a.ctypes.data, C.byref(st))
        else:
            a = np.ascontiguousarray(a, dtype=NP_OF[dtype])
            h = lib.tqp_tensor_from_host(ctx.h, dtype, a.shape[0], a.shape[1], a.ctypes.data, C.byref(st))
        _check(st, bool(h))
        return Tensor(h, ctx)

    @staticmethod
    def from_encoded(codec: "Codec", payload, dtype: int, rows: int, cols: int = 1,
                     ctx: Optional[Context] = None, sync: bool = True) -> "Tensor":
        """Uploads an encoded payload (numpy array or a pinned torch tensor:
        anything with a data pointer) and decodes it on the device (copy
        stream + decode stream; the context stream waits for the decode at
        the tensor's first use). With sync=False the host->device copy may
        still be reading `payload` when this returns: keep it alive and
        unmodified until the tensor has been used (or wait() + ctx.sync())."""
        ctx = ctx or default_context()
        if hasattr(payload, "data_ptr"):
            ptr, nbytes = payload.data_ptr(), payload.numel() * payload.element_size()
        else:
            payload = np.ascontiguousarray(payload)
            ptr, nbytes = payload.ctypes.data, payload.nbytes
        st = Status()
        h = lib.tqp_tensor_from_encoded(ctx.h, dtype, rows, cols, C.byref(codec), ptr, nbytes, C.byref(st))
        _check(st, bool(h))
        t = Tensor(h, ctx)
        if not sync:
            # the copy from `payload` is asynchronous (truly so for pinned
            # memory): the caller keeps it alive and unchanged until used
            return t
        t.wait()
        ctx.sync()
        return t

    def wait(self) -> None:
        """Orders the context stream after this tensor's producer (a decode
        still running on the decode stream)."""
        st = Status()
        lib.tqp_tensor_wait(self.h, C.byref(st))
        _check(st, True)

    @staticmethod
    def from_strings(values: Sequence[str], ctx: Optional[Context] = None) -> "Tensor":
        return Tensor.from_numpy(encode_string_rows(values), ctx=ctx, utf8=True)

    @property
    def dtype(self) -> int:
        return lib.tqp_tensor_dtype(self.h)

    @property
    def rows(self) -> int:
        return lib.tqp_tensor_rows(self.h)

    @property
    def cols(self) -> int:
        return lib.tqp_tensor_cols(self.h)

    @property
    def shape(self) -> Tuple[int, int]:
        return (self.rows, self.cols)

    def data_ptr(self) -> int:
        return lib.tqp_tensor_data(self.h) or 0

    @property
    def __cuda_array_interface__(self) -> dict:
        """Zero-copy view for torch.as_tensor (fixed-width dtypes only); the
        producer stream is synchronised before the view is handed out.

        The view must be treated as READ-ONLY. Tensors are immutable and
        shared by reference (a table column is aliased by LoadColumn results
        and result columns, and its min/max key range is cached with the
        column, executor.hpp Column::range), so an in-place write would change
        every alias and leave the cached range stale. The interface cannot say
        so itself: torch rejects `data: (ptr, True)` ("the read only flag is
        not supported"), so the flag stays False; copy (`.clone()`) before
        writing."""
        if self.dtype == STR8:
            raise TypeError("STR8 tensors have no fixed-width array view")
        self.wait()  # a decode still running on the decode stream
        self.ctx.sync()
        typestr = {BOOL: "|u1", I32: "<i4", I64: "<i8", F64: "<f8"}[self.dtype]
        return {"shape": (self.rows, self.cols), "typestr": typestr, "data": (self.data_ptr(), False),
                "version": 3, "strides": None, "stream": None}

    def numpy(self, widen_strings: bool = True) -> np.ndarray:
        """Host copy; STR8 widens to the reference's Int32-per-byte layout."""
        st = Status()
        if self.dtype == STR8 and widen_strings:
            out = np.empty((self.rows, self.cols), dtype=np.int32)
            _check(st, lib.tqp_tensor_to_host_utf8_i32(self.ctx.h, self.h, out.ctypes.data, C.byref(st)) == 0)
            return out
        out = np.empty((self.rows, self.cols), dtype=NP_OF[self.dtype])
        _check(st, lib.tqp_tensor_to_host(self.ctx.h, self.h, out.ctypes.data, C.byref(st)) == 0)
        return out

    def strings(self) -> List[str]:
        return decode_string_rows(self.numpy())


def encode_string_rows(values: Sequence[str]) -> np.ndarray:
    """columnar.cpp:161-175: (n, m) Int32 UTF-8 bytes, zero padded, m >= 1."""
    bs = [v.encode("utf-8") for v in values]
    m = max([1] + [len(b) for b in bs])
    out = np.zeros((len(bs), m), dtype=np.int32)
    for i, b in enumerate(bs):
        out[i, : len(b)] = np.frombuffer(b, dtype=np.uint8)
    return out


def decode_string_rows(a: np.ndarray) -> List[str]:
    res = []
    for row in np.asarray(a):
        b = bytes(int(x) for x in row)
        res.append(b.split(b"\0", 1)[0].decode("utf-8"))
    return res


def _t(x: Union[Tensor, np.ndarray], ctx=None) -> Tensor:
    return x if isinstance(x, Tensor) else Tensor.from_numpy(x, ctx=ctx)


def _call(fn, ctx: Context, *args) -> Tensor:
    # Tensor arguments stay referenced (alive) for the duration of the call
    st = Status()
    raw = [a.h if isinstance(a, Tensor) else a for a in args]
    h = fn(ctx.h, *raw, C.byref(st))
    del args
    _check(st, bool(h))
    return Tensor(h, ctx)


def _enum(table, v):
    return table[v] if isinstance(v, str) else int(v)


# ---- the kernel set (kernels.hpp:28-78) --------------------------------------
def compare(lhs, rhs, op, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_compare, ctx, _t(lhs, ctx), _t(rhs, ctx), _enum(COMPARE, op))


def arith(lhs, rhs, op, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_arith, ctx, _t(lhs, ctx), _t(rhs, ctx), _enum(ARITH, op))


def logical(lhs, rhs, op, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_logical, ctx, _t(lhs, ctx), _t(rhs, ctx), _enum(LOGICAL, op))


def logical_not(v, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_logical_not, ctx, _t(v, ctx))


def select_where(cond, a, b, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_select_where, ctx, _t(cond, ctx), _t(a, ctx), _t(b, ctx))


def prefix_sum_exclusive(x, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_prefix_sum_exclusive, ctx, _t(x, ctx))


def compact(values, mask, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_compact, ctx, _t(values, ctx), _t(mask, ctx))


def argsort_stable(keys, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_argsort_stable, ctx, _t(keys, ctx))


def gather(values, idx, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_gather, ctx, _t(values, ctx), _t(idx, ctx))


def searchsorted(sorted_, probes, side, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_searchsorted, ctx, _t(sorted_, ctx), _t(probes, ctx), _enum(SIDE, side))


def expand_segments(starts, counts, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_expand_segments, ctx, _t(starts, ctx), _t(counts, ctx))


def segment_starts(sorted_keys, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_segment_starts, ctx, _t(sorted_keys, ctx))


def segmented_reduce(values, segment_ids, num_segments: int, op, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_segmented_reduce, ctx, _t(values, ctx), _t(segment_ids, ctx), int(num_segments),
                 _enum(REDUCE, op))


def matmul(a, b, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_matmul, ctx, _t(a, ctx), _t(b, ctx))


def substring_match(chars, pattern: str, anchor, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    p = pattern.encode("utf-8")
    return _call(lib.tqp_substring_match, ctx, _t(chars, ctx), p, len(p), _enum(ANCHOR, anchor))


# ---- plumbing ops (executor.cpp:190-278) -----------------------------------
def iota(n: int, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_iota, ctx, int(n))


def cast(t, to, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_cast, ctx, _t(t, ctx), _enum(DTYPE_NAMES, to))


def exp_f64(t, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_exp_f64, ctx, _t(t, ctx))


def last_or_zero(t, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_last_or_zero, ctx, _t(t, ctx))


def broadcast_rows(value, n: int, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_broadcast_rows, ctx, _t(value, ctx), int(n))


def pad_width_like(t, like, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_pad_width_like, ctx, _t(t, ctx), _t(like, ctx))


def sort_perm_rows(key, perm, ascending: bool, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_sort_perm_rows, ctx, _t(key, ctx), _t(perm, ctx), 1 if ascending else 0)


def string_compare(a, b, op, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    return _call(lib.tqp_string_compare, ctx, _t(a, ctx), _t(b, ctx), _enum(COMPARE, op))


def pack_cols(cols: Sequence, ctx=None) -> Tensor:
    ctx = ctx or default_context()
    ts = [_t(c, ctx) for c in cols]
    arr = (C.c_void_p * len(ts))(*[t.h for t in ts])
    return _call(lib.tqp_pack_cols, ctx, arr, len(ts))


# ---- tables (EncodedTable, columnar.hpp:41-54) --------------------------------
class Table:
    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_table_free(self.h)
            self.h = None

    @staticmethod
    def create(ctx=None) -> "Table":
        ctx = ctx or default_context()
        st = Status()
        h = lib.tqp_table_create(ctx.h, C.byref(st))
        _check(st, bool(h))
        return Table(h, ctx)

    @staticmethod
    def from_columns(cols: Sequence[Tuple[str, str, object]], ctx=None) -> "Table":
        """cols: (name, logical type name, numpy array | list of str)."""
        ctx = ctx or default_context()
        t = Table.create(ctx)
        for name, lt, data in cols:
            t.add_column(name, lt, data)
        return t

    def add_column(self, name: str, logical: str, data):
        lt = LOGICAL_NAMES[logical]
        if isinstance(data, Tensor):
            tensor = data
        elif lt == LT_UTF8:
            arr = data if isinstance(data, np.ndarray) else encode_string_rows(list(data))
            tensor = Tensor.from_numpy(arr, ctx=self.ctx, utf8=True)
        else:
            dt = {LT_INT64: I64, LT_DATE: I64, LT_FLOAT64: F64, LT_BOOL: BOOL}[lt]
            tensor = Tensor.from_numpy(np.asarray(data).reshape(-1, 1), dtype=dt, ctx=self.ctx)
        st = Status()
        _check(st, lib.tqp_table_add_column(self.h, name.encode(), lt, tensor.h, C.byref(st)) == 0)

    @staticmethod
    def generate(table: str, sf: float, seed: int = 7, shard: int = 0, nshards: int = 1, ctx=None) -> "Table":
        ctx = ctx or default_context()
        st = Status()
        h = lib.tqp_gen_table(ctx.h, table.encode(), float(sf), int(seed), shard, nshards, C.byref(st))
        _check(st, bool(h))
        return Table(h, ctx)

    @staticmethod
    def _csv_schema(schema):
        n = len(schema)
        names = (C.c_char_p * max(1, n))(*[name.encode() for name, _ in schema])
        types = (C.c_int * max(1, n))(*[LOGICAL_NAMES[lt] for _, lt in schema])
        return names, types, n

    @staticmethod
    def from_csv_text(text, schema: Sequence[Tuple[str, str]], delimiter: str = ",", origin: str = "<csv>",
                      ctx=None) -> "Table":
        """tensql::parse_csv_text (columnar.cpp:453-519) on the device:
        schema is [(name, logical type name)]; errors raise EncodingError
        with the reference's messages."""
        ctx = ctx or default_context()
        data = text.encode() if isinstance(text, str) else bytes(text)
        names, types, n = Table._csv_schema(schema)
        st = Status()
        h = lib.tqp_csv_parse(ctx.h, data, len(data), names, types, n, delimiter.encode(), origin.encode(),
                              C.byref(st))
        _check(st, bool(h))
        return Table(h, ctx)

    @staticmethod
    def load_csv(path, schema: Sequence[Tuple[str, str]], delimiter: str = ",", ctx=None) -> "Table":
        """tensql::load_csv (columnar.cpp:521-527): pinned read, one copy to HBM."""
        ctx = ctx or default_context()
        names, types, n = Table._csv_schema(schema)
        st = Status()
        h = lib.tqp_csv_load(ctx.h, str(path).encode(), names, types, n, delimiter.encode(), C.byref(st))
        _check(st, bool(h))
        return Table(h, ctx)

    @property
    def rows(self) -> int:
        return lib.tqp_table_rows(self.h)

    def columns(self) -> List[Tuple[str, str]]:
        n = lib.tqp_table_num_columns(self.h)
        return [(lib.tqp_table_column_name(self.h, i).decode(), LOGICAL_BY_ID[lib.tqp_table_column_type(self.h, i)])
                for i in range(n)]

    def column(self, name: str) -> Tensor:
        for i, (n, _) in enumerate(self.columns()):
            if n.lower() == name.lower():
                return Tensor(lib.tqp_table_column(self.h, i), self.ctx)
        raise EncodingError(f"table: no column named '{name}'")

    def to_numpy(self) -> Dict[str, np.ndarray]:
        return {n: self.column(n).numpy() for n, _ in self.columns()}


# ---- plans + executor (operator_plan.hpp:16-92, executor.hpp:43-59) ----------
class Plan:
    """A lowered tensql OperatorPlan, built through the C ABI."""

    def __init__(self, doc: Mapping):
        self.doc = doc
        st = Status()
        self.h = lib.tqp_plan_create(int(doc["num_slots"]), C.byref(st))
        _check(st, bool(self.h))
        keep = []
        for step in doc["steps"]:
            _check(st, lib.tqp_plan_begin_step(self.h, step["id"].encode(), step["kind"].encode(), C.byref(st)) == 0)
            for ins in step["instrs"]:
                d = InstrDesc()
                d.op = ins["op"].encode()
                inputs = (C.c_int * max(1, len(ins["inputs"])))(*ins["inputs"])
                keep.append(inputs)
                d.inputs = C.cast(inputs, C.POINTER(C.c_int))
                d.num_inputs = len(ins["inputs"])
                d.output = ins["output"]
                d.cmp = COMPARE.get(ins.get("cmp", "eq"), 0)
                d.arith = ARITH.get(ins.get("arith", "add"), 0)
                d.logic = LOGICAL.get(ins.get("logic", "and"), 0)
                d.side = SIDE.get(ins.get("side", "left"), 0)
                d.reduce = REDUCE.get(ins.get("reduce", "sum"), 0)
                d.anchor = ANCHOR.get(ins.get("anchor", "start"), 0)
                d.cast_to = DTYPE_NAMES.get(ins.get("cast_to", "int64"), I64)
                pat = ins.get("pattern", "").encode("utf-8")
                keep.append(pat)
                d.pattern = pat
                d.pattern_len = len(pat)
                d.table = ins.get("table", "").encode()
                d.column = ins.get("column", "").encode()
                d.param = int(ins.get("param", -1))
                if ins["op"] == "const":
                    c = ins["constant"]
                    dt = DTYPE_NAMES[c["dtype"]]
                    arr = np.ascontiguousarray(np.array([_num(v) for v in c["data"]], dtype=NP_OF[dt]))
                    keep.append(arr)
                    d.const_dtype = dt
                    d.const_rows = c["rows"]
                    d.const_cols = c["cols"]
                    d.const_data = arr.ctypes.data
                _check(st, lib.tqp_plan_add_instr(self.h, C.byref(d), C.byref(st)) == 0)
            outs = (C.c_int * max(1, len(step["output_slots"])))(*step["output_slots"])
            _check(st, lib.tqp_plan_set_step_outputs(self.h, outs, len(step["output_slots"]), C.byref(st)) == 0)
        for o in doc["outputs"]:
            _check(st, lib.tqp_plan_add_output(self.h, o["name"].encode(), LOGICAL_NAMES[o["type"]], o["slot"],
                                               C.byref(st)) == 0)
        for t in doc["input_tables"]:
            for c in t["schema"]:
                _check(st, lib.tqp_plan_add_input_column(self.h, t["name"].encode(), c["name"].encode(),
                                                         LOGICAL_NAMES[c["type"]], C.byref(st)) == 0)

    def fusion(self) -> dict:
        """Fused pipelines the executor would choose (host-only planning)."""
        return json.loads(lib.tqp_plan_fusion_explain(self.h).decode())

    @staticmethod
    def from_file(path) -> "Plan":
        with open(path) as f:
            return Plan(json.load(f))

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_plan_free(self.h)
            self.h = None


def _num(v):
    if isinstance(v, str):
        return float(v)  # "nan", "inf", "-inf"
    return v


class Result:
    """Executor output (an EncodedTable on device)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_result_free(self.h)
            self.h = None

    @property
    def rows(self) -> int:
        return lib.tqp_result_rows(self.h)

    def columns(self) -> List[Tuple[str, str]]:
        n = lib.tqp_result_num_columns(self.h)
        return [(lib.tqp_result_column_name(self.h, i).decode(), LOGICAL_BY_ID[lib.tqp_result_column_type(self.h, i)])
                for i in range(n)]

    def column(self, i: int) -> Tensor:
        return Tensor(lib.tqp_tensor_retain(lib.tqp_result_column(self.h, i)), self.ctx)

    def to_numpy(self) -> List[Tuple[str, str, np.ndarray]]:
        return [(n, t, self.column(i).numpy()) for i, (n, t) in enumerate(self.columns())]


class Pending:
    """A queued execution (Executor.execute_async)."""

    def __init__(self, handle, ctx: Context, tables):
        self.h = handle
        self.ctx = ctx
        self._tables = tables  # alive until the result is taken

    def result(self) -> Result:
        h, self.h = self.h, None
        if not h:
            raise RuntimeError("result already taken")
        st = Status()
        r = lib.tqp_pending_wait(h, C.byref(st))
        self._tables = None
        _check(st, bool(r))
        return Result(r, self.ctx)

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_pending_free(self.h)
            self.h = None


SHARD_REPLICATED, SHARD_COPARTITIONED, SHARD_ROWS = 0, 1, 2
# layout of the generator's sharded TPC-H tables (tqp_gen_table shard/nshards):
# lineitem and orders cut on order boundaries, part and customer by rows
TPCH_SHARD_KINDS = {"lineitem": SHARD_COPARTITIONED, "orders": SHARD_COPARTITIONED,
                    "part": SHARD_ROWS, "customer": SHARD_ROWS}


class Comm:
    """A rank of a communicator for Executor.execute_sharded: NCCL (one
    process per GPU; `nccl_unique_id()` on one rank, sent to the others by
    the caller) or an in-process group of thread ranks (`local_group(n)`)."""

    def __init__(self, h):
        self.h = h

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = Status()
        _check(st, lib.tqp_comm_nccl_unique_id(buf, C.byref(st)) == 0)
        return buf.raw

    @staticmethod
    def nccl(uid: bytes, nranks: int, rank: int, ctx: Optional[Context] = None) -> "Comm":
        ctx = ctx or default_context()
        idb = C.create_string_buffer(bytes(uid), 128)
        st = Status()
        h = lib.tqp_comm_init_nccl(ctx.h, idb, nranks, rank, C.byref(st))
        _check(st, bool(h))
        return Comm(h)

    @staticmethod
    def local_group(n: int) -> list:
        arr = (C.c_void_p * n)()
        st = Status()
        _check(st, lib.tqp_comm_init_local(n, arr, C.byref(st)) == 0)
        return [Comm(arr[i]) for i in range(n)]

    @property
    def rank(self) -> int:
        return lib.tqp_comm_rank(self.h)

    @property
    def size(self) -> int:
        return lib.tqp_comm_size(self.h)

    @property
    def kind(self) -> str:
        return lib.tqp_comm_kind(self.h).decode()

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_comm_free(self.h)
            self.h = None


class Executor:
    """tensql::Executor over device tables; fuse=False runs one device kernel
    per instruction (the reference's dispatch loop, executor.cpp:378-408)."""

    def __init__(self, plan: Union[Plan, Mapping], fuse: bool = True, ctx=None):
        self.ctx = ctx or default_context()
        self.plan = plan if isinstance(plan, Plan) else Plan(plan)
        st = Status()
        self.h = lib.tqp_executor_create(self.ctx.h, self.plan.h, EXEC_FUSE if fuse else EXEC_NO_FUSE, C.byref(st))
        _check(st, bool(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            lib.tqp_executor_free(self.h)
            self.h = None

    def set_timing(self, on=True):
        """True: units, steps and every kernel; "scan": the fused fact-scan
        kernels only (cheapest: one event pair per query); False: off."""
        lib.tqp_executor_set_timing(self.h, 2 if on == "scan" else (1 if on else 0))

    def timings(self) -> dict:
        """{unit: {"calls", "total_ms"}} measured with CUDA events."""
        return json.loads(lib.tqp_executor_timings(self.h).decode())

    @property
    def fallbacks(self) -> int:
        """Fused units that ran the exact per-instruction path instead."""
        return int(lib.tqp_executor_fallbacks(self.h))

    def reset_timings(self):
        lib.tqp_executor_reset_timings(self.h)

    def explain(self) -> dict:
        return json.loads(lib.tqp_executor_explain(self.h).decode())

    def _args(self, tables: Mapping[str, Table]):
        # the ctypes arrays are rebuilt only when the table set changes (a
        # repeated query over the same tables skips their construction)
        key = tuple((name, t.h) for name, t in tables.items())
        cached = getattr(self, "_args_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        n = len(key)
        cn = (C.c_char_p * max(1, n))(*[name.encode() for name, _ in key])
        th = (C.c_void_p * max(1, n))(*[h for _, h in key])
        self._args_cache = (key, (cn, th, n))
        return cn, th, n

    def execute(self, tables: Mapping[str, Table]) -> Result:
        cn, th, n = self._args(tables)
        st = Status()
        h = lib.tqp_executor_execute(self.h, cn, th, n, C.byref(st))
        _check(st, bool(h))
        return Result(h, self.ctx)

    def execute_async(self, tables: Mapping[str, Table]) -> "Pending":
        """execute() without the final synchronisation (tqp_executor_execute_async):
        Pending.result() returns the same result and raises the same errors.
        Keep `tables` alive until then."""
        cn, th, n = self._args(tables)
        st = Status()
        h = lib.tqp_executor_execute_async(self.h, cn, th, n, C.byref(st))
        _check(st, bool(h))
        return Pending(h, self.ctx, tables)

    # ---- sharded execution; see distributed.py ----
    def shardable(self) -> Tuple[bool, str]:
        why = C.c_char_p()
        ok = lib.tqp_executor_shardable(self.h, C.byref(why))
        return bool(ok), (why.value or b"").decode()

    def execute_partial(self, tables: Mapping[str, Table]) -> Tensor:
        """Phase 1 over this shard's tables: an opaque I64-word device tensor."""
        cn, th, n = self._args(tables)
        st = Status()
        h = lib.tqp_executor_execute_partial(self.h, cn, th, n, C.byref(st))
        _check(st, bool(h))
        return Tensor(h, self.ctx)

    def finish(self, parts: Sequence) -> Result:
        """Phase 2: merge the partials of every shard (in shard order). Each
        part is a tqp Tensor or a CUDA tensor of int64 words (e.g. from an
        NCCL all-gather); the caller keeps them alive and synchronised."""
        ptrs, words = [], []
        for p in parts:
            if isinstance(p, Tensor):
                ptrs.append(p.data_ptr())
                words.append(p.rows * p.cols)
            else:  # torch.Tensor on this device
                if not p.is_cuda or p.dtype.itemsize != 8 or not p.is_contiguous():
                    raise TypeError("partials must be contiguous 8-byte CUDA tensors")
                ptrs.append(p.data_ptr())
                words.append(p.numel())
        n = len(ptrs)
        pa = (C.c_void_p * max(1, n))(*ptrs)
        wa = (C.c_int64 * max(1, n))(*words)
        st = Status()
        h = lib.tqp_executor_finish(self.h, pa, wa, n, C.byref(st))
        _check(st, bool(h))
        return Result(h, self.ctx)

    def execute_sharded(self, tables: Mapping[str, Table], comm: Comm, kinds: Optional[Mapping[str, int]] = None) -> "Result":
        """One call per rank (tqp_executor_execute_sharded); every rank gets
        the whole result. kinds: table -> SHARD_* (default TPCH_SHARD_KINDS,
        replicated for other names)."""
        kinds = kinds if kinds is not None else TPCH_SHARD_KINDS
        cn, th, n = self._args(tables)
        ka = (C.c_int * max(1, n))(*[int(kinds.get(name.lower(), SHARD_REPLICATED)) for name in tables])
        st = Status()
        h = lib.tqp_executor_execute_sharded(self.h, comm.h, cn, th, ka, n, C.byref(st))
        _check(st, bool(h))
        return Result(h, self.ctx)

    def shard_stats(self) -> dict:
        """What the last execute_sharded did (path, bitmap merges, re-aligned
        tables, bytes exchanged by this rank)."""
        return json.loads(lib.tqp_executor_shard_stats(self.h).decode())

    def profile_execute(self, tables: Mapping[str, Table]) -> Tuple[Result, list]:
        cn, th, n = self._args(tables)
        st = Status()
        out = C.c_void_p()
        h = lib.tqp_executor_profile(self.h, cn, th, n, C.byref(out), C.byref(st))
        _check(st, bool(h))
        trace = json.loads(C.string_at(out.value).decode())
        lib.tqp_free_str(out)
        return Result(h, self.ctx), trace
