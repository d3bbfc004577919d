"""ctypes binding of libflern.so (include/flern.h) — argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module only converts
Python/NumPy/torch arguments into the C structs. If the library is missing it raises
ImportError (there is no fallback of any kind).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FLERN_LIB: diagnostic builds of the same library (e.g. -DFLERN_TRACE_WAITS) under lib/
LIB_PATH = os.path.join(_HERE, "lib", os.environ.get("FLERN_LIB", "libflern.so"))
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
_lib = ctypes.CDLL(LIB_PATH)

c_i32, c_i64, c_u32, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p

FLERN_OK = 0
ERRORS = {-1: "FLERN_E_INVALID_ARG", -2: "FLERN_E_NOT_FOUND", -3: "FLERN_E_DUPLICATE", -4: "FLERN_E_TYPE",
          -5: "FLERN_E_ARITY", -6: "FLERN_E_SHAPE", -7: "FLERN_E_DUP_KEY", -8: "FLERN_E_CUDA", -9: "FLERN_E_OOM",
          -10: "FLERN_E_UNSUPPORTED"}
FLERN_I32, FLERN_F32, FLERN_DATE32, FLERN_DEC32, FLERN_DICT32 = 1, 2, 3, 4, 5
FLERN_COPY_HOST, FLERN_COPY_DEVICE, FLERN_BORROW_DEVICE = 0x1, 0x2, 0x4
FLERN_HT_MULTI = 0x1
FLERN_Q_RESULT_DEVICE, FLERN_Q_ASYNC, FLERN_Q_BOTH_CLASSES, FLERN_Q_NO_MODEL, FLERN_Q_GENERIC_KERNEL = 0x1, 0x2, 0x4, 0x8, 0x10
EXPORTED = ["flern_create", "flern_destroy", "flern_last_error", "flern_version", "flern_load_table",
            "flern_update_table", "flern_run_query_streamed", "flern_drop_table", "flern_load_model", "flern_build_hashtable", "flern_build_hashtable_ex", "flern_run_query", "flern_train_step", "flern_get_model",
            "flern_query_launches"]


class FlernColumn(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("dtype", ctypes.c_int), ("scale", c_i32), ("data", c_p)]


class FlernProbe(ctypes.Structure):
    _fields_ = [("ht_id", c_i32), ("src", c_i32), ("key_col", ctypes.c_char_p)]


class FlernColref(ctypes.Structure):
    _fields_ = [("src", c_i32), ("col", ctypes.c_char_p)]


class FlernQuery(ctypes.Structure):
    _fields_ = [("fact_table", c_i32), ("prefilter_col", ctypes.c_char_p), ("pf_lo", c_i64), ("pf_hi", c_i64),
                ("nprobes", c_i32), ("probes", ctypes.POINTER(FlernProbe)), ("model_id", c_i32),
                ("nfeat", c_i32), ("feats", ctypes.POINTER(FlernColref)), ("threshold", ctypes.c_float),
                ("group_col", FlernColref), ("ngroups", c_i32), ("sum_col", FlernColref), ("flags", c_u32)]


class FlernResult(ctypes.Structure):
    _fields_ = [("count", c_p), ("sum", c_p), ("counters", c_p), ("dbg_score", c_p), ("dbg_match", c_p),
                ("dbg_selected", c_p), ("dbg_trace", c_p), ("rows_scanned", c_i64), ("rows_joined", c_i64), ("rows_scored", c_i64),
                ("rows_selected", c_i64), ("elapsed_ms", ctypes.c_float)]


_lib.flern_create.argtypes = [ctypes.c_int, c_p, ctypes.POINTER(c_p)]
_lib.flern_create.restype = c_i32
_lib.flern_destroy.argtypes = [c_p]
_lib.flern_destroy.restype = None
_lib.flern_last_error.argtypes = [c_p]
_lib.flern_last_error.restype = ctypes.c_char_p
_lib.flern_version.argtypes = []
_lib.flern_version.restype = ctypes.c_char_p
_lib.flern_load_table.argtypes = [c_p, ctypes.c_char_p, c_i64, c_i32, ctypes.POINTER(FlernColumn), c_u32,
                                  ctypes.POINTER(c_i32)]
_lib.flern_load_table.restype = c_i32
_lib.flern_update_table.argtypes = [c_p, c_i32, c_i64, c_i32, ctypes.POINTER(FlernColumn), c_u32]
_lib.flern_update_table.restype = c_i32
_lib.flern_run_query_streamed.argtypes = [c_p, ctypes.POINTER(FlernQuery), c_i64, c_i32, ctypes.POINTER(FlernColumn),
                                          c_i64, ctypes.POINTER(FlernResult)]
_lib.flern_run_query_streamed.restype = c_i32
_lib.flern_drop_table.argtypes = [c_p, c_i32]
_lib.flern_drop_table.restype = c_i32
_lib.flern_load_model.argtypes = [c_p, ctypes.c_char_p, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_p),
                                  ctypes.POINTER(c_p), c_p, c_p, ctypes.POINTER(c_i32)]
_lib.flern_load_model.restype = c_i32
_lib.flern_build_hashtable.argtypes = [c_p, c_i32, ctypes.c_char_p, c_i32, ctypes.POINTER(ctypes.c_char_p),
                                       ctypes.POINTER(c_i32)]
_lib.flern_build_hashtable.restype = c_i32
_lib.flern_build_hashtable_ex.argtypes = [c_p, c_i32, ctypes.c_char_p, c_i32, ctypes.POINTER(ctypes.c_char_p), c_u32,
                                          ctypes.POINTER(c_i32)]
_lib.flern_build_hashtable_ex.restype = c_i32
_lib.flern_run_query.argtypes = [c_p, ctypes.POINTER(FlernQuery), ctypes.POINTER(FlernResult)]
_lib.flern_run_query.restype = c_i32
class FlernTrainResult(ctypes.Structure):
    _fields_ = [("rows_scanned", c_i64), ("rows_joined", c_i64), ("loss", ctypes.c_double), ("elapsed_ms", ctypes.c_float)]


_lib.flern_train_step.argtypes = [c_p, ctypes.POINTER(FlernQuery), c_i64, c_i64, ctypes.c_float,
                                  ctypes.POINTER(FlernTrainResult)]
_lib.flern_train_step.restype = c_i32
_lib.flern_get_model.argtypes = [c_p, c_i32, ctypes.POINTER(c_p), ctypes.POINTER(c_p)]
_lib.flern_get_model.restype = c_i32
_lib.flern_query_launches.argtypes = []
_lib.flern_query_launches.restype = c_i32


class FlernError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()   # torch tensor (host or device)


def _dtype_of(a, name):
    dt = a.dtype if isinstance(a, np.ndarray) else str(a.dtype)
    if dt in (np.float32, "torch.float32"):
        return FLERN_F32
    if dt in (np.int32, "torch.int32"):
        return FLERN_I32
    raise TypeError(f"column {name}: 4-byte int32/float32 expected, got {dt}")


def flern_version() -> str:
    return _lib.flern_version().decode()


def flern_query_launches() -> int:
    return _lib.flern_query_launches()


def flern_create(device: int = 0, stream: int | None = None):
    h = c_p()
    rc = _lib.flern_create(device, c_p(stream) if stream else None, ctypes.byref(h))
    if rc != FLERN_OK:
        raise FlernError(rc, "flern_create failed (an sm_100 device is required)")
    return h.value


def flern_destroy(ctx):
    _lib.flern_destroy(ctx)


def flern_last_error(ctx) -> str:
    return _lib.flern_last_error(ctx).decode()


def _check(ctx, rc):
    if rc != FLERN_OK:
        raise FlernError(rc, flern_last_error(ctx))


def _columns(columns: dict, dtypes: dict | None):
    names = list(columns)
    n = len(columns[names[0]]) if names else 0
    arr = (FlernColumn * len(names))()
    keep = []
    for i, c in enumerate(names):
        a = columns[c]
        if isinstance(a, np.ndarray):
            a = np.ascontiguousarray(a)
            keep.append(a)
        if len(a) != n:
            raise ValueError(f"column {c}: length {len(a)} != {n}")
        dt = (dtypes or {}).get(c, _dtype_of(a, c))
        b = c.encode()
        keep.append(b)
        arr[i] = FlernColumn(b, dt, 0, _ptr(a))
    return n, arr, keep


def flern_update_table(ctx, table_id: int, columns: dict, flags: int = FLERN_COPY_HOST, dtypes: dict | None = None):
    """Refill a copied table in place with the next batch of the same columns (no allocation)."""
    n, arr, keep = _columns(columns, dtypes)
    _check(ctx, _lib.flern_update_table(ctx, table_id, n, len(arr), arr, flags))


def flern_load_table(ctx, name: str, columns: dict, flags: int = FLERN_COPY_HOST, dtypes: dict | None = None) -> int:
    """columns: {name: array} (numpy host arrays, or torch tensors on host / device per flags)."""
    n, arr, keep = _columns(columns, dtypes)
    tid = c_i32()
    _check(ctx, _lib.flern_load_table(ctx, name.encode(), n, len(arr), arr, flags, ctypes.byref(tid)))
    return tid.value


def flern_drop_table(ctx, table_id: int):
    _check(ctx, _lib.flern_drop_table(ctx, table_id))


def flern_load_model(ctx, name: str, dims, W, b, shift, scale) -> int:
    L = len(dims) - 1
    cd = (c_i32 * (L + 1))(*dims)
    Ws = [np.ascontiguousarray(w, dtype=np.float32) for w in W]
    bs = [np.ascontiguousarray(x, dtype=np.float32) for x in b]
    sh = np.ascontiguousarray(shift, dtype=np.float32)
    sc = np.ascontiguousarray(scale, dtype=np.float32)
    mid = c_i32()
    _check(ctx, _lib.flern_load_model(ctx, name.encode(), L, cd, (c_p * L)(*[w.ctypes.data for w in Ws]),
                                      (c_p * L)(*[x.ctypes.data for x in bs]), sh.ctypes.data, sc.ctypes.data,
                                      ctypes.byref(mid)))
    return mid.value


def flern_build_hashtable(ctx, table_id: int, key_col: str, payload_cols) -> int:
    pcs = [c.encode() for c in payload_cols]
    arr = (ctypes.c_char_p * max(1, len(pcs)))(*pcs)
    hid = c_i32()
    _check(ctx, _lib.flern_build_hashtable(ctx, table_id, key_col.encode(), len(pcs), arr, ctypes.byref(hid)))
    return hid.value


def flern_build_hashtable_ex(ctx, table_id: int, key_col: str, payload_cols, flags: int = 0) -> int:
    """flern_build_hashtable with flags (FLERN_HT_MULTI: the build key may repeat)."""
    pcs = [c.encode() for c in payload_cols]
    arr = (ctypes.c_char_p * max(1, len(pcs)))(*pcs)
    hid = c_i32()
    _check(ctx, _lib.flern_build_hashtable_ex(ctx, table_id, key_col.encode(), len(pcs), arr, flags, ctypes.byref(hid)))
    return hid.value


class Query:
    """Marshals a query once (keeps the ctypes objects alive) so it can be run many times."""

    def __init__(self, fact_table, probes, model_id, feats, group, ngroups, sum_col, threshold=0.5,
                 prefilter=None, flags=0):
        self._keep = []

        def s(x):
            b = x.encode()
            self._keep.append(b)
            return b

        pr = (FlernProbe * len(probes))(*[FlernProbe(h, src, s(k)) for h, src, k in probes])
        fs = (FlernColref * max(1, len(feats)))(*[FlernColref(src, s(c)) for src, c in feats])
        self._keep += [pr, fs]
        self.q = FlernQuery(fact_table, s(prefilter[0]) if prefilter else None,
                            prefilter[1] if prefilter else 0, prefilter[2] if prefilter else 0,
                            len(probes), pr, model_id, len(feats), fs, float(threshold),
                            FlernColref(group[0], s(group[1])), ngroups, FlernColref(sum_col[0], s(sum_col[1])), flags)
        self.ngroups = ngroups


TRACE_EVENTS = 26
TRACE_TILES = 256


def flern_run_query(ctx, query: Query, count=None, sum=None, counters=None, dbg_score=None, dbg_match=None,
                    dbg_selected=None, dbg_trace=None, flags: int | None = None) -> FlernResult:
    """Runs `query`. Output buffers: numpy host arrays (default) or device tensors with
    FLERN_Q_RESULT_DEVICE in flags. Returns the FlernResult (count/sum written in place)."""
    if flags is not None:
        query.q.flags = flags
    res = FlernResult(_ptr(count), _ptr(sum), _ptr(counters), _ptr(dbg_score), _ptr(dbg_match), _ptr(dbg_selected),
                      _ptr(dbg_trace), 0, 0, 0, 0, 0.0)
    _check(ctx, _lib.flern_run_query(ctx, ctypes.byref(query.q), ctypes.byref(res)))
    return res


def flern_run_query_streamed(ctx, query: Query, columns: dict, chunk_rows: int, count=None, sum=None,
                             counters=None) -> FlernResult:
    """Runs `query` over host columns {name: array} (pinned torch tensors or numpy arrays) streamed into
    the query's fact table in chunks of `chunk_rows`, copies overlapped with the chunk queries."""
    n, arr, keep = _columns(columns, None)
    res = FlernResult(_ptr(count), _ptr(sum), _ptr(counters), None, None, None, None, 0, 0, 0, 0, 0.0)
    _check(ctx, _lib.flern_run_query_streamed(ctx, ctypes.byref(query.q), n, len(arr), arr, chunk_rows,
                                              ctypes.byref(res)))
    return res


def flern_train_step(ctx, query: Query, row_lo: int, row_hi: int, lr: float) -> FlernTrainResult:
    """One SGD step of the query's model on the joined tuples of fact rows [row_lo, row_hi) (target: the
    query's sum column)."""
    res = FlernTrainResult(0, 0, 0.0, 0.0)
    _check(ctx, _lib.flern_train_step(ctx, ctypes.byref(query.q), row_lo, row_hi, lr, ctypes.byref(res)))
    return res


def flern_get_model(ctx, model_id: int, dims):
    """The model's current fp32 weights: (W list of [out][in], b list of [out])."""
    L = len(dims) - 1
    W = [np.zeros((dims[l + 1], dims[l]), np.float32) for l in range(L)]
    b = [np.zeros(dims[l + 1], np.float32) for l in range(L)]
    _check(ctx, _lib.flern_get_model(ctx, model_id, (c_p * L)(*[w.ctypes.data for w in W]),
                                     (c_p * L)(*[x.ctypes.data for x in b])))
    return W, b
