"""ctypes wrapper of the CPU oracle (oracle.cpp). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module. The product path never does (and has no way to: it
shares no code with it). The oracle is pinned by tests/test_oracle_*.py; see
DESIGN.md §Oracle for what pins each function.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

c_i32, c_i64, c_dbl, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class OrColumn(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("is_float", c_i32), ("data", c_p)]


class OrTable(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i32), ("cols", ctypes.POINTER(OrColumn))]


class OrProbe(ctypes.Structure):
    _fields_ = [("build_table", c_i32), ("src", c_i32), ("key_col", ctypes.c_char_p),
                ("build_key_col", ctypes.c_char_p), ("multi", c_i32)]


class OrColref(ctypes.Structure):
    _fields_ = [("src", c_i32), ("col", ctypes.c_char_p)]


class OrModel(ctypes.Structure):
    _fields_ = [("nlayers", c_i32), ("dims", ctypes.POINTER(c_i32)), ("W", ctypes.POINTER(c_p)),
                ("b", ctypes.POINTER(c_p)), ("shift", c_p), ("scale", c_p)]


class OrQuery(ctypes.Structure):
    _fields_ = [("prefilter_col", ctypes.c_char_p), ("pf_lo", c_i64), ("pf_hi", c_i64),
                ("nprobes", c_i32), ("probes", ctypes.POINTER(OrProbe)),
                ("nfeat", c_i32), ("feats", ctypes.POINTER(OrColref)),
                ("threshold", c_dbl), ("group", OrColref), ("ngroups", c_i32), ("sum", OrColref),
                ("band", c_dbl), ("emulate_bf16", c_i32), ("nthreads", c_i32),
                ("row_lo", c_i64), ("row_hi", c_i64)]


class OrResult(ctypes.Structure):
    _fields_ = [(n, c_p) for n in ("count", "sum", "count_rej", "sum_rej", "count_hi", "sum_hi",
                                   "count_band", "sum_band", "score", "logit", "match", "selected",
                                   "tuple_x", "tuple_t")] + [("tuple_cap", c_i64)] + \
               [(n, c_i64) for n in ("rows_scanned", "rows_prefiltered", "rows_joined", "rows_selected",
                                     "rows_band")] + [("error", ctypes.c_char * 256)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(_LIB_PATH)
        L.or_run.argtypes = [ctypes.POINTER(OrTable), c_i32, ctypes.POINTER(OrTable), ctypes.POINTER(OrModel),
                             ctypes.POINTER(OrQuery), ctypes.POINTER(OrResult)]
        L.or_run.restype = ctypes.c_int
        L.or_mlp_forward.argtypes = [ctypes.POINTER(OrModel), c_i64, c_p, c_p, c_p, c_i32]
        L.or_mlp_forward.restype = ctypes.c_int
        L.or_mlp_train_step.argtypes = [ctypes.POINTER(OrModel), c_i64, c_p, c_p, c_dbl, ctypes.POINTER(c_p),
                                         ctypes.POINTER(c_p), ctypes.POINTER(c_p), ctypes.POINTER(c_p), c_p]
        L.or_mlp_train_step.restype = ctypes.c_int
        L.or_bf16_rne.argtypes = [ctypes.c_float]
        L.or_bf16_rne.restype = ctypes.c_float
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _src(s):
    return -1 if s == "fact" else int(s)


class _Keep:
    """Holds ctypes objects / arrays alive for the duration of a call."""

    def __init__(self):
        self.items = []

    def __call__(self, x):
        self.items.append(x)
        return x


def _table(cols: dict, nrows: int, keep) -> OrTable:
    arr = (OrColumn * max(1, len(cols)))()
    for i, (name, a) in enumerate(cols.items()):
        a = keep(np.ascontiguousarray(a))
        assert a.dtype.itemsize == 4, name
        arr[i] = OrColumn(keep(name.encode()), 1 if a.dtype == np.float32 else 0, a.ctypes.data)
    keep(arr)
    return OrTable(nrows, len(cols), arr)


def _model(model, keep) -> OrModel:
    L = len(model.dims) - 1
    dims = keep((c_i32 * (L + 1))(*model.dims))
    Ws = [keep(np.ascontiguousarray(w, dtype=np.float32)) for w in model.W]
    bs = [keep(np.ascontiguousarray(b, dtype=np.float32)) for b in model.b]
    Wp = keep((c_p * L)(*[w.ctypes.data for w in Ws]))
    bp = keep((c_p * L)(*[b.ctypes.data for b in bs]))
    shift = keep(np.ascontiguousarray(model.shift, dtype=np.float32))
    scale = keep(np.ascontiguousarray(model.scale, dtype=np.float32))
    return OrModel(L, dims, Wp, bp, shift.ctypes.data, scale.ctypes.data)


@dataclass
class OracleResult:
    count: np.ndarray
    sum: np.ndarray
    count_rej: np.ndarray
    sum_rej: np.ndarray
    count_hi: np.ndarray
    sum_hi: np.ndarray
    count_band: np.ndarray
    sum_band: np.ndarray
    rows_scanned: int
    rows_prefiltered: int
    rows_joined: int
    rows_selected: int
    rows_band: int
    score: np.ndarray | None = None
    logit: np.ndarray | None = None
    match: np.ndarray | None = None
    selected: np.ndarray | None = None


def run(cfg, db, model, threshold=None, band=1e-2, per_row=False, emulate_bf16=False, nthreads=0,
        row_lo=0, row_hi=-1, tuples=None) -> OracleResult:
    """Run the oracle on a datagen.Database with a datagen.Model-like object."""
    keep = _Keep()
    fact = _table(db.fact, db.fact_n, keep)
    btables = (OrTable * max(1, len(db.builds)))()
    for i, (_, m, cols) in enumerate(db.builds):
        btables[i] = _table(cols, m, keep)
    probes = (OrProbe * max(1, len(cfg.probes)))()
    for p, (bt, src, key, bkey) in enumerate(cfg.probes):
        probes[p] = OrProbe(p, _src(src), keep(key.encode()), keep(bkey.encode()),
                            1 if p in getattr(cfg, "multi", ()) else 0)
    feats = (OrColref * max(1, len(cfg.feats)))()
    for k, (src, c) in enumerate(cfg.feats):
        feats[k] = OrColref(_src(src), keep(c.encode()))
    pf = cfg.prefilter
    q = OrQuery(keep(pf[0].encode()) if pf else None, pf[1] if pf else 0, pf[2] if pf else 0,
                len(cfg.probes), probes, len(cfg.feats), feats,
                float(cfg.threshold if threshold is None else threshold),
                OrColref(_src(cfg.group[0]), keep(cfg.group[1].encode())), cfg.ngroups,
                OrColref(_src(cfg.sum_col[0]), keep(cfg.sum_col[1].encode())),
                float(band), 1 if emulate_bf16 else 0, int(nthreads), int(row_lo), int(row_hi))
    G = cfg.ngroups
    outs = {k: np.zeros(G, np.int64) for k in ("count", "sum", "count_rej", "sum_rej", "count_hi", "sum_hi",
                                               "count_band", "sum_band")}
    nrows = (db.fact_n if row_hi < 0 else row_hi) - row_lo
    res = OrResult()
    for k, a in outs.items():
        setattr(res, k, a.ctypes.data)
    extra = {}
    if per_row:
        extra["score"] = np.empty(nrows, np.float64)
        extra["logit"] = np.empty(nrows, np.float64)
        extra["match"] = np.empty((nrows, max(1, len(cfg.probes))), np.int64)
        extra["selected"] = np.empty(nrows, np.uint8)
        for k, a in extra.items():
            setattr(res, k, a.ctypes.data)
    if tuples is not None:   # (X [cap][nfeat], T [cap]) float64 arrays: per-tuple model inputs and targets
        X, T = tuples
        res.tuple_x, res.tuple_t, res.tuple_cap = X.ctypes.data, T.ctypes.data, len(T)
    m = _model(model, keep)
    rc = lib().or_run(ctypes.byref(fact), len(db.builds), btables, ctypes.byref(m), ctypes.byref(q),
                      ctypes.byref(res))
    if rc != 0:
        raise OracleError(res.error.decode())
    if per_row:
        extra["selected"] = extra["selected"].astype(bool)
        extra["match"] = extra["match"][:, :len(cfg.probes)]
    return OracleResult(**outs, rows_scanned=res.rows_scanned, rows_prefiltered=res.rows_prefiltered,
                        rows_joined=res.rows_joined, rows_selected=res.rows_selected, rows_band=res.rows_band,
                        **extra)


def mlp_forward(model, x: np.ndarray, emulate_bf16=False):
    """The oracle's MLP on given (already normalised) feature rows; returns (logits, scores)."""
    keep = _Keep()
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    logits = np.empty(n, np.float64)
    scores = np.empty(n, np.float64)
    m = _model(model, keep)
    lib().or_mlp_forward(ctypes.byref(m), n, x.ctypes.data, logits.ctypes.data, scores.ctypes.data,
                         1 if emulate_bf16 else 0)
    return logits, scores


def bf16_rne(v: float) -> float:
    return lib().or_bf16_rne(v)


def batch(cfg, db, model, row_lo=0, row_hi=-1, cap=None):
    """The joined tuples of fact rows [row_lo, row_hi) as a training batch: (X [B][nfeat] normalised model
    inputs, T [B] targets = the query's sum column), fp64, in the oracle's enumeration order."""
    hi = db.fact_n if row_hi < 0 else row_hi
    cap = cap if cap is not None else max(1, 8 * (hi - row_lo))
    X = np.zeros((cap, len(cfg.feats)), np.float64)
    T = np.zeros(cap, np.float64)
    r = run(cfg, db, model, threshold=-np.inf, nthreads=1, row_lo=row_lo, row_hi=hi, tuples=(X, T))
    assert r.rows_joined <= cap, "tuple capacity"
    return X[:r.rows_joined], T[:r.rows_joined]


def mlp_train_step(model, X, T, lr):
    """One SGD step on rows X with targets T (or_mlp_train_step): returns dict(loss, dW, db, W, b) in fp64."""
    keep = _Keep()
    X = np.ascontiguousarray(X, dtype=np.float64)
    T = np.ascontiguousarray(T, dtype=np.float64)
    dims = list(model.dims)
    L = len(dims) - 1
    outs = {k: [np.zeros((dims[l + 1], dims[l]) if k in ("dW", "W") else dims[l + 1], np.float64) for l in range(L)]
            for k in ("dW", "db", "W", "b")}
    ptrs = {k: keep((c_p * L)(*[a.ctypes.data for a in v])) for k, v in outs.items()}
    loss = ctypes.c_double(0.0)
    m = _model(model, keep)
    rc = lib().or_mlp_train_step(ctypes.byref(m), len(T), X.ctypes.data, T.ctypes.data, float(lr), ptrs["dW"],
                                 ptrs["db"], ptrs["W"], ptrs["b"], ctypes.addressof(loss))
    if rc != 0:
        raise OracleError("or_mlp_train_step: bad model")
    return dict(loss=loss.value, **outs)


def train_step(cfg, db, model, lr, row_lo=0, row_hi=-1):
    """NEXT-3: one SGD step on the batch the query yields for fact rows [row_lo, row_hi)."""
    X, T = batch(cfg, db, model, row_lo, row_hi)
    r = mlp_train_step(model, X, T, lr)
    r["batch"] = len(T)
    return r
