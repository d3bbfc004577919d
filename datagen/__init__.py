"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Input plumbing only: this package draws TPC-H-shaped column values and random
model parameters. It holds none of the method's arithmetic (no join, no
normalisation, no MLP forward, no predicate, no aggregate). Both `oracle/` and
`paper_2311_02781_b200/` consume what it produces; neither imports the other.

Recipe: DESIGN.md "Input recipe"; C++ core in flern_gen.cpp.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

SEED = 231102781  # the arXiv id

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libflern_gen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, dbl, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        pp = ctypes.POINTER(ctypes.c_char_p)
        vp = ctypes.POINTER(ctypes.c_void_p)
        L.fg_num_order_slots.argtypes = [dbl]; L.fg_num_order_slots.restype = i64
        L.fg_num_customers.argtypes = [dbl]; L.fg_num_customers.restype = i64
        L.fg_lineitem_rows.argtypes = [u64, dbl, i64, i64]; L.fg_lineitem_rows.restype = i64
        L.fg_orders_rows.argtypes = [u64, dbl, dbl, i64, i64]; L.fg_orders_rows.restype = i64
        L.fg_gen_lineitem.argtypes = [u64, dbl, i64, i64, i32, pp, vp, i32]; L.fg_gen_lineitem.restype = i64
        L.fg_gen_orders.argtypes = [u64, dbl, dbl, i64, i64, i32, pp, vp, i32]; L.fg_gen_orders.restype = i64
        L.fg_gen_customer.argtypes = [u64, dbl, i64, i64, i32, pp, vp, i32]; L.fg_gen_customer.restype = i64
        L.fg_uniform.argtypes = [u64, ctypes.c_uint32, u64, i64, ctypes.c_void_p]; L.fg_uniform.restype = None
        L.fg_perm_keys.argtypes = [u64, i64, ctypes.c_void_p]; L.fg_perm_keys.restype = None
        _lib = L
    return _lib


# Column dtypes: every column is 4 bytes; these are float32, the rest int32.
def col_dtype(name: str):
    base = name.split("_", 1)[1] if "_" in name else name
    return np.float32 if base.startswith("f") and base[1:].isdigit() else np.int32


def _alloc(n, names, alloc):
    outs = {}
    for nm in names:
        dt = col_dtype(nm)
        outs[nm] = alloc(n, dt) if alloc is not None else np.empty(n, dtype=dt)
    return outs


def _ptr(a):
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch (pinned) CPU tensor


def _call(fn, pre_args, names, outs, nthreads):
    cn = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    cp = (ctypes.c_void_p * len(names))(*[_ptr(outs[n]) for n in names])
    r = fn(*pre_args, len(names), cn, cp, nthreads)
    if r < 0:
        raise KeyError(f"unknown column {names[-1 - r]!r}")
    return r


def num_order_slots(sf: float) -> int:
    return lib().fg_num_order_slots(sf)


def num_customers(sf: float) -> int:
    return lib().fg_num_customers(sf)


def shard_slots(sf: float, rank: int, world: int):
    """Contiguous order-slot range of `rank` (fact table sharded by orderkey range)."""
    n = num_order_slots(sf)
    return n * rank // world, n * (rank + 1) // world


def gen_lineitem(sf, names, slot_lo=None, slot_hi=None, seed=SEED, nthreads=0, alloc=None):
    if slot_lo is None:
        slot_lo, slot_hi = 0, num_order_slots(sf)
    n = lib().fg_lineitem_rows(seed, sf, slot_lo, slot_hi)
    outs = _alloc(n, names, alloc)
    if names:
        _call(lib().fg_gen_lineitem, (seed, sf, slot_lo, slot_hi), list(names), outs, nthreads)
    return n, outs


def gen_orders(sf, names, match_rate=1.0, seed=SEED, nthreads=0, slot_lo=None, slot_hi=None):
    if slot_lo is None:
        slot_lo, slot_hi = 0, num_order_slots(sf)
    n = lib().fg_orders_rows(seed, sf, match_rate, slot_lo, slot_hi)
    outs = _alloc(n, names, None)
    if names:
        _call(lib().fg_gen_orders, (seed, sf, match_rate, slot_lo, slot_hi), list(names), outs, nthreads)
    return n, outs


def gen_customer(sf, names, seed=SEED, nthreads=0):
    n = num_customers(sf)
    outs = _alloc(n, names, None)
    if names:
        _call(lib().fg_gen_customer, (seed, sf, 0, n), list(names), outs, nthreads)
    return n, outs


def uniform(seed: int, stream: int, n: int, ctr0: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().fg_uniform(seed, stream, ctr0, n, out.ctypes.data)
    return out


def permutation(seed: int, n: int) -> np.ndarray:
    keys = np.empty(n, dtype=np.uint64)
    lib().fg_perm_keys(seed, n, keys.ctypes.data)
    return np.argsort(keys, kind="stable")


def bf16_round(x) -> np.ndarray:
    """fp32 -> nearest bf16 (round-to-nearest-even), returned as fp32. Format step only."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


# ---------------------------------------------------------------------------------------------
# Query configurations (BASELINE.json configs; SURVEY.md §8(d) feature lists).
# A column reference is (src, name): src = "fact" or the probe index (0, 1) whose build table
# supplies the column.
# ---------------------------------------------------------------------------------------------
C1_L = ["l_quantity", "l_extendedprice", "l_discount", "l_tax", "l_shipdate", "l_receiptdate"]
C2_L = C1_L + ["l_commitdate", "l_linenumber", "l_partkey", "l_suppkey", "l_returnflag", "l_shipmode"]
C3_L = C2_L + ["l_linestatus", "l_shipinstruct"] + [f"l_f{k}" for k in range(6)]
C1_O = ["o_totalprice", "o_orderdate"]
C2_O = C1_O + ["o_orderstatus", "o_f0"]
C3_O = C2_O + [f"o_f{k}" for k in range(1, 5)]
C3_C = ["c_acctbal", "c_nationkey", "c_mktsegment", "c_f0"]

PREFILTER_C4 = ("l_shipdate", 9190, 9238)  # [1995-03-01, 1995-04-18), ~2% of lineitem


@dataclass
class QueryConfig:
    name: str
    sf: float
    dims: list                      # MLP dims [K0, h..., 1]
    feats: list                     # [(src, col)]
    probes: list                    # [(build_table, src, fact_or_src_key_col, build_key_col)]
    prefilter: tuple | None = None  # (col, lo, hi) on the fact table
    group: tuple = (0, "o_orderpriority")
    ngroups: int = 5
    sum_col: tuple = ("fact", "l_extendedprice")
    threshold: float = 0.5
    model_seed: int = SEED
    match_rate: float = 1.0
    multi: tuple = ()               # probes whose build keys may repeat (every match is emitted)

    def fact_cols(self):
        cols = []
        if self.prefilter:
            cols.append(self.prefilter[0])
        for bt, src, key, bkey in self.probes:
            if src == "fact":
                cols.append(key)
        for src, c in self.feats + [self.group, self.sum_col]:
            if src == "fact":
                cols.append(c)
        return list(dict.fromkeys(cols))

    def build_cols(self, p):
        """Columns of probe p's build table needed by the query (key first)."""
        bt, src, key, bkey = self.probes[p]
        cols = [bkey]
        for q, (bt2, src2, key2, bkey2) in enumerate(self.probes):
            if src2 == p:
                cols.append(key2)
        for src, c in self.feats + [self.group, self.sum_col]:
            if src == p:
                cols.append(c)
        return list(dict.fromkeys(cols))


def _feats(l, o, c=()):
    return [("fact", x) for x in l] + [(0, x) for x in o] + [(1, x) for x in c]


PROBE_O = ("orders", "fact", "l_orderkey", "o_orderkey")
PROBE_C = ("customer", 0, "o_custkey", "c_custkey")

CONFIGS = {
    "c1": QueryConfig("c1", 0.01, [8, 64, 1], _feats(C1_L, C1_O), [PROBE_O], model_seed=SEED + 1),
    "c2": QueryConfig("c2", 1.0, [16, 256, 256, 1], _feats(C2_L, C2_O), [PROBE_O], model_seed=SEED + 2),
    "c3": QueryConfig("c3", 10.0, [32, 1024, 1024, 1024, 1], _feats(C3_L, C3_O, C3_C), [PROBE_O, PROBE_C],
                      model_seed=SEED + 3),
    "c4": QueryConfig("c4", 10.0, [32, 1024, 1024, 1024, 1], _feats(C3_L, C3_O, C3_C), [PROBE_O, PROBE_C],
                      prefilter=PREFILTER_C4, model_seed=SEED + 3),
    # secondary rows: C2's query/MLP at C4's filter and at C5's scale
    "c4p": QueryConfig("c4p", 10.0, [16, 256, 256, 1], _feats(C2_L, C2_O), [PROBE_O], prefilter=PREFILTER_C4,
                       model_seed=SEED + 2),
    "c5": QueryConfig("c5", 100.0, [16, 256, 256, 1], _feats(C2_L, C2_O), [PROBE_O], model_seed=SEED + 2),
}


def with_sf(cfg: QueryConfig, sf: float, **kw) -> QueryConfig:
    d = dict(cfg.__dict__)
    d["sf"] = sf
    d.update(kw)
    return QueryConfig(**d)


@dataclass
class Database:
    sf: float
    fact_n: int
    fact: dict                               # lineitem columns (this shard)
    builds: list = field(default_factory=list)   # [(name, nrows, {col: array})] per probe


def make_database(cfg: QueryConfig, rank: int = 0, world: int = 1, seed: int = SEED, alloc=None,
                  shuffle_seed: int | None = None, max_slots: int | None = None) -> Database:
    """Fact shard `rank` of `world` + full build tables. `max_slots` keeps only the first order
    slots (a prefix database: same first rows as the full one, for calibration/sampling)."""
    lo, hi = shard_slots(cfg.sf, rank, world)
    if max_slots is not None:
        hi = min(hi, lo + max_slots)
    n, fact = gen_lineitem(cfg.sf, cfg.fact_cols(), lo, hi, seed=seed, alloc=alloc)
    if shuffle_seed is not None:
        perm = permutation(shuffle_seed, n)
        fact = {k: np.ascontiguousarray(v[perm]) for k, v in fact.items()}
    builds = []
    for p, (bt, src, key, bkey) in enumerate(cfg.probes):
        cols = cfg.build_cols(p)
        if bt == "orders":
            ohi = None if max_slots is None else min(num_order_slots(cfg.sf), max_slots)
            m, d = gen_orders(cfg.sf, cols, match_rate=cfg.match_rate, seed=seed,
                              slot_lo=None if ohi is None else 0, slot_hi=ohi)
        elif bt == "customer":
            m, d = gen_customer(cfg.sf, cols, seed=seed)
        else:
            raise ValueError(bt)
        builds.append((bt, m, d))
    return Database(cfg.sf, n, fact, builds)


# ---------------------------------------------------------------------------------------------
# Random model (seeded input). Hidden layers: W ~ U(±sqrt(6/fan_in)) (He-uniform), b ~ U(±0.1),
# both rounded to bf16 so the GPU's bf16 copy is lossless. Feature
# normalisation (shift, scale) = (mean, 1/std) of the column's first 65,536 values (fp64 -> fp32).
# Output layer: w = bf16(s*u), b = bf16(-s*mu) with u ~ U(±1); (s, mu) come from
# calibration.json, written by scripts/calibrate_models.py from the oracle's logits so that
# std(logit) ~ 1 and the mean logit ~ 0 (selectivity ~50%, band |B| ~ 3.2%).
# ---------------------------------------------------------------------------------------------
@dataclass
class Model:
    dims: list
    W: list          # fp32 [out][in], bf16-exact
    b: list          # fp32 [out], bf16-exact
    shift: np.ndarray
    scale: np.ndarray


_CALIB = os.path.join(_HERE, "calibration.json")


def calibration():
    if os.path.exists(_CALIB):
        with open(_CALIB) as f:
            return json.load(f)
    return {}


# Order slots of the prefix database a model's normalisation is drawn from: make_model(cfg,
# make_database(cfg, max_slots=MODEL_SLOTS)) gives every rank of a sharded run the model of the unsharded
# table (its first 65,536 fact rows and build rows; a slot holds 1-7 lines).
MODEL_SLOTS = 65536


def feature_stats(db: Database, cfg: QueryConfig, nsample: int = 65536):
    shift = np.zeros(len(cfg.feats), np.float32)
    scale = np.ones(len(cfg.feats), np.float32)
    for k, (src, c) in enumerate(cfg.feats):
        col = db.fact[c] if src == "fact" else db.builds[src][2][c]
        x = np.asarray(col[:nsample], dtype=np.float64)
        if x.size == 0:
            continue
        mu, sd = float(x.mean()), float(x.std())
        shift[k] = np.float32(mu)
        scale[k] = np.float32(1.0 / sd) if sd > 0 else np.float32(1.0)
    return shift, scale


def make_model(cfg: QueryConfig, db: Database, out_scale=None, out_shift=None) -> Model:
    dims = list(cfg.dims)
    seed = cfg.model_seed
    W, b = [], []
    L = len(dims) - 1
    for l in range(L):
        fi, fo = dims[l], dims[l + 1]
        u = uniform(seed, 2 * l, fi * fo).reshape(fo, fi)
        ub = uniform(seed, 2 * l + 1, fo)
        if l < L - 1:
            a = math.sqrt(6.0 / fi)
            W.append(bf16_round((2 * u - 1) * a).reshape(fo, fi))
            b.append(bf16_round((2 * ub - 1) * 0.1))
        else:
            cal = calibration().get(cfg.name, {})
            s = out_scale if out_scale is not None else cal.get("out_scale", 1.0)
            mu = out_shift if out_shift is not None else cal.get("out_shift", 0.0)
            W.append(bf16_round((2 * u - 1) * s).reshape(fo, fi))
            b.append(bf16_round(np.full(fo, -s * mu)))
    shift, scale = feature_stats(db, cfg)
    return Model(dims, W, b, shift, scale)
