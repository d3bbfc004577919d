"""Test fixtures: small seeded databases, pin models and brute-force references.

Brute-force references here are deliberately different algorithms from the oracle
(nested loops, sorted-array search), so that agreement pins the oracle to something
other than itself.
"""
from __future__ import annotations

import json
import os

import numpy as np

import datagen as D

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


class SimpleModel:
    def __init__(self, dims, W, b, shift=None, scale=None):
        self.dims = list(dims)
        self.W = [np.asarray(w, dtype=np.float32).reshape(dims[l + 1], dims[l]) for l, w in enumerate(W)]
        self.b = [np.asarray(x, dtype=np.float32).reshape(dims[l + 1]) for l, x in enumerate(b)]
        self.shift = np.zeros(dims[0], np.float32) if shift is None else np.asarray(shift, np.float32)
        self.scale = np.ones(dims[0], np.float32) if scale is None else np.asarray(scale, np.float32)


def zero_model(dims, out_bias=0.0):
    W = [np.zeros((dims[l + 1], dims[l]), np.float32) for l in range(len(dims) - 1)]
    b = [np.zeros(dims[l + 1], np.float32) for l in range(len(dims) - 1)]
    b[-1][:] = out_bias
    return SimpleModel(dims, W, b)


def linear_threshold_model(cfg, qty_col="l_quantity", shift=25.5):
    """SURVEY.md §8(c) pin (iii): every weight 0 except x_q = l_quantity - 25.5 routed as
    unit0 = +x_q, unit1 = -x_q through every hidden layer, output w = [+1, -1]:
    logit = relu(x) - relu(-x) = q - 25.5, exact in bf16 and fp32 (half-integers <= 24.5).
    So `score > 0.5` is exactly `l_quantity >= 26`, and no row lies within 0.5 of the
    threshold logit."""
    dims = cfg.dims
    k = cfg.feats.index(("fact", qty_col))
    L = len(dims) - 1
    W = [np.zeros((dims[l + 1], dims[l]), np.float32) for l in range(L)]
    b = [np.zeros(dims[l + 1], np.float32) for l in range(L)]
    W[0][0, k] = 1.0
    W[0][1, k] = -1.0
    for l in range(1, L - 1):
        W[l][0, 0] = 1.0
        W[l][1, 1] = 1.0
    W[L - 1][0, 0] = 1.0
    W[L - 1][0, 1] = -1.0
    shift_v = np.zeros(dims[0], np.float32)
    shift_v[k] = shift
    return SimpleModel(dims, W, b, shift=shift_v, scale=np.ones(dims[0], np.float32))


def join_sorted(fact_keys, build_keys):
    """Inner equi-join by sorted-array search: build row of each fact key, -1 on miss."""
    order = np.argsort(build_keys, kind="stable")
    sk = np.asarray(build_keys)[order]
    pos = np.searchsorted(sk, fact_keys)
    pos = np.clip(pos, 0, max(0, len(sk) - 1))
    hit = (len(sk) > 0) & (sk[pos] == fact_keys) if len(sk) else np.zeros(len(fact_keys), bool)
    return np.where(hit, order[pos] if len(sk) else -1, -1)


def chain_matches(cfg, db):
    """Build-row ids of every probe for every fact row (-1 = miss/not reached), via join_sorted."""
    n = db.fact_n
    P = len(cfg.probes)
    m = -np.ones((n, P), np.int64)
    alive = np.ones(n, bool)
    if cfg.prefilter:
        c, lo, hi = cfg.prefilter
        v = db.fact[c]
        alive &= (v >= lo) & (v < hi)
    for p, (bt, src, key, bkey) in enumerate(cfg.probes):
        if src == "fact":
            keys = db.fact[key]
        else:
            rows = m[:, src]
            keys = np.where(rows >= 0, db.builds[src][2][key][np.maximum(rows, 0)], np.iinfo(np.int32).min)
        r = join_sorted(keys, db.builds[p][2][bkey])
        r = np.where(alive, r, -1)
        m[:, p] = r
        alive &= r >= 0
    return m, alive


def column_for_rows(cfg, db, ref, match):
    src, c = ref
    if src == "fact":
        return db.fact[c]
    rows = match[:, src]
    return db.builds[src][2][c][np.maximum(rows, 0)]


def brute_aggregate(cfg, db, selected_mask):
    """Per-group COUNT/SUM over the rows of `selected_mask` (numpy bincount)."""
    match, alive = chain_matches(cfg, db)
    g = column_for_rows(cfg, db, cfg.group, match).astype(np.int64)
    s = column_for_rows(cfg, db, cfg.sum_col, match).astype(np.int64)
    m = selected_mask & alive
    cnt = np.bincount(g[m], minlength=cfg.ngroups)[:cfg.ngroups]
    sm = np.bincount(g[m], weights=None, minlength=cfg.ngroups)
    sm = np.zeros(cfg.ngroups, np.int64)
    np.add.at(sm, g[m], s[m])
    return cnt.astype(np.int64), sm


def small_db(name="c1", sf=0.002, match_rate=0.9, **kw):
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=match_rate, **kw)
    db = D.make_database(cfg)
    return cfg, db


def expand_join(cfg, db):
    """Every joined tuple of the query's probe chain by sorted-array search (a different algorithm from the
    oracle's hash maps): (fact_row[T], build_rows[T, P]) in nested-loop order: fact rows ascending, probes
    in order, the matches of a probe in build-row order (cfg.multi probes may match several rows; the
    others at most one). Pre-filter applied."""
    n = db.fact_n
    rows = np.arange(n, dtype=np.int64)
    if cfg.prefilter:
        c, lo, hi = cfg.prefilter
        v = db.fact[c]
        rows = rows[(v >= lo) & (v < hi)]
    cur = rows[:, None]                      # [T, 1 + p]: fact row, build rows of probes so far
    for p, (bt, src, key, bkey) in enumerate(cfg.probes):
        if src == "fact":
            keys = db.fact[key][cur[:, 0]]
        else:
            keys = db.builds[src][2][key][cur[:, 1 + src]]
        bk = np.asarray(db.builds[p][2][bkey])
        order = np.argsort(bk, kind="stable")  # equal keys keep build-row order
        sk = bk[order]
        lo = np.searchsorted(sk, keys, side="left")
        hi = np.searchsorted(sk, keys, side="right")
        cnt = hi - lo
        if p not in cfg.multi:
            assert cnt.max(initial=0) <= 1, "duplicate key on a unique probe"
        rep = np.repeat(np.arange(len(cur)), cnt)
        within = np.arange(len(rep)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        cur = np.concatenate([cur[rep], order[lo[rep] + within][:, None]], axis=1)
    return cur[:, 0], cur[:, 1:]


def tuple_column(cfg, db, ref, fact_row, build_rows):
    src, c = ref
    if src == "fact":
        return db.fact[c][fact_row]
    return db.builds[src][2][c][build_rows[:, src]]


def tuple_aggregate(cfg, db, fact_row, build_rows, mask):
    g = tuple_column(cfg, db, cfg.group, fact_row, build_rows).astype(np.int64)[mask]
    s = tuple_column(cfg, db, cfg.sum_col, fact_row, build_rows).astype(np.int64)[mask]
    cnt = np.bincount(g, minlength=cfg.ngroups)[:cfg.ngroups].astype(np.int64)
    sm = np.zeros(cfg.ngroups, np.int64)
    np.add.at(sm, g, s)
    return cnt, sm


def star_chain_db(seed=0, nfact=3000, dup=True):
    """A small schema for join chains and duplicate build keys (NEXT-4, the Favorita-style multi-table
    natural join P:1163-1168): fact F(k_a, k_c, v, f0, f1, g) probes A on k_a (A keys repeat when `dup`:
    up to 3 rows per key), A's a_b probes B (unique), and F's k_c probes C (unique). Seeded numpy."""
    rng = np.random.default_rng(seed)
    na, nb, nc = 400, 150, 90
    a_keys = rng.integers(0, 300, na) if dup else rng.permutation(2000)[:na]
    A = {"a_key": a_keys.astype(np.int32), "a_b": rng.integers(0, nb + 20, na).astype(np.int32),
         "a_f": rng.normal(size=na).astype(np.float32), "a_g": rng.integers(0, 4, na).astype(np.int32)}
    B = {"b_key": rng.permutation(nb + 40)[:nb].astype(np.int32), "b_f": rng.normal(size=nb).astype(np.float32),
         "b_q": rng.integers(0, 50, nb).astype(np.int32)}
    C = {"c_key": (np.arange(nc) * 7 - 100).astype(np.int32), "c_f": rng.normal(size=nc).astype(np.float32)}
    F = {"k_a": rng.integers(-10, 320 if dup else 2100, nfact).astype(np.int32),
         "k_c": (rng.integers(-5, nc + 5, nfact) * 7 - 100).astype(np.int32),
         "v": rng.integers(0, 100000, nfact).astype(np.int32),
         "f0": rng.normal(size=nfact).astype(np.float32), "f1": rng.integers(0, 9, nfact).astype(np.int32),
         "ship": rng.integers(0, 100, nfact).astype(np.int32)}
    import datagen as D
    cfg = D.QueryConfig("star", 0.0, [8, 64, 1],
                        [("fact", "f0"), ("fact", "f1"), (0, "a_f"), (0, "a_b"), (1, "b_f"), (1, "b_q"), (2, "c_f"),
                         ("fact", "v")],
                        [("A", "fact", "k_a", "a_key"), ("B", 0, "a_b", "b_key"), ("C", "fact", "k_c", "c_key")],
                        group=(0, "a_g"), ngroups=4, sum_col=("fact", "v"), multi=(0,) if dup else ())
    db = D.Database(0.0, nfact, F, [("A", na, A), ("B", nb, B), ("C", nc, C)])
    return cfg, db
