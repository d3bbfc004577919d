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
