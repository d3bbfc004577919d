"""Parity rules between the CUDA path (through the C ABI) and the oracle (SURVEY.md §8(c),
BASELINE.json north_star):
  1. join results bit-exact: build-row id of every probe for every fact row;
  2. scores: max |score_gpu - score_oracle| <= 1e-2 over rows that reached the model (and the
     same set of rows reaches the model);
  3. selection: outside the band B = {|score_oracle - t| <= 1e-2} the selected flags are equal;
  4. aggregates over the agreed row set: A_gpu == sum over (i not in B, oracle selects i) +
     sum over (i in B, GPU selects i), int64-exact; and the bracket A_hi <= A_gpu <= A_hi + A_band.
"""
from __future__ import annotations

import math

import numpy as np

import oracle as O
from paper_2311_02781_b200 import flern as F
from paper_2311_02781_b200.session import GpuQuery
from tests import helpers as H

SCORE_TOL = 1e-2   # north_star: max-abs 1e-2 (bf16) vs the fp64 oracle
BAND = 1e-2        # rows within this of the threshold are excluded from the predicate comparison


def unpack_bits(words, n):
    b = np.unpackbits(words.view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


def run_gpu(cfg, db, model, threshold=None, both=False, debug=True, gq=None, flags=0):
    own = gq is None
    gq = gq or GpuQuery(cfg, db, model)
    try:
        n = db.fact_n
        G = cfg.ngroups
        P = len(cfg.probes)
        count = np.zeros(2 * G, np.int64)
        sm = np.zeros(2 * G, np.int64)
        counters = np.zeros(4, np.int64)
        score = np.empty(max(1, n), np.float32) if debug else None
        match = np.empty(max(1, n * P), np.int32) if debug else None
        sel = np.zeros(max(1, (n + 31) // 32), np.uint32) if debug else None
        q = gq.make_query(gq.fact_id, threshold=threshold, flags=(F.FLERN_Q_BOTH_CLASSES if both else 0) | flags)
        res = gq.run(q, count=count, sum=sm, counters=counters, dbg_score=score, dbg_match=match, dbg_selected=sel)
        out = dict(count=count[:G].copy(), sum=sm[:G].copy(), count_rej=count[G:].copy(), sum_rej=sm[G:].copy(),
                   counters=counters, rows_joined=res.rows_joined, rows_selected=res.rows_selected,
                   rows_scanned=res.rows_scanned, elapsed_ms=res.elapsed_ms)
        if debug:
            out["score"] = score[:n]
            out["match"] = match[:n * P].reshape(n, P)
            out["selected"] = unpack_bits(sel, n)
        return out
    finally:
        if own:
            gq.close()


def check(cfg, db, model, threshold=None, both=False, emu_tol=None, gq=None, flags=0):
    t = cfg.threshold if threshold is None else threshold
    g = run_gpu(cfg, db, model, threshold=t, both=both, gq=gq, flags=flags)
    o = O.run(cfg, db, model, threshold=t, band=BAND, per_row=True)
    n = db.fact_n
    # 1. join ids, bit-exact
    assert np.array_equal(g["match"], o.match.astype(np.int32)), "join ids differ"
    assert g["rows_joined"] == o.rows_joined
    assert g["rows_scanned"] == n
    # 2. scores
    reached_o = ~np.isnan(o.score)
    reached_g = ~np.isnan(g["score"])
    assert np.array_equal(reached_o, reached_g), "different rows reached the model"
    err = np.abs(g["score"][reached_o].astype(np.float64) - o.score[reached_o])
    max_err = float(err.max()) if err.size else 0.0
    assert max_err <= SCORE_TOL, f"max |score diff| {max_err}"
    if emu_tol is not None and err.size:
        e = O.run(cfg, db, model, threshold=t, band=BAND, per_row=True, emulate_bf16=True)
        emax = float(np.abs(g["score"][reached_o].astype(np.float64) - e.score[reached_o]).max())
        assert emax <= emu_tol, f"GPU vs bf16-emulating oracle {emax}"
    # 3. selection outside the band
    in_band = reached_o & (np.abs(o.score - t) <= BAND)
    outside = reached_o & ~in_band
    assert np.array_equal(g["selected"][outside], o.selected[outside]), "selection differs outside the band"
    assert not g["selected"][~reached_o].any()
    # 4. aggregates over the agreed row set (exact), and the export-free bracket
    match, alive = H.chain_matches(cfg, db)
    gcode = H.column_for_rows(cfg, db, cfg.group, match).astype(np.int64)
    sval = H.column_for_rows(cfg, db, cfg.sum_col, match).astype(np.int64)
    agreed = (o.selected & ~in_band) | (g["selected"] & in_band)
    G = cfg.ngroups
    cnt = np.bincount(gcode[agreed], minlength=G)[:G]
    sm = np.zeros(G, np.int64)
    np.add.at(sm, gcode[agreed], sval[agreed])
    assert g["count"].tolist() == cnt.tolist(), (g["count"], cnt)
    assert g["sum"].tolist() == sm.tolist()
    assert np.all(o.count_hi <= g["count"]) and np.all(g["count"] <= o.count_hi + o.count_band)
    assert np.all(o.sum_hi <= g["sum"]) and np.all(g["sum"] <= o.sum_hi + o.sum_band)
    assert g["rows_selected"] == int(g["count"].sum())
    if both:   # conservation: selected + rejected == joined, per group
        cnt_all, sum_all = H.brute_aggregate(cfg, db, np.ones(n, bool))
        assert (g["count"] + g["count_rej"]).tolist() == cnt_all.tolist()
        assert (g["sum"] + g["sum_rej"]).tolist() == sum_all.tolist()
    return dict(max_err=max_err, band=int(in_band.sum()), scored=int(reached_o.sum()), gpu=g, oracle=o)


def sample_check(cfg, db, model, gq, rows, threshold=None):
    """Full-size parity on sampled rows: the GPU runs on the whole table (the launch configuration
    bench.py times); the oracle computes the sampled rows one range at a time."""
    t = cfg.threshold if threshold is None else threshold
    g = run_gpu(cfg, db, model, threshold=t, gq=gq)
    worst = 0.0
    for lo, hi in rows:
        o = O.run(cfg, db, model, threshold=t, band=BAND, per_row=True, row_lo=lo, row_hi=hi)
        assert np.array_equal(g["match"][lo:hi], o.match.astype(np.int32))
        ro = ~np.isnan(o.score)
        assert np.array_equal(ro, ~np.isnan(g["score"][lo:hi]))
        if ro.any():
            worst = max(worst, float(np.abs(g["score"][lo:hi][ro] - o.score[ro]).max()))
        outside = ro & (np.abs(o.score - t) > BAND)
        assert np.array_equal(g["selected"][lo:hi][outside], o.selected[outside])
    assert worst <= SCORE_TOL, worst
    return g, worst
