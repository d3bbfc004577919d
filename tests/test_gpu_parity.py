"""CUDA path vs the oracle, through the C ABI, on the same seeded inputs (`-m gpu`)."""
import math

import numpy as np
import pytest

import datagen as D
import oracle as O
from tests import helpers as H
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


# ---------------------------------------------------------------------------------- configs
@pytest.mark.parametrize("match_rate", [1.0, 0.9])
def test_c1_full_config(match_rate):
    """Config 1 (SF0.01, L⋈O, 8-64-1) at its full size, with and without probe misses."""
    cfg = D.with_sf(D.CONFIGS["c1"], 0.01, match_rate=match_rate)
    db = D.make_database(cfg)
    r = parity.check(cfg, db, D.make_model(cfg, db), emu_tol=3e-3)
    assert r["scored"] > 0.85 * db.fact_n * match_rate


@pytest.mark.parametrize("sf", [0.003, 0.02])
def test_c2_mlp_small(sf):
    """Config 2's query and 16-256-256-1 MLP at sizes the oracle finishes in seconds (many tiles
    and a ragged tail), with probe misses."""
    cfg = D.with_sf(D.CONFIGS["c2"], sf, match_rate=0.9)
    db = D.make_database(cfg)
    parity.check(cfg, db, D.make_model(cfg, db), emu_tol=3e-3)


def test_c2_both_classes_conservation():
    """The paper's two-class CASE WHEN query: selected + rejected == joined."""
    cfg = D.with_sf(D.CONFIGS["c2"], 0.004, match_rate=0.9)
    db = D.make_database(cfg)
    parity.check(cfg, db, D.make_model(cfg, db), both=True)


def test_c4p_prefilter_before_inference():
    """Config 4's selective l_shipdate pre-filter (~2%) before inference, C2's MLP."""
    cfg = D.with_sf(D.CONFIGS["c4p"], 0.1, match_rate=0.95)
    db = D.make_database(cfg)
    r = parity.check(cfg, db, D.make_model(cfg, db))
    assert 0.015 * db.fact_n < r["scored"] < 0.03 * db.fact_n


@pytest.mark.parametrize("name", ["c1", "c2", "c4p"])
def test_linear_threshold_model_bit_exact(name):
    """Pin (iii): with the linear-threshold model the query is exactly `l_quantity >= 26`; no row
    is in the band, so join, selection and aggregates must be bit-exact."""
    sf = 0.1 if name == "c4p" else 0.01
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    model = H.linear_threshold_model(cfg)
    r = parity.check(cfg, db, model)
    assert r["band"] == 0
    cnt, sm = H.brute_aggregate(cfg, db, db.fact["l_quantity"] >= 26)
    assert r["gpu"]["count"].tolist() == cnt.tolist() and r["gpu"]["sum"].tolist() == sm.tolist()


@pytest.mark.parametrize("t", [-math.inf, 0.0, math.inf, 1.0, 0.3])
def test_threshold_extremes(t):
    cfg = D.with_sf(D.CONFIGS["c1"], 0.004, match_rate=0.9)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    r = parity.check(cfg, db, model, threshold=t)
    if t <= 0:
        assert r["gpu"]["rows_selected"] == r["gpu"]["rows_joined"]
    if t >= 1:
        assert r["gpu"]["rows_selected"] == 0


# ---------------------------------------------------------------------------------- edge cases
def _custom_db(cfg, nfact, seed=0, miss=0.2):
    rng = np.random.default_rng(seed)
    full = D.make_database(D.with_sf(cfg, 0.002))
    bname, m, bcols = full.builds[0]
    keys = bcols["o_orderkey"]
    take = rng.integers(0, m, size=nfact)
    fact = {}
    src = D.make_database(D.with_sf(cfg, 0.002)).fact
    rows = rng.integers(0, full.fact_n, size=nfact)
    for c, v in src.items():
        fact[c] = np.ascontiguousarray(v[rows]) if nfact else v[:0].copy()
    fk = keys[take].copy()
    u = rng.random(nfact)
    fk[u < miss] = -7   # misses
    # and some probe keys equal to the empty-slot marker INT32_MIN: they must miss too
    fk[u < miss / 4] = np.iinfo(np.int32).min
    fact["l_orderkey"] = fk.astype(np.int32)
    return D.Database(cfg.sf, nfact, fact, full.builds)


@pytest.mark.parametrize("nfact", [0, 1, 127, 128, 129, 255, 256, 257, 1000, 33_333])
def test_ragged_sizes(nfact):
    cfg = D.with_sf(D.CONFIGS["c1"], 0.002)
    db = _custom_db(cfg, nfact, seed=nfact)
    model = D.make_model(cfg, D.make_database(cfg))
    r = parity.check(cfg, db, model)
    assert r["gpu"]["rows_scanned"] == nfact


@pytest.mark.parametrize("name", ["c2", "c3", "c4p"])
@pytest.mark.parametrize("nfact", [0, 1, 129, 255, 4_097])
def test_ragged_sizes_other_kernels(name, nfact):
    """Ragged fact sizes (empty, one row, a partial tile, a partial last batch) on the two-hidden-layer
    narrow kernel (C2, the bench's), the wide kernel (C3) and the pre-filter path (C4p)."""
    cfg = D.with_sf(D.CONFIGS[name], 0.002)
    db = _custom_db(cfg, nfact, seed=nfact + 11)
    model = D.make_model(cfg, D.make_database(cfg))
    r = parity.check(cfg, db, model)
    assert r["gpu"]["rows_scanned"] == nfact


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_int32_min_probe_key_misses(name):
    """A fact key equal to INT32_MIN (the fat table's empty-entry key) hashes onto an empty entry: it
    must be a miss, not a join with build row -1 (P:328-331 emits joinCond matches only). Every third
    fact row carries it; join ids, scores, selection and aggregates against the oracle."""
    cfg = D.with_sf(D.CONFIGS[name], 0.004, match_rate=0.9)
    db = D.make_database(cfg)
    fk = db.fact["l_orderkey"].copy()
    fk[::3] = np.iinfo(np.int32).min
    db.fact["l_orderkey"] = fk
    r = parity.check(cfg, db, D.make_model(cfg, db))
    assert r["oracle"].match[::3].max() == -1 and r["gpu"]["rows_joined"] < 0.7 * db.fact_n


@pytest.mark.parametrize("name,miss", [("c2", 1.0), ("c1", 1.0), ("c1", 0.97)])
def test_all_probes_miss(name, miss):
    """Every (or nearly every) probe misses: empty tiles never reach the MLP; with per-warp tiles (C1)
    most warp batches publish no stage at all."""
    cfg = D.with_sf(D.CONFIGS[name], 0.002)
    db = _custom_db(cfg, 5000, miss=miss)
    if miss < 1.0:
        r = parity.check(cfg, db, D.make_model(cfg, D.make_database(cfg)))
        assert 0 < r["gpu"]["rows_joined"] < 0.1 * 5000
        return
    r = parity.check(cfg, db, D.make_model(cfg, D.make_database(cfg)))
    assert r["gpu"]["rows_joined"] == 0 and r["gpu"]["count"].sum() == 0


def test_wide_pairs_unbalanced_tiles():
    """The wide kernel runs on CTA pairs whose two CTAs produce different numbers of tiles: here the
    fact rows after the first tenth all miss their first probe, so most CTAs run out of joined rows at
    once while the CTAs that claimed the first chunks still have many tiles (their pair partners run
    dummy tiles until the pair stops). Join ids, scores, selection and aggregates against the oracle."""
    cfg = D.with_sf(D.CONFIGS["c3"], 0.02, match_rate=0.9)
    db = D.make_database(cfg)
    fk = db.fact["l_orderkey"].copy()
    cut = db.fact_n // 10
    fk[cut:] = np.iinfo(np.int32).max - 7   # no such order key
    db.fact["l_orderkey"] = fk
    r = parity.check(cfg, db, _calibrated(cfg, db))
    assert 0 < r["gpu"]["rows_joined"] <= cut


def test_shuffled_fact_rows_same_aggregates():
    """Permutation invariance on the GPU: shuffled lineitem gives bit-identical aggregates
    (integer atomics; the tile decomposition changes, the result must not)."""
    cfg = D.with_sf(D.CONFIGS["c1"], 0.01, match_rate=0.9)
    db = D.make_database(cfg)
    model = H.linear_threshold_model(cfg)
    a = parity.run_gpu(cfg, db, model, debug=False)
    b = parity.run_gpu(cfg, D.make_database(cfg, shuffle_seed=3), model, debug=False)
    assert a["count"].tolist() == b["count"].tolist() and a["sum"].tolist() == b["sum"].tolist()


def test_repeated_runs_deterministic():
    cfg = D.with_sf(D.CONFIGS["c2"], 0.01, match_rate=0.9)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    from paper_2311_02781_b200.session import GpuQuery
    gq = GpuQuery(cfg, db, model)
    try:
        r1 = parity.run_gpu(cfg, db, model, gq=gq)
        r2 = parity.run_gpu(cfg, db, model, gq=gq)
        assert r1["count"].tolist() == r2["count"].tolist() and r1["sum"].tolist() == r2["sum"].tolist()
        assert np.array_equal(r1["score"], r2["score"], equal_nan=True)
    finally:
        gq.close()


# ---------------------------------------------------------------------------------- errors
def test_errors_name_the_offender():
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS["c1"], 0.002)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    gq = GpuQuery(cfg, db, model)
    try:
        with pytest.raises(F.FlernError, match="DUPLICATE.*fact"):
            F.flern_load_table(gq.ctx, "fact", db.fact)
        q = gq.make_query(gq.fact_id)
        q.q.nfeat = 7
        with pytest.raises(F.FlernError, match="ARITY"):
            gq.run(q, count=np.zeros(5, np.int64), sum=np.zeros(5, np.int64))
        q = gq.make_query(gq.fact_id, threshold=float("nan"))
        with pytest.raises(F.FlernError, match="NaN"):
            gq.run(q, count=np.zeros(5, np.int64), sum=np.zeros(5, np.int64))
        dup = F.flern_load_table(gq.ctx, "dupdim", {"k": np.array([1, 2, 1], np.int32)})
        with pytest.raises(F.FlernError, match="DUP_KEY"):
            F.flern_build_hashtable(gq.ctx, dup, "k", [])
        with pytest.raises(F.FlernError, match="NOT_FOUND.*nope"):
            F.flern_build_hashtable(gq.ctx, dup, "nope", [])
        with pytest.raises(F.FlernError, match="SHAPE"):
            F.flern_load_model(gq.ctx, "bad", [8, 64, 2], [np.zeros((64, 8)), np.zeros((2, 64))],
                               [np.zeros(64), np.zeros(2)], np.zeros(8), np.ones(8))
        with pytest.raises(F.FlernError, match="UNSUPPORTED"):
            F.flern_load_model(gq.ctx, "big", [8, 1024, 1], [np.zeros((1024, 8)), np.zeros((1, 1024))],
                               [np.zeros(1024), np.zeros(1)], np.zeros(8), np.ones(8))
        # the context is still usable after errors
        r = parity.run_gpu(cfg, db, model, gq=gq, debug=False)
        assert r["rows_joined"] > 0
    finally:
        gq.close()


def test_bad_group_code_is_reported():
    from paper_2311_02781_b200 import flern as F
    cfg = D.with_sf(D.CONFIGS["c1"], 0.002)
    db = D.make_database(cfg)
    cfg.ngroups = 3   # o_orderpriority takes 5 values
    with pytest.raises(F.FlernError, match="group code"):
        parity.run_gpu(cfg, db, D.make_model(D.with_sf(D.CONFIGS["c1"], 0.002), db), debug=False)


# ---------------------------------------------------------------------------------- full size
@pytest.mark.slow
@pytest.mark.parametrize("name,sf", [("c2", 1.0), ("c1", 10.0)])
def test_c2_full_size_sampled(name, sf):
    """Config 2 at its full size (SF1, 6.0M rows), and the C1 shape at SF10 (bench's c1x row, 60M
    rows, per-warp tiles), in the launch configuration bench.py times: join ids, scores and selection on
    sampled row ranges against the oracle; aggregates at -INF and with the linear-threshold model exact
    at full size."""
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS[name], sf)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    gq = GpuQuery(cfg, db, model)
    try:
        n = db.fact_n
        rng = np.random.default_rng(5)
        starts = sorted(rng.integers(0, n - 2000, size=8).tolist()) + [n - 1500]
        _, worst = parity.sample_check(cfg, db, model, gq, [(s, min(n, s + 1500)) for s in starts])
        g = parity.run_gpu(cfg, db, model, threshold=-math.inf, gq=gq, debug=False)
        cnt, sm = H.brute_aggregate(cfg, db, np.ones(n, bool))
        assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()
    finally:
        gq.close()
    lt = H.linear_threshold_model(cfg)
    g = parity.run_gpu(cfg, db, lt, debug=False)
    cnt, sm = H.brute_aggregate(cfg, db, db.fact["l_quantity"] >= 26)
    assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()


@pytest.mark.slow
@pytest.mark.parametrize("name,sf", [("c2", 1.0), ("c1", 10.0), ("c4p", 10.0)])
def test_full_size_real_model_aggregates(name, sf):
    """Bench launch configurations with the real (calibrated) model and no debug exports, so the kernel
    variant bench.py times runs (C1x: the pipelined one-layer producer and lean epilogue; C2: SF1 in
    full; C4p: the pre-filter path at SF10): join and selection counts and the aggregates against the
    oracle over the whole table, through parity rule 4's export-free bracket: rows the oracle scores
    above the band are selected, rows inside the band may go either way (A_hi <= A_gpu <= A_hi + A_band),
    and the GPU's selected-row count equals the sum of its group counts."""
    import oracle as O
    cfg = D.with_sf(D.CONFIGS[name], sf)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    g = parity.run_gpu(cfg, db, model, debug=False)
    o = O.run(cfg, db, model, band=parity.BAND)
    assert g["rows_scanned"] == db.fact_n
    assert g["rows_joined"] == o.rows_joined
    assert np.all(o.count_hi <= g["count"]) and np.all(g["count"] <= o.count_hi + o.count_band), (g["count"], o.count_hi)
    assert np.all(o.sum_hi <= g["sum"]) and np.all(g["sum"] <= o.sum_hi + o.sum_band)
    assert g["rows_selected"] == int(g["count"].sum())
    # the band is a small share of the scored rows (calibrated models: std(logit) ~ 1)
    assert int(o.count_band.sum()) <= 0.10 * max(1, o.rows_joined)


def test_no_model_mode_is_join_aggregate():
    """FLERN_Q_NO_MODEL (diagnostic used for the HBM roofline of scan/probe/gather): every joined
    row is selected, so the aggregates equal the brute-force join aggregate."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    for name in ("c1", "c2"):
        cfg = D.with_sf(D.CONFIGS[name], 0.01, match_rate=0.9)
        db = D.make_database(cfg)
        gq = GpuQuery(cfg, db, D.make_model(cfg, db))
        try:
            cnt = np.zeros(cfg.ngroups, np.int64)
            sm = np.zeros(cfg.ngroups, np.int64)
            q = gq.make_query(gq.fact_id, flags=F.FLERN_Q_NO_MODEL)
            gq.run(q, count=cnt, sum=sm)
            c2, s2 = H.brute_aggregate(cfg, db, np.ones(db.fact_n, bool))
            assert cnt.tolist() == c2.tolist() and sm.tolist() == s2.tolist()
        finally:
            gq.close()


@pytest.mark.parametrize("kind", ["skewed", "sparse", "negative"])
def test_hash_build_key_distributions(kind):
    """The build picks an order-preserving range hash for dense key ranges and falls back to
    Fibonacci hashing for sparse or skewed ones; either way the join ids equal the oracle's,
    including probe keys outside the build key range."""
    rng = np.random.default_rng(11)
    n = 20000
    if kind == "skewed":     # a dense cluster plus a few far-away keys: long chains under the range hash
        bkeys = np.concatenate([np.arange(5000, 5000 + n - 50), rng.choice(10**9, 50, replace=False) + 10**6])
    elif kind == "sparse":   # range far larger than 16 x capacity
        bkeys = rng.choice(2**31 - 2, n, replace=False) - 2**30
    else:
        bkeys = np.arange(-n, 0) * 3
    bkeys = rng.permutation(bkeys).astype(np.int32)
    cfg = D.QueryConfig("h", 0.0, [8, 64, 1], [("fact", f"f{k}") for k in range(8)],
                        [("dim", "fact", "k", "dk")], group=(0, "dg"), ngroups=4, sum_col=("fact", "v"))
    nf = 50000
    fk = rng.choice(np.concatenate([bkeys, rng.integers(-2**31 + 1, 2**31 - 1, 5000).astype(np.int32),
                                    np.full(500, np.iinfo(np.int32).min, np.int32)]), nf)
    fact = {"k": fk.astype(np.int32), "v": rng.integers(0, 1000, nf).astype(np.int32)}
    for k in range(8):
        fact[f"f{k}"] = rng.normal(size=nf).astype(np.float32)
    dim = {"dk": bkeys, "dg": rng.integers(0, 4, n).astype(np.int32)}
    db = D.Database(0.0, nf, fact, [("dim", n, dim)])
    model = H.SimpleModel([8, 64, 1], [rng.normal(size=(64, 8)) * 0.3, rng.normal(size=(1, 64)) * 0.2],
                          [np.zeros(64), np.zeros(1)])
    model.W = [D.bf16_round(w) for w in model.W]
    parity.check(cfg, db, model)


def _calibrated(cfg, db):
    """Random model for `cfg`, output layer scaled (via the oracle) to std(logit) ~ 1."""
    raw = D.make_model(cfg, db, out_scale=1.0, out_shift=0.0)
    r = O.run(cfg, db, raw, per_row=True, threshold=-math.inf)
    lg = r.logit[~np.isnan(r.logit)]
    return D.make_model(cfg, db, out_scale=1.0 / float(lg.std()), out_shift=float(lg.mean()))


@pytest.mark.parametrize("pf", [False, True])
def test_two_probe_chain(pf):
    """Config 3's join chain lineitem ⋈ orders ⋈ customer (two probes, the second keyed by a payload
    word of the first) with its 32 features, on a 32-128-128-1 MLP this build supports; with and
    without config 4's pre-filter."""
    base = D.CONFIGS["c4" if pf else "c3"]
    cfg = D.with_sf(base, 0.1 if pf else 0.01, match_rate=0.9, dims=[32, 128, 128, 1], name="c3s")
    db = D.make_database(cfg)
    r = parity.check(cfg, db, _calibrated(cfg, db))
    assert r["scored"] > 0
    lt = H.linear_threshold_model(cfg)
    r = parity.check(cfg, db, lt)
    assert r["band"] == 0


@pytest.mark.parametrize("name,sf", [("c3", 0.001), ("c4", 0.03)])
def test_wide_mlp_configs(name, sf):
    """Configs 3 and 4 with their real 32-1024-1024-1024-1 MLP (the streamed-weight wide kernel):
    two probes, 32 features, pre-filter for config 4; scores within 1e-2 of the fp64 oracle."""
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    r = parity.check(cfg, db, D.make_model(cfg, db))
    assert r["scored"] > 0
    lt = H.linear_threshold_model(cfg)
    assert parity.check(cfg, db, lt)["band"] == 0


@pytest.mark.parametrize("name", ["c1", "c2", "c4p"])
def test_generic_producer_path(name):
    """The benchmark shapes run a producer specialised for their feature layout; the same queries
    through the generic (run-time shape) producer (FLERN_Q_GENERIC_KERNEL) must give the same parity
    results."""
    from paper_2311_02781_b200 import flern as F
    sf = 0.1 if name == "c4p" else 0.004
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    parity.check(cfg, db, D.make_model(cfg, db), flags=F.FLERN_Q_GENERIC_KERNEL)


def test_update_table_refills_in_place():
    """flern_update_table: the next batch of a copied fact table, no allocation; the result equals a
    fresh load of the same rows, fewer rows are fine, more rows / borrowed tables / unknown columns are
    errors that name the offender."""
    import torch
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS["c2"], 0.004, match_rate=0.9)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    G = cfg.ngroups
    gq = GpuQuery(cfg, db, model)
    try:
        base = gq.run(count=np.zeros(G, np.int64), sum=np.zeros(G, np.int64))
        ref_c, ref_s = np.zeros(G, np.int64), np.zeros(G, np.int64)
        gq.run(count=ref_c, sum=ref_s)
        perm = np.random.default_rng(7).permutation(db.fact_n)
        shuffled = {k: np.ascontiguousarray(v[perm]) for k, v in db.fact.items()}
        F.flern_update_table(gq.ctx, gq.fact_id, shuffled, F.FLERN_COPY_HOST)   # same rows, new order
        c, s_ = np.zeros(G, np.int64), np.zeros(G, np.int64)
        r = gq.run(count=c, sum=s_)
        assert r.rows_scanned == db.fact_n and r.rows_joined == base.rows_joined
        assert (c == ref_c).all() and (s_ == ref_s).all()
        half = {k: np.ascontiguousarray(v[: db.fact_n // 2]) for k, v in db.fact.items()}
        F.flern_update_table(gq.ctx, gq.fact_id, half, F.FLERN_COPY_HOST)      # fewer rows
        r = gq.run(count=np.zeros(G, np.int64), sum=np.zeros(G, np.int64))
        assert r.rows_scanned == db.fact_n // 2
        bigger = {k: np.concatenate([v, v[:8]]) for k, v in db.fact.items()}
        with pytest.raises(F.FlernError, match="capacity"):
            F.flern_update_table(gq.ctx, gq.fact_id, bigger, F.FLERN_COPY_HOST)
        bad = dict(half)
        bad["no_such_col"] = bad.pop(next(iter(bad)))
        with pytest.raises(F.FlernError, match="no_such_col"):
            F.flern_update_table(gq.ctx, gq.fact_id, bad, F.FLERN_COPY_HOST)
        dev = {k: torch.from_numpy(v).cuda() for k, v in db.fact.items()}
        tid = F.flern_load_table(gq.ctx, "borrowed", dev, F.FLERN_BORROW_DEVICE)
        with pytest.raises(F.FlernError, match="borrowed"):
            F.flern_update_table(gq.ctx, tid, db.fact, F.FLERN_COPY_HOST)
    finally:
        gq.close()


@pytest.mark.parametrize("chunk", [1000, 4096, 10**9])
def test_streamed_query_equals_resident(chunk):
    """flern_run_query_streamed (host fact rows through a ring of device chunk buffers, copies overlapped
    with the chunk launches) gives exactly the resident query's aggregates and counters, for
    chunks that do not divide the table, more chunks than ring slots, and a single chunk; the table's
    own rows are neither read nor changed."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS["c2"], 0.003, match_rate=0.9)
    db = D.make_database(cfg)
    gq = GpuQuery(cfg, db, D.make_model(cfg, db))
    G = cfg.ngroups
    try:
        rc, rs = np.zeros(G, np.int64), np.zeros(G, np.int64)
        ref = gq.run(count=rc, sum=rs)
        perm = np.random.default_rng(3).permutation(db.fact_n)
        host = {k: np.ascontiguousarray(v[perm]) for k, v in db.fact.items()}   # new order, same rows
        c, s_ = np.zeros(G, np.int64), np.zeros(G, np.int64)
        r = F.flern_run_query_streamed(gq.ctx, gq.query, host, chunk, count=c, sum=s_)
        assert (c == rc).all() and (s_ == rs).all()
        assert (r.rows_scanned, r.rows_joined, r.rows_selected) == (ref.rows_scanned, ref.rows_joined, ref.rows_selected)
        # the resident table is untouched
        c2, s2 = np.zeros(G, np.int64), np.zeros(G, np.int64)
        gq.run(count=c2, sum=s2)
        assert (c2 == rc).all() and (s2 == rs).all()
    finally:
        gq.close()


@pytest.mark.parametrize("name,chunk", [("c2", 1000), ("c1", 777), ("c4p", 20000)])
def test_streamed_beyond_ring_vs_oracle(name, chunk):
    """NEXT-2 beyond device capacity: the fact table on the device is a schema with 0 rows, the rows live
    in host memory only and stream through the 3-slot ring in many more chunks than slots. Against the
    oracle: exact with the linear-threshold model (no band), and the export-free bracket with the random
    model; counters equal the oracle's."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    sf = 0.05 if name == "c4p" else 0.004
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    G = cfg.ngroups
    for model in (H.linear_threshold_model(cfg), D.make_model(cfg, db)):
        gq = GpuQuery(cfg, db, model, load_fact=False)
        try:
            schema = {k: np.zeros(0, v.dtype) for k, v in db.fact.items()}
            gq.set_fact(F.flern_load_table(gq.ctx, "fact_schema", schema))
            c, s_ = np.zeros(G, np.int64), np.zeros(G, np.int64)
            r = F.flern_run_query_streamed(gq.ctx, gq.query, db.fact, chunk, count=c, sum=s_)
            assert -(-db.fact_n // chunk) > 3
            o = O.run(cfg, db, model, band=parity.BAND)
            assert r.rows_scanned == db.fact_n and r.rows_joined == o.rows_joined
            assert np.all(o.count_hi <= c) and np.all(c <= o.count_hi + o.count_band)
            assert np.all(o.sum_hi <= s_) and np.all(s_ <= o.sum_hi + o.sum_band)
            if o.rows_band == 0:
                assert c.tolist() == o.count.tolist() and s_.tolist() == o.sum.tolist()
        finally:
            gq.close()


def test_streamed_query_validates_before_copying():
    """A streamed query that cannot run (a column it reads is not streamed, a dtype that changes, a
    duplicate column) fails before any copy or launch and leaves the context usable."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS["c2"], 0.002, match_rate=0.9)
    db = D.make_database(cfg)
    gq = GpuQuery(cfg, db, D.make_model(cfg, db))
    G = cfg.ngroups
    try:
        rc, rs = np.zeros(G, np.int64), np.zeros(G, np.int64)
        gq.run(count=rc, sum=rs)
        part = dict(db.fact)
        part.pop("l_shipmode")
        with pytest.raises(F.FlernError, match="NOT_FOUND.*l_shipmode"):
            F.flern_run_query_streamed(gq.ctx, gq.query, part, 1000, count=np.zeros(G, np.int64),
                                       sum=np.zeros(G, np.int64))
        bad = dict(db.fact)
        bad["l_quantity"] = bad["l_quantity"].astype(np.float32)
        with pytest.raises(F.FlernError, match="TYPE"):
            F.flern_run_query_streamed(gq.ctx, gq.query, bad, 1000, count=np.zeros(G, np.int64),
                                       sum=np.zeros(G, np.int64))
        c, s_ = np.zeros(G, np.int64), np.zeros(G, np.int64)
        gq.run(count=c, sum=s_)
        assert (c == rc).all() and (s_ == rs).all()
    finally:
        gq.close()


@pytest.mark.parametrize("sf,both", [(0.0005, False), (0.004, False), (0.004, True)])
def test_large_group_domain(sf, both):
    """NEXT-1: GROUP BY a fact column with more than 64 groups (l_partkey: ~100 and ~800 dense codes),
    aggregated with per-row int64 atomics straight into the result; exact against the oracle, with the
    two-class conservation check."""
    import dataclasses
    base = D.with_sf(D.CONFIGS["c2"], sf, match_rate=0.9)
    db = D.make_database(base)
    G = int(db.fact["l_partkey"].max()) + 1
    assert G > 64
    cfg = dataclasses.replace(base, group=("fact", "l_partkey"), ngroups=G)
    parity.check(cfg, db, D.make_model(cfg, db), both=both)


@pytest.mark.parametrize("col,G,both", [("l_returnflag", 3, False), ("l_shipmode", 7, False), ("l_linenumber", 8, False),
                                         ("l_shipmode", 7, True), ("l_linenumber", 40, False)])
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_small_group_domains(name, col, G, both):
    """Every width of the per-thread group-by registers (<= 4, <= 6, <= 8 groups, one and two classes)
    and the ballot path (9..64 groups): GROUP BY a small-domain fact column, exact against the oracle."""
    import dataclasses
    cfg = dataclasses.replace(D.with_sf(D.CONFIGS[name], 0.003, match_rate=0.9), group=("fact", col), ngroups=G)
    db = D.make_database(cfg)
    assert col in db.fact
    parity.check(cfg, db, D.make_model(cfg, db), both=both)


@pytest.mark.parametrize("name,sf", [("c4p", 0.05), ("c3", 0.01)])
def test_streamed_query_prefilter_and_two_probes(name, sf):
    """flern_run_query_streamed over the pre-filter path (filter column windowed per chunk) and the
    two-probe wide-MLP chain: the streamed aggregates equal the resident query's."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    gq = GpuQuery(cfg, db, D.make_model(cfg, db))
    G = cfg.ngroups
    try:
        rc, rs = np.zeros(G, np.int64), np.zeros(G, np.int64)
        ref = gq.run(count=rc, sum=rs)
        c, s_ = np.zeros(G, np.int64), np.zeros(G, np.int64)
        r = F.flern_run_query_streamed(gq.ctx, gq.query, db.fact, 10000, count=c, sum=s_)
        assert (c == rc).all() and (s_ == rs).all()
        assert (r.rows_scanned, r.rows_joined) == (ref.rows_scanned, ref.rows_joined)
    finally:
        gq.close()


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_wide_full_size_sampled(name):
    """Configs 3 and 4 at their full size (SF10, 60M fact rows, two probes, 32-1024-1024-1024-1) in the
    launch configuration bench.py times: join ids, scores and selection on sampled row ranges against
    the oracle; aggregates at -INF exact against the brute-force join (over the pre-filter survivors
    for C4)."""
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.CONFIGS[name]
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    gq = GpuQuery(cfg, db, model)
    try:
        n = db.fact_n
        rng = np.random.default_rng(11)
        starts = sorted(rng.integers(0, n - 1000, size=5).tolist()) + [n - 700]
        _, worst = parity.sample_check(cfg, db, model, gq, [(s, min(n, s + 700)) for s in starts])
        g = parity.run_gpu(cfg, db, model, threshold=-math.inf, gq=gq, debug=False)
        keep = np.ones(n, bool)
        if cfg.prefilter:
            col, lo, hi = cfg.prefilter
            keep = (db.fact[col] >= lo) & (db.fact[col] < hi)
        cnt, sm = H.brute_aggregate(cfg, db, keep)
        assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()
    finally:
        gq.close()


NARROW_SHAPES = [(k, h, 1) for k in (8, 24, 40) for h in (64, 128, 256)] + \
                [(k, h, 2) for k in (8, 24, 40) for h in (64, 128)] + [(16, 256, 2)]
WIDE_SHAPES = [(16, 512, 2), (16, 1024, 2), (16, 1024, 3), (32, 512, 2), (32, 1024, 3), (40, 1024, 2)]


@pytest.mark.parametrize("k0,h,nl", NARROW_SHAPES + WIDE_SHAPES)
def test_every_kernel_shape(k0, h, nl):
    """Every compiled (K0P, H, hidden layers) kernel with a calibrated random model on config 3's
    two-probe chain (features: the first k0 of config 3's 32, repeated past 32): scores, selection
    and aggregates against the oracle."""
    import dataclasses
    base = D.CONFIGS["c3"]
    feats = (base.feats * 2)[:k0]
    sf = 0.0005 if h >= 512 else 0.002
    cfg = dataclasses.replace(D.with_sf(base, sf, match_rate=0.9), dims=[k0] + [h] * nl + [1], feats=feats,
                              name=f"shape{k0}_{h}_{nl}")
    db = D.make_database(cfg)
    r = parity.check(cfg, db, _calibrated(cfg, db))
    assert r["scored"] > 0
