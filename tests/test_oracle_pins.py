"""Pins of the CPU oracle against things other than itself (CPU-only, `-m "not gpu"`).

Each test names the passage it follows and the mistake it would catch:
 - nested-loop / sorted-search joins (a different algorithm)      -> join bugs, wrong probe source
 - hand-worked golden MLP + query (tests/golden/, dyadic exact)   -> dropped bias, transposed W,
                                                                     ReLU on the output, missing ReLU
 - closed forms: sigmoid(0)=0.5, sigmoid(ln 3)=0.75, zero weights -> sigmoid / predicate bugs
 - the linear-threshold model (score > 0.5 <=> l_quantity >= 26)  -> normalisation sign, chaining
 - invariants: -INF/+INF thresholds, conservation, permutation and shard invariance
"""
import math

import numpy as np
import pytest

import datagen as D
import oracle as O
from tests import helpers as H


# ------------------------------------------------------------------------------------------- MLP
def test_mlp_worked_example_exact():
    """Fig. fig:classifier_generated + ReLU between layers."""
    g = H.golden("mlp_worked.json")
    m = H.SimpleModel(g["dims"], g["W"], g["b"])
    x = np.array([c["x"] for c in g["cases"]], np.float64)
    logits, scores = O.mlp_forward(m, x)
    assert logits.tolist() == [c["logit"] for c in g["cases"]]      # exact: dyadic rationals
    assert np.all((scores > 0.5) == (logits > 0))


def test_sigmoid_closed_forms():
    """sigmoid(0) = 0.5 exactly; sigmoid(ln 3) = 3/4; all-zero weights -> sigmoid(b_out)."""
    _, s0 = O.mlp_forward(H.zero_model([4, 8, 1]), np.random.default_rng(0).normal(size=(16, 4)))
    assert np.all(s0 == 0.5)
    _, s1 = O.mlp_forward(H.zero_model([4, 8, 1], out_bias=np.float32(math.log(3.0))), np.zeros((3, 4)))
    assert np.allclose(s1, 0.75, rtol=0, atol=1e-7)   # ln 3 rounded to fp32: |d score| <= 3/16 * 6e-8


def test_relu_identity_single_unit():
    """relu([-1, 2]) = [0, 2] through identity single-unit layers."""
    m = H.SimpleModel([1, 1, 1], [[[1.0]], [[1.0]]], [[0.0], [0.0]])
    logits, _ = O.mlp_forward(m, np.array([[-1.0], [2.0], [0.0]]))
    assert logits.tolist() == [0.0, 2.0, 0.0]


def test_logistic_regression_no_hidden_layer():
    """Zero hidden layers: logit = w.x + b exactly; score > 0.5 <=> w.x + b > 0."""
    m = H.SimpleModel([2, 1], [[[1.0, -1.0]]], [[0.5]])
    x = np.array([[3, 1], [1, 3], [2, 2.5], [-1, -1]], np.float64)
    logits, scores = O.mlp_forward(m, x)
    assert logits.tolist() == [2.5, -1.5, 0.0, 0.5]
    assert scores[2] == 0.5


def test_bf16_rne_matches_torch():
    """Diagnostic bf16 rounding == torch's fp32->bf16 (round-to-nearest-even) conversion."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.normal(size=2000).astype(np.float32) * 1000,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.005859375, 3.0e38, -2.5, 1e-30], np.float32)])
    ref = torch.from_numpy(v).to(torch.bfloat16).to(torch.float32).numpy()
    got = np.array([O.bf16_rne(float(x)) for x in v], np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


# ----------------------------------------------------------------------------------------- query
def _tiny():
    g = H.golden("tiny_query.json")
    w = H.golden("mlp_worked.json")
    cfg = D.QueryConfig("tiny", 0.0, w["dims"], [(s, c) for s, c in g["features"]],
                        [("dim", "fact", "f_key", "d_key")], group=tuple(g["group"]), ngroups=g["ngroups"],
                        sum_col=tuple(g["sum_col"]))
    fact = {k: np.array(v, np.int32) for k, v in g["fact"].items()}
    dim = {k: np.array(v, np.int32) for k, v in g["dim"].items()}
    db = D.Database(0.0, len(fact["f_key"]), fact, [("dim", len(dim["d_key"]), dim)])
    return g, cfg, db, H.SimpleModel(w["dims"], w["W"], w["b"])


def test_tiny_query_golden():
    """Hand-worked join -> classifier -> predicate -> GROUP BY (tests/golden/tiny_query.json)."""
    g, cfg, db, m = _tiny()
    r = O.run(cfg, db, m, per_row=True)
    assert r.match[:, 0].tolist() == g["match"]
    assert r.rows_joined == g["joined"]
    lg = [None if np.isnan(x) else x for x in r.logit]
    assert lg == g["logit"]
    assert r.count.tolist() == g["count"] and r.sum.tolist() == g["sum"]
    assert r.count_rej.tolist() == g["count_rej"] and r.sum_rej.tolist() == g["sum_rej"]


def test_tiny_query_normalised_golden():
    """The same hand-worked query with a non-unit dyadic normalisation x = (v - shift) * scale on a
    fact feature and a dimension feature (reading Q4) and threshold sigmoid(15)
    (tests/golden/tiny_query_norm.json): catches a divided scale, an added shift, a shift applied
    after the scale, or the normalisation dropped for build-side features."""
    g0, cfg, db, m = _tiny()
    g = H.golden("tiny_query_norm.json")
    m.shift = np.array(g["shift"], np.float32)
    m.scale = np.array(g["scale"], np.float32)
    t = 1.0 / (1.0 + math.exp(-g["threshold_logit"]))
    r = O.run(cfg, db, m, per_row=True, threshold=t)
    assert r.match[:, 0].tolist() == g0["match"]
    assert [None if np.isnan(x) else x for x in r.logit] == g["logit"]
    assert r.count.tolist() == g["count"] and r.sum.tolist() == g["sum"]
    assert r.count_rej.tolist() == g["count_rej"] and r.sum_rej.tolist() == g["sum_rej"]


def test_emulate_bf16_gather_rounding():
    """The diagnostic bf16 emulation's gather: x = bf16_rne((v - shift) * scale), pinned on values whose
    normalised form is exact in fp32 and falls on or between bf16 steps (ulp 2 at 256): 257 is a tie ->
    256 (even), 259 a tie -> 260, 258 exact. The fp64 path keeps 257 / 259 / 258. Logistic regression
    (no hidden layer), so logit = x."""
    cfg = D.QueryConfig("e", 0.0, [1, 1], [("fact", "v")], [("dim", "fact", "k", "dk")], group=("fact", "g"),
                        ngroups=1, sum_col=("fact", "g"), threshold=-math.inf)
    fact = {"k": np.array([1, 1, 1], np.int32), "g": np.zeros(3, np.int32), "v": np.array([513, 517, 515], np.int32)}
    db = D.Database(0, 3, fact, [("dim", 1, {"dk": np.array([1], np.int32)})])
    m = H.SimpleModel([1, 1], [[[1.0]]], [[0.0]], shift=[-1.0], scale=[0.5])
    assert O.run(cfg, db, m, per_row=True).logit.tolist() == [257.0, 259.0, 258.0]
    assert O.run(cfg, db, m, per_row=True, emulate_bf16=True).logit.tolist() == [256.0, 260.0, 258.0]


def test_spec_join_examples():
    """R={(1,a),(2,b)} ⋈ S={(2,x),(3,y)} -> (2,b,x); empty build side -> no rows."""
    _, cfg, _, _ = _tiny()
    cfg = D.QueryConfig("j", 0.0, [1, 1], [("fact", "f_v")], [("dim", "fact", "f_key", "d_key")],
                        group=(0, "d_g"), ngroups=2, sum_col=("fact", "f_v"), threshold=-math.inf)
    m = H.SimpleModel([1, 1], [[[0.0]]], [[0.0]])
    fact = {"f_key": np.array([2, 3], np.int32), "f_v": np.array([7, 9], np.int32)}   # S (probe side)
    dim = {"d_key": np.array([1, 2], np.int32), "d_g": np.array([0, 1], np.int32)}     # R (build side)
    r = O.run(cfg, D.Database(0, 2, fact, [("dim", 2, dim)]), m, per_row=True)
    assert r.match[:, 0].tolist() == [1, -1] and r.rows_joined == 1
    assert r.count.tolist() == [0, 1] and r.sum.tolist() == [0, 7]
    empty = {"d_key": np.zeros(0, np.int32), "d_g": np.zeros(0, np.int32)}
    r = O.run(cfg, D.Database(0, 2, fact, [("dim", 0, empty)]), m)
    assert r.rows_joined == 0 and r.count.tolist() == [0, 0]


def test_spec_groupby_example():
    """{(1,10),(1,5),(2,7)} -> {(1,15),(2,7)} (threshold -INF selects every joined row)."""
    cfg = D.QueryConfig("g", 0.0, [1, 1], [("fact", "v")], [("dim", "fact", "k", "dk")], group=("fact", "g"),
                        ngroups=3, sum_col=("fact", "v"), threshold=-math.inf)
    fact = {"k": np.array([1, 1, 1], np.int32), "g": np.array([1, 1, 2], np.int32),
            "v": np.array([10, 5, 7], np.int32)}
    dim = {"dk": np.array([1], np.int32)}
    r = O.run(cfg, D.Database(0, 3, fact, [("dim", 1, dim)]), H.zero_model([1, 1]))
    assert r.sum.tolist() == [0, 15, 7] and r.count.tolist() == [0, 2, 1]


def test_duplicate_build_key_is_error():
    cfg = D.QueryConfig("d", 0.0, [1, 1], [("fact", "v")], [("dim", "fact", "k", "dk")], group=("fact", "v"),
                        ngroups=1, sum_col=("fact", "v"))
    fact = {"k": np.array([1], np.int32), "v": np.array([0], np.int32)}
    dim = {"dk": np.array([4, 4], np.int32)}
    with pytest.raises(O.OracleError, match="duplicate build key"):
        O.run(cfg, D.Database(0, 1, fact, [("dim", 2, dim)]), H.zero_model([1, 1]))


def test_arity_mismatch_is_error():
    """The UDF signature must align with its arguments."""
    g, cfg, db, m = _tiny()
    cfg.feats = cfg.feats[:2]
    with pytest.raises(O.OracleError, match="feature count"):
        O.run(cfg, db, m)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_join_matches_nested_loop(seed):
    """Random small tables (≤1000 rows) with misses: oracle join ids == nested-loop join."""
    rng = np.random.default_rng(seed)
    nb, nf = int(rng.integers(1, 300)), int(rng.integers(1, 1000))
    bkeys = rng.choice(np.arange(-5000, 5000), size=nb, replace=False).astype(np.int32)
    fkeys = rng.choice(np.concatenate([bkeys, rng.integers(-6000, 6000, size=nb).astype(np.int32)]), size=nf)
    fkeys = fkeys.astype(np.int32)
    cfg = D.QueryConfig("r", 0.0, [1, 1], [("fact", "k")], [("dim", "fact", "k", "dk")], group=(0, "dg"),
                        ngroups=4, sum_col=("fact", "v"), threshold=-math.inf)
    fact = {"k": fkeys, "v": rng.integers(-1000, 1000, nf).astype(np.int32)}
    dim = {"dk": bkeys, "dg": rng.integers(0, 4, nb).astype(np.int32)}
    r = O.run(cfg, D.Database(0, nf, fact, [("dim", nb, dim)]), H.zero_model([1, 1]), per_row=True)
    expect = []
    for i in range(nf):                      # nested loop, first (only) match
        hit = -1
        for j in range(nb):
            if bkeys[j] == fkeys[i]:
                hit = j
                break
        expect.append(hit)
    assert r.match[:, 0].tolist() == expect
    cnt = np.zeros(4, np.int64)
    sm = np.zeros(4, np.int64)
    for i, j in enumerate(expect):
        if j >= 0:
            cnt[dim["dg"][j]] += 1
            sm[dim["dg"][j]] += fact["v"][i]
    assert r.count.tolist() == cnt.tolist() and r.sum.tolist() == sm.tolist()


def test_two_probe_chain_matches_sorted_search():
    """Config-3 join chain lineitem⋈orders⋈customer (reading Q14) vs sorted-array search."""
    cfg, db = H.small_db("c3", sf=0.002, match_rate=0.9)
    model = H.linear_threshold_model(cfg)
    r = O.run(cfg, db, model, per_row=True, threshold=-math.inf)
    match, alive = H.chain_matches(cfg, db)
    assert np.array_equal(r.match, match)
    assert r.rows_joined == int(alive.sum())


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_linear_threshold_model_is_exact_filter(name):
    """Pin (iii): with the linear-threshold model the whole query is `l_quantity >= 26` over the
    join, checked bit-exactly against an independent numpy filter-join-aggregate."""
    sf = 0.05 if name == "c4" else 0.004
    cfg, db = H.small_db(name, sf=sf, match_rate=0.9)
    model = H.linear_threshold_model(cfg)
    r = O.run(cfg, db, model, per_row=True)
    match, alive = H.chain_matches(cfg, db)
    q = db.fact["l_quantity"]
    assert np.array_equal(r.selected, alive & (q >= 26))
    assert np.all(np.abs(r.logit[alive] - (q[alive] - 25.5)) == 0)
    assert r.rows_band == 0
    cnt, sm = H.brute_aggregate(cfg, db, q >= 26)
    assert r.count.tolist() == cnt.tolist() and r.sum.tolist() == sm.tolist()


def test_threshold_extremes_and_conservation():
    """-INF selects every joined row (sum == Σ extprice over the join); +INF selects none;
    count(score > t) + count(score <= t) == joined, per group."""
    cfg, db = H.small_db("c1", sf=0.004, match_rate=0.9)
    model = D.make_model(cfg, db)
    match, alive = H.chain_matches(cfg, db)
    cnt_all, sum_all = H.brute_aggregate(cfg, db, np.ones(db.fact_n, bool))
    lo = O.run(cfg, db, model, threshold=-math.inf)
    assert lo.count.tolist() == cnt_all.tolist() and lo.sum.tolist() == sum_all.tolist()
    assert lo.rows_joined == int(alive.sum())
    hi = O.run(cfg, db, model, threshold=math.inf)
    assert hi.count.sum() == 0 and hi.sum.sum() == 0
    mid = O.run(cfg, db, model)
    assert (mid.count + mid.count_rej).tolist() == cnt_all.tolist()
    assert (mid.sum + mid.sum_rej).tolist() == sum_all.tolist()


def test_strict_threshold_at_tie():
    """`*y2 > 0.5` is strict: a score of exactly 0.5 is not selected."""
    cfg, db = H.small_db("c1", sf=0.002)
    r = O.run(cfg, db, H.zero_model(cfg.dims))
    assert r.rows_selected == 0 and r.rows_band == r.rows_joined


def test_permutation_and_shard_invariance():
    """Shuffling fact rows leaves the aggregates bit-identical; summing the results of
    contiguous row ranges (and of generator shards) equals the unsharded result."""
    cfg, db = H.small_db("c1", sf=0.004, match_rate=0.9)
    model = D.make_model(cfg, db)
    full = O.run(cfg, db, model)
    dbs = D.make_database(cfg, shuffle_seed=7)
    sh = O.run(cfg, dbs, model)
    assert sh.count.tolist() == full.count.tolist() and sh.sum.tolist() == full.sum.tolist()
    cut = db.fact_n // 3
    a = O.run(cfg, db, model, row_lo=0, row_hi=cut)
    b = O.run(cfg, db, model, row_lo=cut, row_hi=db.fact_n)
    assert (a.count + b.count).tolist() == full.count.tolist()
    assert (a.sum + b.sum).tolist() == full.sum.tolist()
    parts = [O.run(cfg, D.make_database(cfg, rank=r, world=3), model) for r in range(3)]
    assert sum(p.count for p in parts).tolist() == full.count.tolist()
    assert sum(p.sum for p in parts).tolist() == full.sum.tolist()


def test_prefilter_is_scalar_filter():
    """Config-4 pre-filter `lo <= l_shipdate < hi` keeps exactly the rows an independent
    comparison keeps; aggregates at -INF equal the brute-force filter-join-aggregate."""
    cfg, db = H.small_db("c4p", sf=0.05, match_rate=1.0)
    model = H.linear_threshold_model(cfg)
    r = O.run(cfg, db, model, threshold=-math.inf)
    c, lo, hi = cfg.prefilter
    keep = (db.fact[c] >= lo) & (db.fact[c] < hi)
    assert r.rows_prefiltered == int(keep.sum())
    assert 0.015 < keep.mean() < 0.03   # ~2% selectivity (config 4)
    cnt, sm = H.brute_aggregate(cfg, db, keep)
    assert r.count.tolist() == cnt.tolist() and r.sum.tolist() == sm.tolist()


def test_emulate_bf16_close_to_fp64():
    """The diagnostic bf16 emulation stays within the bf16 budget of the fp64 oracle."""
    cfg, db = H.small_db("c1", sf=0.004)
    model = D.make_model(cfg, db)
    a = O.run(cfg, db, model, per_row=True)
    b = O.run(cfg, db, model, per_row=True, emulate_bf16=True)
    ok = ~np.isnan(a.score)
    assert np.nanmax(np.abs(a.score[ok] - b.score[ok])) < 1e-2


def test_multithreaded_equals_single_thread():
    cfg, db = H.small_db("c1", sf=0.01)
    model = D.make_model(cfg, db)
    a = O.run(cfg, db, model, nthreads=1, per_row=True)
    b = O.run(cfg, db, model, nthreads=5, per_row=True)
    assert a.count.tolist() == b.count.tolist() and a.sum.tolist() == b.sum.tolist()
    assert np.array_equal(a.score, b.score, equal_nan=True)


# ------------------------------------------------------------------- NEXT-4: chains, duplicate keys
def test_spec_multimap_example():
    """duplicate left keys {(2,b),(2,c)} ⋈ {(2,x)} -> (2,b,x), (2,c,x): the probe emits every
    match (P:328-331 iterates map(rightHash(rTuple))). Group by the build row, sum the fact value."""
    cfg = D.QueryConfig("m", 0.0, [1, 1], [("fact", "v")], [("dim", "fact", "k", "dk")], group=(0, "dg"),
                        ngroups=3, sum_col=("fact", "v"), threshold=-math.inf, multi=(0,))
    fact = {"k": np.array([2, 5], np.int32), "v": np.array([7, 11], np.int32)}
    dim = {"dk": np.array([2, 2, 9], np.int32), "dg": np.array([0, 1, 2], np.int32)}   # b, c, (no match)
    r = O.run(cfg, D.Database(0, 2, fact, [("dim", 3, dim)]), H.zero_model([1, 1]))
    assert r.rows_joined == 2 and r.count.tolist() == [1, 1, 0] and r.sum.tolist() == [7, 7, 0]
    with pytest.raises(O.OracleError, match="per-row exports need unique build keys"):
        O.run(cfg, D.Database(0, 2, fact, [("dim", 3, dim)]), H.zero_model([1, 1]), per_row=True)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("dup", [True, False])
def test_chain_and_duplicate_keys_match_sorted_expansion(seed, dup):
    """Three probes (fact->A with repeating keys when `dup`, A->B, fact->C), threshold -INF: joined tuple
    count and per-group aggregates equal the vectorised sorted-search expansion (tests/helpers.expand_join);
    with a model selecting on a build-side feature (relu(b_q - 24.5) - relu(24.5 - b_q) > 0, i.e. b_q >= 25)
    the selected aggregates equal the expansion filtered on B's column: each tuple's features come from its
    own build rows."""
    cfg, db = H.star_chain_db(seed, dup=dup)
    fr, br = H.expand_join(cfg, db)
    assert len(fr) > 100 and (not dup or len(fr) > len(np.unique(fr)))
    r = O.run(cfg, db, H.zero_model(cfg.dims), threshold=-math.inf)
    cnt, sm = H.tuple_aggregate(cfg, db, fr, br, np.ones(len(fr), bool))
    assert r.rows_joined == len(fr) and r.count.tolist() == cnt.tolist() and r.sum.tolist() == sm.tolist()
    k = cfg.feats.index((1, "b_q"))
    W1 = np.zeros((64, 8), np.float32)
    W1[0, k], W1[1, k] = 1.0, -1.0
    w2 = np.zeros((1, 64), np.float32)
    w2[0, 0], w2[0, 1] = 1.0, -1.0
    shift = np.zeros(8, np.float32)
    shift[k] = 24.5
    m = H.SimpleModel(cfg.dims, [W1, w2], [np.zeros(64), np.zeros(1)], shift=shift)
    r = O.run(cfg, db, m)
    q = H.tuple_column(cfg, db, (1, "b_q"), fr, br)
    cnt, sm = H.tuple_aggregate(cfg, db, fr, br, q >= 25)
    assert r.rows_band == 0 and r.count.tolist() == cnt.tolist() and r.sum.tolist() == sm.tolist()


def test_three_probe_chain_join_ids_match_sorted_search():
    """Unique keys on every probe: per-row join ids of the 3-probe chain equal a sorted-array search per
    probe (helpers.chain_matches)."""
    cfg, db = H.star_chain_db(3, dup=False)
    r = O.run(cfg, db, H.zero_model(cfg.dims), per_row=True, threshold=-math.inf)
    match, alive = H.chain_matches(cfg, db)
    assert np.array_equal(r.match, match) and r.rows_joined == int(alive.sum()) > 100
