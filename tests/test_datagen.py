"""Input generator properties (SPEC S:582-590 ideas): determinism, shards, match rate, shape."""
import numpy as np

import datagen as D


def test_same_seed_same_bytes():
    a = D.gen_lineitem(0.01, ["l_orderkey", "l_quantity", "l_f0"])[1]
    b = D.gen_lineitem(0.01, ["l_orderkey", "l_quantity", "l_f0"], nthreads=3)[1]
    for k in a:
        assert a[k].tobytes() == b[k].tobytes()
    c = D.gen_lineitem(0.01, ["l_quantity"], seed=D.SEED + 1)[1]
    assert c["l_quantity"].tobytes() != a["l_quantity"].tobytes()


def test_shards_concatenate_to_full_table():
    cols = ["l_orderkey", "l_extendedprice", "l_shipdate"]
    n, full = D.gen_lineitem(0.01, cols)
    parts = [D.gen_lineitem(0.01, cols, *D.shard_slots(0.01, r, 4))[1] for r in range(4)]
    for c in cols:
        assert np.array_equal(np.concatenate([p[c] for p in parts]), full[c])


def test_orders_keys_unique_sparse_and_lineitem_clustered():
    m, o = D.gen_orders(0.01, ["o_orderkey"])
    k = o["o_orderkey"]
    assert len(np.unique(k)) == m == D.num_order_slots(0.01)
    assert k[7] == 8 and k[8] == 33            # TPC-H sparse keys: 8 dense, then a gap of 24
    n, l = D.gen_lineitem(0.01, ["l_orderkey", "l_linenumber"])
    assert np.all(np.diff(l["l_orderkey"]) >= 0)      # dbgen order (clustered by orderkey)
    assert 3.5 < n / m < 4.5                          # 1..7 lines per order


def test_match_rate_controls_join_cardinality():
    _, o0 = D.gen_orders(0.01, ["o_orderkey"], match_rate=0.0)
    assert len(o0["o_orderkey"]) == 0
    _, o9 = D.gen_orders(0.01, ["o_orderkey"], match_rate=0.9)
    assert 0.88 < len(o9["o_orderkey"]) / D.num_order_slots(0.01) < 0.92
    n, l = D.gen_lineitem(0.01, ["l_orderkey"])
    _, o1 = D.gen_orders(0.01, ["o_orderkey"], match_rate=1.0)
    assert np.isin(l["l_orderkey"], o1["o_orderkey"]).all()   # |L ⋈ O| = |L| at m = 1


def test_value_ranges():
    n, l = D.gen_lineitem(0.01, ["l_quantity", "l_extendedprice", "l_discount", "l_shipdate", "l_receiptdate",
                                 "l_returnflag", "l_f3"])
    assert l["l_quantity"].min() >= 1 and l["l_quantity"].max() <= 50
    assert l["l_extendedprice"].min() > 0
    assert (l["l_receiptdate"] > l["l_shipdate"]).all()
    assert set(np.unique(l["l_returnflag"])) <= {0, 1, 2}
    assert abs(float(l["l_f3"].mean())) < 0.05 and abs(float(l["l_f3"].std()) - 1) < 0.05
    m, c = D.gen_customer(0.01, ["c_custkey", "c_acctbal", "c_mktsegment"])
    assert np.array_equal(c["c_custkey"], np.arange(1, m + 1))
    _, o = D.gen_orders(0.01, ["o_custkey"])
    assert (o["o_custkey"] % 3 != 0).all() and o["o_custkey"].max() <= m


def test_model_weights_bf16_exact_and_seeded():
    cfg = D.with_sf(D.CONFIGS["c2"], 0.002)
    db = D.make_database(cfg)
    m1 = D.make_model(cfg, db)
    m2 = D.make_model(cfg, db)
    for w1, w2 in zip(m1.W, m2.W):
        assert np.array_equal(w1, w2)
        assert np.array_equal(D.bf16_round(w1), w1)
    assert [w.shape for w in m1.W] == [(256, 16), (256, 256), (1, 256)]
