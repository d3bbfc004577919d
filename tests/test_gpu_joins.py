"""NEXT-4 on the GPU (`-m gpu`): join chains beyond the fused kernel's own probes and build sides whose
keys repeat (multimap), through the C ABI, against the oracle and an independent sorted-search expansion
(tests/helpers.expand_join). The paper's probe emits every match; its data-manipulation
workload is a six-table natural join.

The schema (helpers.star_chain_db): fact F probes A on k_a (A's keys repeat: up to ~3 rows per key), A's
a_b probes B, and F's k_c probes C: a 3-probe star/snowflake, expanded into joined tuples
(join_kernel.cuh) that the fused gather -> MLP -> predicate -> group-by kernel then consumes."""
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


def _bq_model(cfg):
    """relu(b_q - 24.5) - relu(24.5 - b_q) > 0 <=> b_q >= 25 (B's column, two probes deep): exact in bf16,
    no tuple near the threshold, so selection and aggregates are bit-exact; every hidden layer passes
    units 0 and 1 through (the linear-threshold pin of SURVEY.md §8(c), on a build-side feature)."""
    dims = cfg.dims
    k = cfg.feats.index((1, "b_q"))
    L = len(dims) - 1
    W = [np.zeros((dims[l + 1], dims[l]), np.float32) for l in range(L)]
    b = [np.zeros(dims[l + 1], np.float32) for l in range(L)]
    W[0][0, k], W[0][1, k] = 1.0, -1.0
    for l in range(1, L - 1):
        W[l][0, 0], W[l][1, 1] = 1.0, 1.0
    W[L - 1][0, 0], W[L - 1][0, 1] = 1.0, -1.0
    shift = np.zeros(dims[0], np.float32)
    shift[k] = 24.5
    return H.SimpleModel(dims, W, b, shift=shift)


def _random_model(cfg, db):
    m = D.make_model(cfg, db, out_scale=0.25, out_shift=0.0)
    return m


DIMS = [[8, 64, 1], [8, 128, 128, 1], [8, 512, 512, 1]]


@pytest.mark.parametrize("dims", DIMS, ids=["nl1", "nl2", "wide"])
@pytest.mark.parametrize("dup", [True, False], ids=["multimap", "unique"])
def test_three_probe_chain(dims, dup):
    import dataclasses
    cfg, db = H.star_chain_db(5, nfact=6000, dup=dup)
    cfg = dataclasses.replace(cfg, dims=dims)
    fr, br = H.expand_join(cfg, db)
    assert len(fr) > (1000 if dup else 500) and (not dup or len(fr) > len(np.unique(fr)))
    # exact: the build-side threshold model
    m = _bq_model(cfg)
    g = parity.run_gpu(cfg, db, m, debug=False)
    q = H.tuple_column(cfg, db, (1, "b_q"), fr, br)
    cnt, sm = H.tuple_aggregate(cfg, db, fr, br, q >= 25)
    o = O.run(cfg, db, m)
    assert o.rows_band == 0 and o.count.tolist() == cnt.tolist() and o.sum.tolist() == sm.tolist()
    assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()
    assert g["rows_joined"] == len(fr) and g["rows_scanned"] == db.fact_n
    # threshold -INF: every joined tuple
    g = parity.run_gpu(cfg, db, m, threshold=-math.inf, debug=False)
    cnt, sm = H.tuple_aggregate(cfg, db, fr, br, np.ones(len(fr), bool))
    assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()
    # a random model: the band bracket against the oracle, and conservation over both classes
    m = _random_model(cfg, db)
    g = parity.run_gpu(cfg, db, m, both=True, debug=False)
    o = O.run(cfg, db, m, band=parity.BAND)
    c = g["count"]
    assert np.all(o.count_hi <= c) and np.all(c <= o.count_hi + o.count_band)
    assert np.all(o.sum_hi <= g["sum"]) and np.all(g["sum"] <= o.sum_hi + o.sum_band)
    assert (g["count"] + g["count_rej"]).tolist() == cnt.tolist()
    assert (g["sum"] + g["sum_rej"]).tolist() == sm.tolist()
    assert 0 < o.rows_selected < o.rows_joined


def test_multimap_with_prefilter_and_streaming():
    """The expansion applies the pre-filter; a streamed query (host rows through the ring) expands chunk by
    chunk and sums to the resident result."""
    import dataclasses
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg, db = H.star_chain_db(7, nfact=20000, dup=True)
    cfg = dataclasses.replace(cfg, prefilter=("ship", 10, 60))
    m = _bq_model(cfg)
    fr, br = H.expand_join(cfg, db)
    q = H.tuple_column(cfg, db, (1, "b_q"), fr, br)
    cnt, sm = H.tuple_aggregate(cfg, db, fr, br, q >= 25)
    g = parity.run_gpu(cfg, db, m, debug=False)
    assert g["count"].tolist() == cnt.tolist() and g["sum"].tolist() == sm.tolist()
    gq = GpuQuery(cfg, db, m)
    try:
        c, s_ = np.zeros(cfg.ngroups, np.int64), np.zeros(cfg.ngroups, np.int64)
        r = F.flern_run_query_streamed(gq.ctx, gq.query, db.fact, 3000, count=c, sum=s_)
        assert c.tolist() == cnt.tolist() and s_.tolist() == sm.tolist()
        assert r.rows_scanned == db.fact_n and r.rows_joined == len(fr)
    finally:
        gq.close()


def test_multimap_build_errors_and_exports():
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg, db = H.star_chain_db(2, nfact=500, dup=True)
    gq = GpuQuery(cfg, db, _bq_model(cfg))
    try:
        tid = F.flern_load_table(gq.ctx, "dupk", {"k": np.array([3, 1, 3, np.iinfo(np.int32).min], np.int32)})
        with pytest.raises(F.FlernError, match="INT32_MIN"):
            F.flern_build_hashtable_ex(gq.ctx, tid, "k", [], F.FLERN_HT_MULTI)
        tid = F.flern_load_table(gq.ctx, "dupk2", {"k": np.array([3, 1, 3], np.int32)})
        with pytest.raises(F.FlernError, match="DUP_KEY"):
            F.flern_build_hashtable(gq.ctx, tid, "k", [])
        with pytest.raises(F.FlernError, match="expanded joins"):   # per-row exports are per fact row
            parity.run_gpu(cfg, db, gq=gq, model=None, debug=True)
    finally:
        gq.close()
