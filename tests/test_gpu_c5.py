"""Config 5 at its full size on one GPU (`-m gpu`, slow): SF100, 600M lineitem rows, lineitem ⋈ orders,
16-256-256-1, in the launch configuration `bench.py --workload c5` times at N=1 (the whole shard in one
flern_run_query, the fact table and the replicated orders table generated chunk by chunk into HBM).

  - join ids, scores and selection on sampled slot ranges against the oracle: the oracle gets the lineitem
    rows of the sampled order slots and the orders rows of the same slots (match rate 1: a line's order is
    in its own slot, so the restricted build side gives the same join; orders row id = slot id);
  - aggregates at threshold -INF exact against an independent chunked numpy join-aggregate over all 600M
    rows (sorted-array search, bincount)."""
import math

import numpy as np
import pytest

import datagen as D
import oracle as O
from tests import helpers as H
from tests import parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c5():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from datagen import device as DD
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = D.CONFIGS["c5"]
    S = D.num_order_slots(cfg.sf)
    n, fact = DD.fact_to_device(cfg, 0, S, "cuda:0")
    db = D.Database(cfg.sf, n, fact, DD.builds_to_device(cfg, "cuda:0"))
    model = D.make_model(cfg, D.make_database(cfg, max_slots=D.MODEL_SLOTS))
    gq = GpuQuery(cfg, db, model, load_fact=False)
    gq.set_fact(F.flern_load_table(gq.ctx, "fact", fact, F.FLERN_BORROW_DEVICE))
    yield cfg, db, model, gq, S
    gq.close()


def test_c5_sf100_sampled_rows(c5):
    import torch
    from paper_2311_02781_b200 import flern as F
    from datagen import device as DD
    cfg, db, model, gq, S = c5
    n, G = db.fact_n, cfg.ngroups
    assert n > 599_000_000
    dev = "cuda:0"
    score = torch.empty(n, dtype=torch.float32, device=dev)
    match = torch.empty(n, dtype=torch.int32, device=dev)
    sel = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    cnt = torch.zeros(G, dtype=torch.int64, device=dev)
    sm = torch.zeros(G, dtype=torch.int64, device=dev)
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    gq.run(gq.make_query(gq.fact_id, flags=F.FLERN_Q_RESULT_DEVICE), count=cnt, sum=sm, counters=ctr,
           dbg_score=score, dbg_match=match, dbg_selected=sel)
    torch.cuda.synchronize()
    assert int(ctr[0]) == n and int(ctr[1]) == n   # match rate 1: every line joins its order
    rng = np.random.default_rng(100)
    starts = [0, S - 300] + sorted(rng.integers(0, S - 300, size=6).tolist())
    worst = 0.0
    for a in starts:
        b = a + 300
        row0 = DD.lineitem_rows(cfg.sf, 0, a)
        m, lf = D.gen_lineitem(cfg.sf, cfg.fact_cols(), a, b)
        mo, of = D.gen_orders(cfg.sf, cfg.build_cols(0), slot_lo=a, slot_hi=b)
        sub = D.Database(cfg.sf, m, lf, [("orders", mo, of)])
        o = O.run(cfg, sub, model, band=parity.BAND, per_row=True)
        gm = match[row0:row0 + m].cpu().numpy()
        assert np.array_equal(gm, (o.match[:, 0] + a).astype(np.int32)), a
        gs = score[row0:row0 + m].cpu().numpy().astype(np.float64)
        worst = max(worst, float(np.abs(gs - o.score).max()))
        bits = sel.cpu().numpy().view(np.uint32)
        gsel = parity.unpack_bits(bits, n)[row0:row0 + m]
        outside = np.abs(o.score - cfg.threshold) > parity.BAND
        assert np.array_equal(gsel[outside], o.selected[outside]), a
    assert worst <= parity.SCORE_TOL, worst


def test_c5_sf100_aggregates_at_minus_inf(c5):
    cfg, db, model, gq, S = c5
    G = cfg.ngroups
    cnt, sm = np.zeros(G, np.int64), np.zeros(G, np.int64)
    r = gq.run(gq.make_query(gq.fact_id, threshold=-math.inf), count=cnt, sum=sm)
    assert r.rows_joined == db.fact_n
    ref_c, ref_s = np.zeros(G, np.int64), np.zeros(G, np.int64)
    step = 5_000_000
    for a in range(0, S, step):
        b = min(S, a + step)
        _, lf = D.gen_lineitem(cfg.sf, ["l_orderkey", "l_extendedprice"], a, b)
        _, of = D.gen_orders(cfg.sf, ["o_orderkey", "o_orderpriority"], slot_lo=a, slot_hi=b)
        j = H.join_sorted(lf["l_orderkey"], of["o_orderkey"])
        assert (j >= 0).all()
        g = of["o_orderpriority"][j].astype(np.int64)
        ref_c += np.bincount(g, minlength=G)[:G]
        # per-chunk sums < 2^53: exact in the fp64 bincount
        ref_s += np.bincount(g, weights=lf["l_extendedprice"].astype(np.float64), minlength=G)[:G].astype(np.int64)
    assert cnt.tolist() == ref_c.tolist() and sm.tolist() == ref_s.tolist()
