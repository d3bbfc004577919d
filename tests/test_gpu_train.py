"""NEXT-3 on the GPU (`-m gpu`): the ML-in-charge training step (flern_train_step: gather -> forward ->
MSE -> backward on tcgen05 -> SGD, §4.5) against the fp64 oracle
(oracle.train_step, pinned in tests/test_oracle_train.py), on the same seeded inputs.

Tolerance: the GPU rounds x, H1, H2, dZ2, dZ1 and dy to bf16 (relative 2^-9 each) and
accumulates in fp32, so a layer's gradient matches the fp64 one to a relative Frobenius error well under
2e-2, the loss to 1e-2 relative; the gradient is recovered from the step as (W_before - W_after) / lr."""
import dataclasses

import numpy as np
import pytest

import datagen as D
import oracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu
GRAD_TOL = 2e-2
LOSS_TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _c2_train_cfg(sf=0.004):
    """C2's query (lineitem ⋈ orders, 16 features) training a 16-128-128-1 regression of l_quantity."""
    return D.with_sf(D.CONFIGS["c2"], sf, match_rate=0.9, dims=[16, 128, 128, 1], sum_col=("fact", "l_quantity"),
                     name="train")


def _model(cfg, db, out_scale=0.05):
    return D.make_model(cfg, db, out_scale=out_scale, out_shift=0.0)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(1e-30, np.linalg.norm(b)))


def _step_and_compare(cfg, db, model, lo, hi, lr):
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    gq = GpuQuery(cfg, db, model)
    try:
        q = gq.make_query(gq.fact_id)
        r = F.flern_train_step(gq.ctx, q, lo, hi, lr)
        W, b = F.flern_get_model(gq.ctx, gq.model_id, cfg.dims)
    finally:
        gq.close()
    o = O.train_step(cfg, db, model, lr, lo, hi)
    assert r.rows_joined == o["batch"] > 0
    assert abs(r.loss - o["loss"]) <= LOSS_TOL * o["loss"], (r.loss, o["loss"])
    for l in range(len(cfg.dims) - 1):
        gW = (model.W[l].astype(np.float64) - W[l]) / lr
        gb = (model.b[l].astype(np.float64) - b[l]) / lr
        assert _rel(gW, o["dW"][l]) <= GRAD_TOL, ("W", l, _rel(gW, o["dW"][l]))
        assert _rel(gb, o["db"][l]) <= GRAD_TOL, ("b", l, _rel(gb, o["db"][l]))
    return r, o, W, b


@pytest.mark.parametrize("lo,hi", [(0, 8192), (4096, 4096 + 1337), (0, -1)])
def test_train_step_matches_oracle(lo, hi):
    """One step on a batch of fact rows (many tiles, a ragged last tile, probe misses): loss and every
    layer's weight and bias gradient against the fp64 oracle."""
    cfg = _c2_train_cfg()
    db = D.make_database(cfg)
    _step_and_compare(cfg, db, _model(cfg, db), lo, hi, 1.0)


def test_train_steps_follow_the_oracle_trajectory():
    """Five steps on consecutive batches, each side updating its own weights: the GPU's weights stay within
    the tolerance of the oracle's, and the loss falls."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    cfg = _c2_train_cfg(0.01)
    db = D.make_database(cfg)
    model = _model(cfg, db)
    lr, batch = 1e-4, 8000
    gq = GpuQuery(cfg, db, model)
    ref = H.SimpleModel(cfg.dims, [w.copy() for w in model.W], [x.copy() for x in model.b], model.shift, model.scale)
    losses = []
    try:
        q = gq.make_query(gq.fact_id)
        for s in range(5):
            lo = (s * batch) % (db.fact_n - batch) // 4 * 4
            r = F.flern_train_step(gq.ctx, q, lo, lo + batch, lr)
            o = O.train_step(cfg, db, ref, lr, lo, lo + batch)
            assert abs(r.loss - o["loss"]) <= LOSS_TOL * o["loss"]
            losses.append(o["loss"])
            ref = H.SimpleModel(cfg.dims, [w.astype(np.float32) for w in o["W"]], [x.astype(np.float32) for x in o["b"]],
                                model.shift, model.scale)
        W, b = F.flern_get_model(gq.ctx, gq.model_id, cfg.dims)
    finally:
        gq.close()
    for l in range(3):
        dW_gpu, dW_ref = W[l] - model.W[l], ref.W[l] - model.W[l]
        assert _rel(dW_gpu, dW_ref) <= 3 * GRAD_TOL, (l, _rel(dW_gpu, dW_ref))
    assert losses[-1] < losses[0]


def test_train_step_on_an_expanded_join():
    """Training batches from a 3-probe chain with a multimap build side (NEXT-4 tuples): target f1."""
    cfg, db = H.star_chain_db(13, nfact=6000, dup=True)
    cfg = dataclasses.replace(cfg, dims=[8, 128, 128, 1], sum_col=("fact", "f1"), name="train_star")
    _step_and_compare(cfg, db, _model(cfg, db, 0.1), 0, 6000, 1.0)


def test_trained_model_serves_queries():
    """After a step the registered model's inference path uses the updated weights: a query's scores
    match the oracle run with the weights flern_get_model returns."""
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery
    from tests import parity
    cfg = _c2_train_cfg(0.003)
    db = D.make_database(cfg)
    model = _model(cfg, db, 0.2)
    gq = GpuQuery(cfg, db, model)
    try:
        F.flern_train_step(gq.ctx, gq.make_query(gq.fact_id), 0, -1, 1e-4)
        W, b = F.flern_get_model(gq.ctx, gq.model_id, cfg.dims)
        trained = H.SimpleModel(cfg.dims, W, b, model.shift, model.scale)
        qcfg = dataclasses.replace(cfg, sum_col=("fact", "l_extendedprice"))
        gq.query = gq.make_query(gq.fact_id)
        g = parity.run_gpu(qcfg, db, trained, gq=gq)
        # the inference kernels compute with bf16 hidden-layer weights (flern_load_model): the oracle sees
        # the trained weights rounded the same way (reading Q7)
        served = H.SimpleModel(cfg.dims, [D.bf16_round(W[0]).reshape(W[0].shape), D.bf16_round(W[1]).reshape(W[1].shape),
                                          W[2]], b, model.shift, model.scale)
        o = O.run(qcfg, db, served, per_row=True)
        ok = ~np.isnan(o.score)
        err = np.abs(g["score"][ok] - o.score[ok])
        print("serving max |score diff|", err.max(), "mean signed", float((g["score"][ok] - o.score[ok]).mean()))
        o0 = O.run(qcfg, db, model, per_row=True)
        print("untrained vs trained oracle max", np.abs(o0.score[ok] - o.score[ok]).max())
        assert err.max() <= parity.SCORE_TOL
    finally:
        gq.close()
