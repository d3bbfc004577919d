"""Pins of the oracle's training step (NEXT-3: ML-in-charge, §4.5), CPU only.

 - hand-worked dyadic SGD step (tests/golden/train_worked.json)           -> wrong sign, missing 2/n,
                                                                            transposed dW, ReLU'(0)
 - central finite differences of the loss computed with the oracle's (separately pinned) forward pass
   (or_mlp_forward) against the analytic gradients of every parameter    -> any backward mistake
 - a least-squares fit (numpy lstsq) has zero gradient under a linear model (no hidden layer)
 - an SGD step with a small learning rate lowers the loss; lr = 0 leaves the weights unchanged
 - the batch export: the tuples the query yields, in order, with their targets
"""
import numpy as np
import pytest

import datagen as D
import oracle as O
from tests import helpers as H


def test_train_step_worked_example_exact():
    g = H.golden("train_worked.json")
    m = H.SimpleModel(g["dims"], g["W"], g["b"])
    r = O.mlp_train_step(m, np.array(g["x"], np.float64), np.array(g["t"], np.float64), g["lr"])
    assert r["loss"] == g["loss"]
    for l in range(2):
        assert r["dW"][l].tolist() == g["dW"][l] and r["db"][l].tolist() == g["db"][l]
        assert r["W"][l].tolist() == g["W_new"][l] and r["b"][l].tolist() == g["b_new"][l]


def _loss(model, X, T):
    _, _ = None, None
    logits, _ = O.mlp_forward(model, X)   # the pinned forward pass; the output layer is linear
    return float(np.mean((logits - T) ** 2))


@pytest.mark.parametrize("dims", [[3, 5, 1], [4, 6, 5, 1]])
def test_gradients_match_central_differences(dims):
    rng = np.random.default_rng(len(dims))
    L = len(dims) - 1
    W = [rng.normal(size=(dims[l + 1], dims[l])).astype(np.float32) for l in range(L)]
    b = [rng.normal(size=dims[l + 1]).astype(np.float32) * 0.3 for l in range(L)]
    X = rng.normal(size=(17, dims[0]))
    T = rng.normal(size=17)
    r = O.mlp_train_step(H.SimpleModel(dims, W, b), X, T, 0.0)
    for l in range(L):
        for kind, P, G in (("W", W, r["dW"]), ("b", b, r["db"])):
            flat = P[l].reshape(-1)
            for e in range(flat.size):
                eps = np.float32(2.0 ** -12)
                saved = flat[e]
                flat[e] = saved + eps
                lp = _loss(H.SimpleModel(dims, W, b), X, T)
                up = flat[e]
                flat[e] = saved - eps
                lm = _loss(H.SimpleModel(dims, W, b), X, T)
                dn = flat[e]
                flat[e] = saved
                num = (lp - lm) / (float(up) - float(dn))
                ana = G[l].reshape(-1)[e]
                assert abs(num - ana) <= 1e-4 * max(1.0, abs(ana)), (kind, l, e, num, ana)


def test_least_squares_fit_has_zero_gradient():
    """Linear regression (no hidden layer): at numpy's least-squares solution the MSE gradient vanishes."""
    rng = np.random.default_rng(4)
    X = rng.normal(size=(200, 3))
    T = X @ np.array([0.5, -2.0, 1.25]) + 0.75 + rng.normal(size=200) * 0.1
    A = np.hstack([X, np.ones((200, 1))])
    sol = np.linalg.lstsq(A, T, rcond=None)[0]
    # the oracle model holds fp32 weights: fit the residual of the rounded weights again in fp64
    m = H.SimpleModel([3, 1], [sol[:3].astype(np.float32).reshape(1, 3)], [np.float32([sol[3]])])
    r = O.mlp_train_step(m, X, T, 0.0)
    w32 = np.concatenate([m.W[0].reshape(-1), m.b[0]]).astype(np.float64)
    expect = 2.0 / 200 * A.T @ (A @ w32 - T)   # gradient of the exact quadratic at the rounded point
    got = np.concatenate([r["dW"][0].reshape(-1), r["db"][0]])
    assert np.allclose(got, expect, rtol=0, atol=1e-10)
    assert np.abs(got).max() < 1e-5   # ~0: the fp32 rounding of the optimum only


def test_sgd_step_descends_and_zero_lr_is_identity():
    rng = np.random.default_rng(9)
    dims = [4, 8, 8, 1]
    W = [rng.normal(size=(dims[l + 1], dims[l])).astype(np.float32) * 0.5 for l in range(3)]
    b = [np.zeros(dims[l + 1], np.float32) for l in range(3)]
    X, T = rng.normal(size=(64, 4)), rng.normal(size=64)
    m = H.SimpleModel(dims, W, b)
    r0 = O.mlp_train_step(m, X, T, 0.0)
    for l in range(3):
        assert np.array_equal(r0["W"][l], W[l].astype(np.float64)) and np.array_equal(r0["b"][l], b[l].astype(np.float64))
    r = O.mlp_train_step(m, X, T, 1e-3)
    m2 = H.SimpleModel(dims, [w.astype(np.float32) for w in r["W"]], [x.astype(np.float32) for x in r["b"]])
    assert _loss(m2, X, T) < r["loss"]


def test_batch_export_is_the_query_tuples():
    """O.batch yields one row per joined tuple, fact rows in order (nested-loop order for a multimap
    chain), x = (v - shift) * scale of each feature's column and t = the sum column."""
    for dup in (False, True):
        cfg, db = H.star_chain_db(11, nfact=800, dup=dup)
        model = D.make_model(cfg, db)
        X, T = O.batch(cfg, db, model)
        fr, br = H.expand_join(cfg, db)
        assert len(T) == len(fr)
        for k, ref in enumerate(cfg.feats):
            v = H.tuple_column(cfg, db, ref, fr, br).astype(np.float64)
            assert np.array_equal(X[:, k], (v - np.float64(model.shift[k])) * np.float64(model.scale[k]))
        assert np.array_equal(T, H.tuple_column(cfg, db, cfg.sum_col, fr, br).astype(np.float64))
