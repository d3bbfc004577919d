"""One small run of every kernel family through the C ABI (for compute-sanitizer): the one-layer kernel
on its lean path and with debug exports, the two-layer kernel, the pre-filter path, the wide kernel, an
expanded 3-probe join, and a training step. Checks the results against the oracle where cheap."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen as D
import oracle as O
from tests import parity, helpers as H

def agg_check(name, cfg, db, model, debug):
    g = parity.run_gpu(cfg, db, model, debug=debug)
    o = O.run(cfg, db, model, band=parity.BAND)
    ok = (g["rows_joined"] == o.rows_joined and np.all(o.count_hi <= g["count"]) and
          np.all(g["count"] <= o.count_hi + o.count_band))
    print(name, "rows", db.fact_n, "joined", g["rows_joined"], "ok", ok, flush=True)
    assert ok

for name, sf, kw in (("c1", 0.01, {}), ("c2", 0.005, {}), ("c4p", 0.05, {}), ("c3", 0.002, {})):
    cfg = D.with_sf(D.CONFIGS[name], sf, **kw)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    agg_check(name, cfg, db, model, debug=False)
    if name in ("c1", "c2"):
        parity.check(cfg, db, model)   # debug exports: per-row join ids, scores, selection
        print(name, "per-row parity ok", flush=True)
print("sanitize run done")
