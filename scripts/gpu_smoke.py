"""Quick GPU sanity run: one small C1 and C2 query vs the oracle, printing the diffs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen as D
from tests import parity

for name, sf in (("c1", 0.002), ("c2", 0.002)):
    cfg = D.with_sf(D.CONFIGS[name], sf, match_rate=0.9)
    db = D.make_database(cfg)
    model = D.make_model(cfg, db)
    t = time.time()
    g = parity.run_gpu(cfg, db, model)
    import oracle as O
    o = O.run(cfg, db, model, per_row=True)
    ok = ~np.isnan(o.score)
    print(name, "rows", db.fact_n, "joined gpu/oracle", g["rows_joined"], o.rows_joined,
          "match eq", np.array_equal(g["match"], o.match.astype(np.int32)),
          "reached eq", np.array_equal(ok, ~np.isnan(g["score"])), flush=True)
    d = np.abs(g["score"][ok] - o.score[ok])
    print("  score maxdiff", np.nanmax(d) if d.size else None, "nan in gpu", np.isnan(g["score"][ok]).sum())
    print("  gpu count", g["count"].tolist(), "oracle", o.count.tolist())
    print("  first scores gpu", g["score"][:6], "oracle", o.score[:6], flush=True)
    print("  kernel ms", g["elapsed_ms"], "wall", time.time() - t)

# error decomposition on C2: GPU vs fp64 oracle vs bf16-emulating oracle
cfg = D.with_sf(D.CONFIGS["c2"], 0.01, match_rate=1.0)
db = D.make_database(cfg)
model = D.make_model(cfg, db)
g = parity.run_gpu(cfg, db, model)
o = O.run(cfg, db, model, per_row=True)
e = O.run(cfg, db, model, per_row=True, emulate_bf16=True)
ok = ~np.isnan(o.score)
for nm, a, b in (("gpu-fp64", g["score"][ok], o.score[ok]), ("gpu-emu", g["score"][ok], e.score[ok]),
                 ("emu-fp64", e.score[ok], o.score[ok])):
    d = np.abs(a.astype(np.float64) - b)
    print(nm, "max %.5f p99.9 %.5f p99 %.5f mean %.6f" % (d.max(), np.percentile(d, 99.9), np.percentile(d, 99), d.mean()))
