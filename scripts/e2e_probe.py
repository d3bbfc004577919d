"""Where does the e2e step's time go? (load_table COPY_HOST / run_query / drop_table), C2 at SF1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as D
from paper_2311_02781_b200 import flern as F
from paper_2311_02781_b200.session import GpuQuery
cfg = D.with_sf(D.CONFIGS["c2"], 1.0)
db = D.make_database(cfg)
gq = GpuQuery(cfg, db, D.make_model(cfg, db), load_fact=False)
pinned = {k: torch.from_numpy(v).pin_memory() for k, v in db.fact.items()}
G = cfg.ngroups
hc, hs = np.zeros(G, np.int64), np.zeros(G, np.int64)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tid = F.flern_load_table(gq.ctx, "f", pinned, F.FLERN_COPY_HOST); torch.cuda.synchronize(); t1 = time.perf_counter()
    r = F.flern_run_query(gq.ctx, gq.make_query(tid), count=hc, sum=hs); t2 = time.perf_counter()
    F.flern_drop_table(gq.ctx, tid); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  query {1e3*(t2-t1):.2f} ms (kernel {r.elapsed_ms:.3f})  drop {1e3*(t3-t2):.2f} ms")
