"""Wait accounting of the wide kernel's first CTA pair (diagnostic build: FLERN_LIB=libflern_diag.so).

usage: FLERN_LIB=paper_2311_02781_b200/lib/libflern_diag.so python scripts/trace_wide.py [workload] [sf]
Prints, per CTA of pair 0, the cycles each role spent in each wait as a fraction of the MMA loop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen as D
from paper_2311_02781_b200 import flern as F
from paper_2311_02781_b200.session import GpuQuery

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
sf = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = D.with_sf(D.CONFIGS[name], sf)
db = D.make_database(cfg)
gq = GpuQuery(cfg, db, D.make_model(cfg, db))
G = cfg.ngroups
names = ["mma decb", "mma dempty", "mma rfull L1", "mma rfull hidden", "ld xfull", "ld pair exch", "ld rempty",
         "ld actrdy", "wg0 decb", "wg0 dfull", "wg1 dfull", "wg1 xchg"]
for it in range(2):
    tr = np.zeros(F.TRACE_EVENTS * F.TRACE_TILES, np.uint64)
    r = gq.run(gq.make_query(gq.fact_id), count=np.zeros(G, np.int64), sum=np.zeros(G, np.int64), dbg_trace=tr)
tr = tr.reshape(F.TRACE_EVENTS, F.TRACE_TILES).astype(np.int64)
w = tr[F.TRACE_EVENTS_WAITS if hasattr(F, "TRACE_EVENTS_WAITS") else 20]
print("kernel ms", r.elapsed_ms, "rows", cfg.name, sf)
for cta in range(2):
    b = 32 + 16 * cta
    loop = w[b + 13] - w[b + 12] if cta == 0 else 0
    tiles = w[b + 14]
    print(f"cta {cta}: MMA loop cycles {loop}, tiles {tiles}, cycles/tile {loop / max(tiles, 1):.0f}")
    base = w[32 + 13] - w[32 + 12]
    for i, n in enumerate(names):
        print(f"   {n:>18s} {w[b + i]:>14d}  {w[b + i] / max(base, 1) * 100:6.1f}% of the MMA loop")
# per-stage timeline (hidden-layer stages from kSeqStage0 on, CTA 0): MMA thread and loader
N = 800
seq = tr[:10].reshape(-1)[: 3 * N].reshape(-1, 3)
lseq = tr[10:20].reshape(-1)[: 2 * N].reshape(-1, 2)
ok = (seq > 0).all(axis=1) & (lseq > 0).all(axis=1)
if ok.sum() > 10:
    idx = np.nonzero(ok)[0]
    seq, lseq = seq[ok], lseq[ok]
    wait = seq[:, 1] - seq[:, 0]
    issue = seq[:, 2] - seq[:, 1]
    period = np.diff(seq[:, 0])
    armed_ahead = seq[:, 0] - lseq[:, 1]   # > 0: the loader armed the stage before the issuer started waiting
    print(f"stages traced {len(seq)}: period median {np.median(period):.0f}; rfull wait median {np.median(wait):.0f}; "
          f"4-MMA issue median {np.median(issue):.0f}; armed before the wait by median {np.median(armed_ahead):.0f}")
    print("stage: wait issue period | loader: armed-vs-wait-start, rempty-return -> armed")
    for i in range(min(30, len(seq) - 1)):
        print(f"  {idx[i]:4d} {wait[i]:6d} {issue[i]:6d} {period[i]:6d} | {armed_ahead[i]:7d} {lseq[i, 1] - lseq[i, 0]:6d}")
# dempty waits of CTA 0's MMA thread per position in the tile's chunk sequence (diagnostic builds)
pos = w[100:100 + 12]
if pos.sum() > 0:
    print("dempty wait per chunk position (cycles, summed over tiles):", " ".join(str(int(x)) for x in pos))
