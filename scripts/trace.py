"""Pipeline trace of CTA 0 (diagnostic): where does each role wait? Prints per-tile deltas."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen as D
from paper_2311_02781_b200 import flern as F
from paper_2311_02781_b200.session import GpuQuery

EV = ["MMA_D2A_FREE", "MMA_L2A_DONE", "MMA_NEXT_READY", "MMA_L1_ISSUED", "MMA_D2B_FREE", "MMA_L2B_ISSUED",
      "W0_FULL", "W0_D1FULL", "W0_HFREE0", "W0_DONE", "W1_FULL", "W1_DFULL0", "W1_DOTA", "W1_DFULL1", "W1_DOTB",
      "W1_AGG", "P_START", "P_PROBED", "P_GATHERED", "P_DONE"]
args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "c2"
sf = float(args[1]) if len(args) > 1 else 1.0
flags = F.FLERN_Q_NO_MODEL if "--no-model" in sys.argv else 0
cfg = D.with_sf(D.CONFIGS[name], sf)
db = D.make_database(cfg)
gq = GpuQuery(cfg, db, D.make_model(cfg, db))
G = cfg.ngroups
for it in range(3):
    tr = np.zeros(F.TRACE_EVENTS * F.TRACE_TILES, np.uint64)
    r = gq.run(gq.make_query(gq.fact_id, flags=flags), count=np.zeros(G, np.int64), sum=np.zeros(G, np.int64),
               dbg_trace=tr)
tr = tr.reshape(F.TRACE_EVENTS, F.TRACE_TILES).astype(np.int64)
t0 = tr[:20][tr[:20] > 0].min() if (tr[:20] > 0).any() else 0   # (release-like builds: no stamps)
print("kernel ms", r.elapsed_ms)
for t in list(range(0, 12)) + [100, 101, 102]:
    row = " ".join(f"{EV[e][:12]}={(tr[e, t] - t0) if tr[e, t] else -1:>8d}" for e in range(16))
    print(t, row)
print("producer batches:")
for b in list(range(0, 8)) + [100, 101]:
    print(b, " ".join(f"{EV[e]}={(tr[e, b] - t0) if tr[e, b] else -1}" for e in range(16, 20)))
# steady-state per-tile period and phase durations (tiles 20..200)
sl = slice(20, 200)
def d(a, b):
    x = tr[b, sl] - tr[a, sl]
    return float(np.median(x[(tr[a, sl] > 0) & (tr[b, sl] > 0)]))
per = np.diff(tr[EV.index("MMA_L2B_ISSUED"), sl])
print("median tile period (cycles):", float(np.median(per)))
for a, b in [("MMA_D2A_FREE", "MMA_L2A_DONE"), ("MMA_L2A_DONE", "MMA_NEXT_READY"), ("MMA_NEXT_READY", "MMA_L1_ISSUED"),
             ("MMA_L1_ISSUED", "MMA_D2B_FREE"), ("MMA_D2B_FREE", "MMA_L2B_ISSUED"), ("W0_FULL", "W0_D1FULL"),
             ("W0_D1FULL", "W0_HFREE0"), ("W0_HFREE0", "W0_DONE"), ("W1_FULL", "W1_DFULL0"), ("W1_DFULL0", "W1_DOTA"),
             ("W1_DOTA", "W1_DFULL1"), ("W1_DFULL1", "W1_DOTB"), ("W1_DOTB", "W1_AGG"), ("P_START", "P_PROBED"),
             ("P_PROBED", "P_GATHERED"), ("P_GATHERED", "P_DONE")]:
    print(f"  {a:>16s} -> {b:<16s} {d(EV.index(a), EV.index(b)):8.0f}")
pd = np.diff(tr[EV.index("P_START"), 10:100])
print("producer batch period:", float(np.median(pd)))
# fact loader (C1 shapes: stamps of stage b before / after its empty wait) vs the producer warp 0 batches
lb, la = tr[EV.index("MMA_D2B_FREE")], tr[EV.index("MMA_L2A_DONE")]
if (la[20:200] > 0).all() and not (tr[EV.index("MMA_L2B_ISSUED"), 20:200] > 0).any():
    print("  loader: stage period", float(np.median(np.diff(la[20:200]))), " empty-wait", float(np.median((la - lb)[20:200])))
    ps = tr[EV.index("P_START")]
    print("  producer w0: issue(b+1) wait", d(EV.index("P_START"), EV.index("P_PROBED")), " gather wait",
          d(EV.index("P_PROBED"), EV.index("P_GATHERED")), " process", d(EV.index("P_GATHERED"), EV.index("P_DONE")),
          " done->next", float(np.median((ps[21:200] - tr[EV.index("P_DONE"), 20:199]))))
    print("  loader publish(b) -> producer w0 start(b-1):", float(np.median(ps[20:200] - la[21:201])))
    for a, b in [("P_START", "P_PROBED"), ("P_PROBED", "W0_FULL"), ("W0_FULL", "P_GATHERED"), ("P_GATHERED", "W0_D1FULL"),
                 ("W0_D1FULL", "W0_HFREE0"), ("W0_HFREE0", "W0_DONE"),
                 ("W0_DONE", "W1_DOTB"), ("W1_DOTB", "P_DONE")]:
        print(f"    process {a:>10s} -> {b:<10s} {d(EV.index(a), EV.index(b)):8.0f}")
# pre-filter scan (c4p): per scan chunk b of producer thread 0: wait for the chunk, scan + gathers
if "--pf" in sys.argv:
    a, w, e = tr[EV.index("MMA_NEXT_READY")], tr[EV.index("MMA_D2A_FREE")], tr[EV.index("MMA_L1_ISSUED")]
    ok = (a[10:250] > 0) & (e[10:250] > 0)
    print("  pf chunk period", float(np.median(np.diff(a[10:250][ok]))), " wait", float(np.median((w - a)[10:250][ok])),
          " scan+gather", float(np.median((e - w)[10:250][ok])), " mean scan+gather", float(np.mean((e - w)[10:250][ok])))
    gs, gd = tr[EV.index("P_START")], tr[EV.index("P_DONE")]
    okg = (gs[:200] > 0) & (gd[:200] > 0)
    if okg.any():
        print("  gather batches", int(okg.sum()), " median duration", float(np.median((gd - gs)[:200][okg])))
# NL = 1 pipeline (C1 shapes): MMA issuer and the epilogue warpgroup of each tile
if (tr[EV.index("W1_FULL"), 20:200] > 0).any() and not (tr[EV.index("MMA_L2B_ISSUED"), 20:200] > 0).any():
    for a, b in [("MMA_NEXT_READY", "MMA_D2A_FREE"), ("MMA_D2A_FREE", "MMA_L1_ISSUED"), ("MMA_L1_ISSUED", "W1_DFULL0"),
                 ("W1_FULL", "W1_DFULL0"), ("W1_DFULL0", "W1_DOTA"), ("W1_DOTA", "W1_AGG")]:
        print(f"  NL1 {a:>16s} -> {b:<16s} {d(EV.index(a), EV.index(b)):8.0f}")
    print("  NL1 tile period (epilogue):", float(np.median(np.diff(tr[EV.index("W1_AGG"), 20:200]))))
    print("  NL1 W1_AGG(t) -> W1_FULL(t+2):", float(np.median(tr[EV.index("W1_FULL"), 22:200] - tr[EV.index("W1_AGG"), 20:198])))
W = ["MMA<-producer(full)", "MMA<-WG1(dempty0)", "MMA<-WG1(dempty1)", "MMA<-WG0(hfull)", "MMA<-WG0(d1empty)",
     "WG0<-producer(full)", "WG0<-MMA(d1full)", "WG0<-MMA(hfree)", "WG1<-producer(full)", "WG1<-MMA(dfull)",
     "producer<-WG1(empty)", "kernel cycles (CTA0 MMA thread)"]
w = tr[20]
print("wait cycles, CTA 0 (fraction of kernel):")
for i, nm in enumerate(W):
    print(f"  {nm:34s} {int(w[i]):>10d}  {w[i] / max(1, w[11]):6.1%}")
# per-CTA timeline (%globaltimer, ns): start skew, loop-end spread (imbalance), final reduce
st, su, le, ex = tr[21], tr[22], tr[23], tr[24]
n = int((st > 0).sum())
if n:
    st, su, le, ex = st[:n], su[:n], le[:n], ex[:n]
    z = st.min()
    print(f"CTAs {n}: start skew {(st.max() - z) / 1e3:.1f} us; setup median/max {np.median(su - st) / 1e3:.1f}/"
          f"{(su - st).max() / 1e3:.1f} us; loop end min/median/max "
          f"{(le.min() - z) / 1e3:.1f}/{np.median(le - z) / 1e3:.1f}/{(le.max() - z) / 1e3:.1f} us; "
          f"last exit {(ex.max() - z) / 1e3:.1f} us; kernel (events) {r.elapsed_ms * 1e3:.1f} us")
    te = (ex - le) / 1e3
    print(f"  teardown (exit - loop end) us: min {te.min():.1f} median {np.median(te):.1f} max {te.max():.1f}; "
          f"last CTA to exit: {int(np.argmax(ex))} (loop end {(le[np.argmax(ex)] - z) / 1e3:.1f} us)")
    order = np.argsort(le - st)
    print("  slowest CTAs (loop us):", [(int(i), round(float(le[i] - st[i]) / 1e3, 1)) for i in order[-6:]])
    print("  fastest CTAs (loop us):", [(int(i), round(float(le[i] - st[i]) / 1e3, 1)) for i in order[:6]])

# MMA thread event sequence from tile 100 (TR_MMA_SEQ): clock deltas and tags
TAGS = {1: "L2a", 2: "L2b", 3: "L1", 4: "bias", 10: "hfull>", 11: "<hfull", 12: "dempty0>", 13: "<dempty0",
        14: "dempty1>", 15: "<dempty1", 16: "d1empty>", 17: "<d1empty", 18: "full>", 19: "<full", 30: "TILE"}
seq = tr[25]
seq = seq[seq != 0]
if len(seq):
    clk = (seq.astype(np.uint64) >> np.uint64(8)).astype(np.int64)
    tag = (seq & 255).astype(np.int64)
    c0 = clk[0]
    line = []
    for i in range(len(seq)):
        d = clk[i] - (clk[i - 1] if i else c0)
        line.append(f"{TAGS.get(int(tag[i]), tag[i])}+{d}")
    print("MMA sequence (event+cycles since previous):")
    for i in range(0, min(len(line), 96), 12):
        print("   ", " ".join(line[i:i + 12]))
    import collections
    agg = collections.defaultdict(list)
    for i in range(1, len(seq)):
        agg[TAGS.get(int(tag[i]), int(tag[i]))].append(int(clk[i] - clk[i - 1]))
    nt = max(1, int((tag == 30).sum()) - 1)
    span = int(clk[np.where(tag == 30)[0][-1]] - clk[np.where(tag == 30)[0][0]]) if (tag == 30).sum() > 1 else 0
    print(f"per tile ({nt} tiles, {span / nt:.0f} cycles/tile): total cycles attributed to each event (time since previous)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"   {k:>10s}: n/tile {len(v) / nt:5.1f}  mean {np.mean(v):7.1f}  total/tile {sum(v) / nt:8.1f}")
