"""Rank SASS instructions (with their CUDA line) by one ncu source-page column, e.g. "L1 Wavefronts Shared".

usage: python scripts/ncu_col.py src.csv "L1 Wavefronts Shared" [N]"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
col = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur_file, cur_line, hdr = "?", 0, None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[2] == "-":
        try:
            cur_line = int(r[0])
        except ValueError:
            pass
        continue
    try:
        int(r[2], 16)
    except ValueError:
        continue
    v = dict(zip(hdr[2:], r[2:]))
    try:
        x = float(v.get(col, "0").replace("-", "0") or 0)
    except ValueError:
        x = 0.0
    out.append((x, f"{cur_file}:{cur_line}", r[3].strip()[:60], v.get("Instructions Executed", "")))
T = sum(o[0] for o in out)
print(f"total {col}: {T:.0f}")
for x, where, sass, ex in sorted(out, reverse=True)[:n]:
    print(f"{x:12.0f} {100 * x / max(T, 1):5.1f}%  exec {ex:>10s}  {where:26s} {sass}")
