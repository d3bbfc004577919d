"""Instructions executed per CUDA source line (SASS attributed to the line it follows).

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
       python scripts/ncu_lines.py src.csv [N] [units]   (units: divide counts by this, e.g. rows)"""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
cur_file, cur_line, hdr = "?", 0, None
ex, st = collections.Counter(), collections.Counter()
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
    v = dict(zip(hdr[2:], r[2:]))
    try:
        int(r[2], 16)
    except ValueError:
        continue
    key = f"{cur_file}:{cur_line}"
    ex[key] += int(v.get("Instructions Executed", "0").replace("-", "0") or 0)
    st[key] += int(v.get("Warp Stall Sampling (All Samples)", "0").replace("-", "0") or 0)
T = sum(ex.values())
print(f"total warp-instr {T} ({T / units:.2f} per unit)")
for k, x in ex.most_common(n):
    print(f"{x / units:8.3f}  {100 * x / T:5.1f}%  stall-samples {st[k]:6d}  {k}")
