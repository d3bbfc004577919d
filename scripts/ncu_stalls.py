"""Per-source-line warp-stall breakdown from an ncu source CSV (SASS attributed to the CUDA line it follows).

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
       python scripts/ncu_stalls.py src.csv [file-substring] [N]"""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
filt = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur_file, cur_line, hdr = "?", 0, None
samp, ex = collections.Counter(), collections.Counter()
reasons = collections.defaultdict(collections.Counter)
sass = collections.defaultdict(list)
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
    key = f"{cur_file}:{cur_line}"
    s = int(v.get("Warp Stall Sampling (All Samples)", "0").replace("-", "0") or 0)
    samp[key] += s
    ex[key] += int(v.get("Instructions Executed", "0").replace("-", "0") or 0)
    for k, x in v.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                reasons[key][k[6:]] += int(x)
            except ValueError:
                pass
    sass[key].append((s, r[3].strip()[:50]))
T = sum(samp.values())
print(f"total stall samples {T}")
for k, s in samp.most_common():
    if filt and filt not in k:
        continue
    rs = ", ".join(f"{a} {100 * x / max(1, s):.0f}%" for a, x in reasons[k].most_common(3))
    top = max(sass[k])[1] if sass[k] else ""
    print(f"{s:7d} {100 * s / T:5.1f}%  exec {ex[k]:>10d}  {k:24s} | {rs} | {top}")
    n -= 1
    if n <= 0:
        break
