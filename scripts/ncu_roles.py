"""Attribute ncu warp-stall samples (SASS level) to the fused kernel's warp roles.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv; python scripts/ncu_roles.py src.csv
Each SASS instruction inherits the file:line of the CUDA line it follows; inlined helpers (sm100.cuh,
intrinsics) inherit the role of the nearest preceding instruction with a role-defining line."""
import csv, sys, collections

def _c(marker):
    import os
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2311_02781_b200", "csrc", "common.cuh")
    for i, l in enumerate(open(src).read().split("\n")):
        if marker in l:
            return i + 1
    return 99999


def _ranges():
    """Role line ranges of query_kernel.cuh, found from the section markers in the source."""
    import os
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2311_02781_b200", "csrc",
                       "query_kernel.cuh")
    lines = open(src).read().split("\n")
    def find(marker, start=0):
        for i in range(start, len(lines)):
            if marker in lines[i]:
                return i + 1
        return len(lines)
    setup = find("one-time setup")
    mma = find("MMA ISSUER")
    epi = find("EPILOGUE (warps")
    wg0 = find("---- warpgroup 0:", epi)
    wg1 = find("---- warpgroup 1:", epi)
    nl1 = find("---- NL == 1:", epi)
    tear = find("---- teardown", epi)
    return {
        ("pw_producer.cuh", 1, 99999): "producer",
        ("producer.cuh", 1, 99999): "producer",
        ("query_kernel.cuh", setup, mma - 1): "setup/dispatch",
        ("query_kernel.cuh", mma, epi - 1): "mma",
        ("query_kernel.cuh", epi, wg0 - 1): "epi-common",
        ("query_kernel.cuh", wg0, wg1 - 1): "wg0",
        ("query_kernel.cuh", wg1, nl1 - 1): "wg1",
        ("query_kernel.cuh", nl1, tear - 1): "nl1-epilogue",
        ("query_kernel.cuh", tear, 99999): "teardown",
        ("common.cuh", _c("Predicate + group-by of one"), _c("Guided work distribution") - 1): "groupby",
        ("common.cuh", _c("write_partials_and_reduce("), 99999): "teardown",
        ("wide_kernel.cuh", 1, 99999): "wide",
    }


ROLE_LINES = _ranges()


def role_of(f, line):
    for (suf, lo, hi), r in ROLE_LINES.items():
        if f.endswith(suf) and lo <= line <= hi:
            return r
    return None


rows = list(csv.reader(open(sys.argv[1])))
cur_file, cur_line, hdr = None, 0, None
ins = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] in ("Function Name",):
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
        addr = int(r[2], 16)
    except ValueError:
        continue
    vals = dict(zip(hdr[2:], r[2:]))
    ins.append((addr, cur_file, cur_line, r[3], vals))
ins.sort(key=lambda x: x[0])
role = "?"
tot = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
execd = collections.Counter()
top = collections.defaultdict(list)
for addr, f, line, sass, v in ins:
    rr = role_of(f or "", line)
    if rr:
        role = rr
    s = int(v.get("Warp Stall Sampling (All Samples)", "0") or 0)
    tot[role] += s
    execd[role] += int(v.get("Instructions Executed", "0") or 0)
    for k, x in v.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                reasons[role][k[6:]] += int(x)
            except ValueError:
                pass
    top[role].append((s, f.split("/")[-1] if f else "?", line, sass.strip()[:60]))
T = sum(tot.values())
for role, s in tot.most_common():
    rs = ", ".join(f"{k} {100 * x / max(1, s):.0f}%" for k, x in reasons[role].most_common(5))
    print(f"{role:10s} samples {s:7d} ({100 * s / T:4.1f}%)  warp-instr {execd[role]:>11d}  | {rs}")
    for t in sorted(top[role], reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
        print(f"      {t[0]:6d} {t[1]}:{t[2]}  {t[3]}")
