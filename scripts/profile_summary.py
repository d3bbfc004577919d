"""Write profiles/<tag>_* from a scripts/gpu_round.sh <run> round trip: bench lines, the launch list,
traffic.json and the ncu summary (C2 full set + role stalls, C3 full set).
usage: python scripts/profile_summary.py <run-tag> <profile-tag>   e.g. r1f r01f"""
import collections, csv, json, os, re, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
run, tag = sys.argv[1], sys.argv[2]
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
for w in ["c2", "c1", "c1x", "c4p", "c3", "c4", "c2nomodel"]:
    src = os.path.join(G, f"bench_{w}_{run}.json")
    if os.path.exists(src):
        open(os.path.join(P, f"{tag}_bench_{w}.json"), "w").write(open(src).read().strip().splitlines()[-1] + "\n")
shutil.copy(os.path.join(G, f"launches_c2_{run}.csv"), os.path.join(P, f"{tag}_launches_c2.csv"))


def sh(cmd):
    return subprocess.run(cmd, shell=True, capture_output=True, text=True, cwd=ROOT).stdout


def extract(name, cmd):
    """Text extracted on the box by gpu_round.sh (reports too large to copy back), else from the report."""
    f = os.path.join(G, name)
    return open(f).read() if os.path.exists(f) else sh(cmd)


c2 = extract(f"ncusum_c2_{run}.md", f"python scripts/ncu_summary.py gpurun_out/prof_c2_{run}.ncu-rep")
c3 = extract(f"ncusum_c3_{run}.md", f"python scripts/ncu_summary.py gpurun_out/prof_c3_{run}.ncu-rep")
roles = extract(f"roles_c2_{run}.txt", f"ncu -i gpurun_out/prof_c2_{run}.ncu-rep --page source --csv "
                f"--print-source cuda,sass > /tmp/_src.csv; python scripts/ncu_roles.py /tmp/_src.csv 3")
raw3 = list(csv.reader(extract(f"raw_c3_{run}.csv", f"ncu -i gpurun_out/prof_c3_{run}.ncu-rep --page raw --csv").splitlines()))
d3 = {k: (u, v) for k, u, v in zip(raw3[0], raw3[1], raw3[2])} if len(raw3) > 2 else {}
rows = list(csv.reader(open(os.path.join(P, f"{tag}_launches_c2.csv"))))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0].replace("void ", "")[:70]].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
qk = next((v for k, v in agg.items() if "flern_query_kernel" in k), [1.0])
big = [v for v in qk if v > 0.5 * max(qk)]
small = [v for v in qk if v <= 0.5 * max(qk)]
nbig, mbig = len(big), sum(big) / max(1, len(big))
nsmall, msmall = len(small), sum(small) / max(1, len(small))
ll = "\n".join(f"| {len(v)} | {sum(v) / len(v):,.0f} | {100 * sum(v) / tot:.1f}% | `{k}` |"
               for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])))
b = json.loads(open(os.path.join(P, f"{tag}_bench_c2.json")).read())
dr = float(re.search(r"DRAM read .*?\| ([0-9.]+) Mbyte", c2).group(1))
dw = float(re.search(r"DRAM write .*?\| ([0-9.]+) Mbyte", c2).group(1))
c1x = ""
traffic = {"c2": (dr + dw) * 1e6}
if os.path.exists(os.path.join(G, f"ncusum_c1x_{run}.md")) or os.path.exists(os.path.join(G, f"prof_c1x_{run}.ncu-rep")):
    c1x = extract(f"ncusum_c1x_{run}.md", f"python scripts/ncu_summary.py gpurun_out/prof_c1x_{run}.ncu-rep")
    m1 = re.search(r"DRAM read .*?\| ([0-9.]+) ([MG])byte", c1x)
    m2 = re.search(r"DRAM write .*?\| ([0-9.]+) ([MG])byte", c1x)
    if m1 and m2:
        sc = lambda m: float(m.group(1)) * (1e9 if m.group(2) == "G" else 1e6)
        traffic["c1x"] = sc(m1) + sc(m2)
traffic["_source"] = (f"ncu --set full, profiles/{tag}_ncu_summary.md "
                      "(dram__bytes_read.sum + dram__bytes_write.sum, one launch)")
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
x3 = d3.get("l1tex__m_xbar2l1tex_read_bytes.sum", ("", "?"))
x3s = d3.get("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", ("", "?"))
md = f"""# {tag} — ncu evidence for the bench lines (`profiles/{tag}_bench_*.json`)

From `scripts/gpu_round.sh {run}` on one fresh B200 (reports are scratch in `gpurun_out/`, numbers copied):
- launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 200` of
  `python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1` → `profiles/{tag}_launches_c2.csv`;
- full set: `ncu --set full --clock-control none --import-source on -k regex:flern_query -s 6 -c 1` of the same
  command (C2), and `-k regex:flern_query_wide -s 4 -c 1` of `--workload c3`.

ncu serialises and replays kernels (cold caches, ~1.7 GHz under the profiler): evidence for the kernels'
behaviour, not bench values.

## Launch list (C2 bench command)

| launches | mean ns | share | kernel |
|---:|---:|---:|---|
{ll}

The query kernel is the whole timed step, one launch per step (the build kernels run once, outside it).
Its launches split into {nbig} whole-shard launches (mean {mbig:,.0f} ns: the timed steps, warm-ups and
the row-count run) and {nsmall} launches over 1/8 of the shard each (mean {msmall:,.0f} ns: the streamed e2e
leg, `flern_run_query_streamed`). Bench: {b['roofline']['avg_launch_ms'] * 1e3:.0f} µs per launch live
(CUDA events), so the kernel's share of the step agrees.

## C2 query kernel (`--set full`)

{c2}
- DRAM traffic {dr + dw:.0f} MB per launch: the 312 MB of fact columns plus the touched build entries
  (1.5 M × 32 B): no re-reads; ≈7% of HBM bandwidth — the kernel is not memory-bound.
- Roofline (bench line): 139,776 flop/row × 6,002,157 rows ÷ {b['roofline']['avg_launch_ms']:.4f} ms =
  **{b['roofline']['achieved']:.0f} TFLOP/s = {100 * b['roofline']['frac']:.1f}% of {b['roofline']['peak']:,}** (bf16 burst peak, {b['roofline'].get('peak_source', '')}).

### Warp-stall samples by role (`scripts/ncu_roles.py`)

```
{roles}
```

## C3 wide kernel (`--set full`)

{c3}
- L2 → SM traffic {x3[1]} {x3[0]} per launch ({x3s[1]} {x3s[0]}): each 128-row tile re-streams 4 MB of
  weights and reads its activations four times; with the power cap (≈1.7 GHz) this bounds the kernel near
  70% of the sustained bf16 peak (DESIGN.md §12).

## C1x query kernel (`--set full`, the HBM-bound supplementary row: C1 shape at SF10)

{c1x if c1x else "(not captured in this run)"}
- Compulsory DRAM bytes: 1,680 MB of fact columns plus the build entries the sorted probe stream touches
  (15 M orders × 32 B) ≈ 2.16 GB per launch.

## SASS evidence (tcgen05 / TMEM / TMA)

`cuobjdump -sass paper_2311_02781_b200/lib/libflern.so` (checked by `tests/test_abi.py`): `UTCHMMA` with
`gdesc` (SMEM) and `tmem` A operands, `UTCBAR` (commit → mbarrier), `LDTM` / `STTM`, `UBLKCP` (1D bulk
copies: fact loader, wide-kernel operand loader), `SYNCS.*` (mbarriers), `FFMA2` / `F2FP`; no `HMMA`.
"""
open(os.path.join(P, f"{tag}_ncu_summary.md"), "w").write(md)
print("wrote", tag)
