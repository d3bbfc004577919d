"""Summarise a round's per-workload ncu counters (scripts/gpu_round2.sh) into profiles/.

usage: python scripts/counters_summary.py TAG
reads  gpurun_out/counters_<workload>_<TAG>.csv (one launch of the workload's query / training kernel)
       gpurun_out/bench_<workload>_<TAG>.json  (the bench line of the same round)
writes profiles/<TAG>_counters.md  (a table per workload: duration, DRAM bytes, HBM share, tensor-memory
                                    and tensor-operand activity, issue, occupancy, achieved rates)
       profiles/traffic.json        ({workload: DRAM read + write bytes of one launch}, with the round tag;
                                    bench.py reports it as roofline.traffic)
"""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_counters(path):
    rows = list(csv.reader(open(path)))
    hdr, vals, kernel = None, {}, ""
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            vals[d["Metric Name"]] = d["Metric Value"]
            kernel = d["Kernel Name"]
    return kernel, vals


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    tag = sys.argv[1]
    out = ["# %s — ncu counters per workload (one launch each)" % tag, "",
           "From `scripts/gpu_round2.sh " + tag + "` on one B200: `ncu --metrics … --clock-control none -k regex:flern_query "
           "-s 2 -c 1` of `bench.py --workload W --steps 2 --warmup 3` (the third query launch; `train`: "
           "`flern_train_kernel`). ncu serialises launches and runs them cold-cache: evidence for what a kernel "
           "does, not bench values. `nm` = `--no-model` (scan → probe → gather → aggregate only)." , "",
           "| workload | kernel | µs | DRAM read MB | DRAM write MB | DRAM % of peak | L2 bytes MB | TMEM active % "
           "| TC operand wavefronts % | issue active % | warps active % | warp-instr / row |", "|" + "---|" * 12]
    traffic = {"round": tag, "source": "dram__bytes_read.sum + dram__bytes_write.sum of one launch (ncu)"}
    for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "counters_*_%s.csv" % tag))):
        w = os.path.basename(path)[len("counters_"):-len("_%s.csv" % tag)]
        kernel, v = read_counters(path)
        if not v:
            continue
        rows = None
        bj = os.path.join(ROOT, "gpurun_out", "bench_%s_%s.json" % ({"c2nm": "c2nomodel", "c1xnm": "c1xnomodel"}.get(w, w), tag))
        if os.path.exists(bj):
            try:
                line = json.loads(open(bj).read().strip().splitlines()[-1])
                cfgd = line.get("config", {})
                rows = cfgd.get("rows_per_gpu")
            except Exception:
                pass
        rd, wr = num(v.get("dram__bytes_read.sum")), num(v.get("dram__bytes_write.sum"))
        if rd is not None and wr is not None and not w.endswith("nm"):
            traffic[w] = rd + wr
        ie = num(v.get("smsp__inst_executed.sum"))
        kname = kernel.split("(")[0].replace("void ", "")[:60]
        out.append("| %s | `%s` | %.1f | %.1f | %.1f | %s | %.1f | %s | %s | %s | %s | %s |" % (
            w, kname, num(v.get("gpu__time_duration.sum")) / 1e3, rd / 1e6, wr / 1e6,
            v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"), num(v.get("lts__t_bytes.sum")) / 1e6,
            v.get("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            v.get("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            v.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "%.1f" % (ie / rows) if (ie and rows) else "—"))
    out += ["", "TMEM active % = `sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed` (cycles the tensor "
            "memory is busy: MMA accumulator reads/writes and `tcgen05.ld/st`); TC operand wavefronts % = "
            "`l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed` (SMEM operand traffic "
            "of the MMAs). The `sm__pipe_tensor_cycles_active_realtime` counters read n/a for tcgen05 kernels on "
            "this driver, and `sm__ops_path_tensor_op_hmma_*` count only legacy HMMA (0 here)."]
    open(os.path.join(ROOT, "profiles", "%s_counters.md" % tag), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
