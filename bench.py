"""bench.py — joined rows scored/sec of the fused query+MLP path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl reference]

One step = one flern_run_query over this rank's whole fact shard (scan -> probe -> gather ->
tcgen05 MLP -> predicate -> group-by: every §8(a) row, one kernel launch) + (N > 1) the NCCL
reduce of the per-group partials. Inputs are resident in HBM when the timed region starts; the
fact columns (312 MB/GPU at SF1) exceed the 126 MB L2, so no flush is needed between steps.
Weak scaling: every rank holds an SF1-sized lineitem shard of an SF=N database (orders table
and weights replicated). `--impl reference` times the CPU oracle (the reference arm for this
tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen as D  # noqa: E402

WORKLOADS = {
    "c2": "TPC-H-shaped lineitem⋈orders (SF1 per GPU), 16 features -> MLP 16-256-256-1 (ReLU, sigmoid), "
          "score>0.5, GROUP BY o_orderpriority COUNT/SUM(l_extendedprice)",
    "c1": "TPC-H-shaped lineitem⋈orders (SF0.01 per GPU), 8 features -> MLP 8-64-1, score>0.5, GROUP BY "
          "o_orderpriority COUNT/SUM(l_extendedprice)",
    "c1x": "C1 query shape at SF10 per GPU (HBM-bound supplementary row), MLP 8-64-1",
    "c4p": "SF10 per GPU, l_shipdate pre-filter (~2%) before inference, lineitem⋈orders, MLP 16-256-256-1",
    "c3": "TPC-H-shaped lineitem⋈orders⋈customer (two probes, SF10 per GPU), 32 features -> MLP "
          "32-1024-1024-1024-1, score>0.5, GROUP BY o_orderpriority COUNT/SUM(l_extendedprice)",
    "c4": "config 3 + l_shipdate pre-filter (~2%) before inference (SF10 per GPU), MLP 32-1024-1024-1024-1",
    "c5": "TPC-H-shaped SF100 lineitem sharded by orderkey range across the GPUs (strong scaling), lineitem⋈orders "
          "(orders + weights replicated), 16 features -> MLP 16-256-256-1, score>0.5, GROUP BY o_orderpriority "
          "COUNT/SUM(l_extendedprice), NCCL reduce of the group partials",
}
WORKLOADS["c2s"] = ("C2 with the order keys scattered over 31 bits by a bijection (k -> k * 0x9E3779B1 mod 2^31): "
                    "the build picks open addressing (Fibonacci hash, 8-byte {key, row} slots + payload rows) and "
                    "every probe is a random access, instead of the direct-addressed fat entries of C2")
WORKLOADS["train"] = ("ML in charge (NEXT-3): one SGD step (MSE, 16-128-128-1 regression of l_quantity) per pass over "
                      "the C2 query's joined rows (SF1 per GPU): gather -> forward -> backward -> update")
STRONG = {"c5"}          # total work fixed as N grows; the others hold a fixed shard per GPU
TRAIN_METRIC = "joined rows trained/sec (one SGD step per batch, MSE, 16-128-128-1)"
TRAIN_DIMS = [16, 128, 128, 1]


def scatter_keys(db):
    """c2s: remap l_orderkey / o_orderkey through the same bijection of [0, 2^31) (odd multiplier), so the
    join result is unchanged but the keys are sparse and unordered."""
    f = lambda k: ((k.astype(np.uint64) * np.uint64(0x9E3779B1)) & np.uint64(0x7FFFFFFF)).astype(np.int32)
    db.fact["l_orderkey"] = f(db.fact["l_orderkey"])
    name, m, cols = db.builds[0]
    cols["o_orderkey"] = f(cols["o_orderkey"])
    return db


def make_db(name, cfg, **kw):
    db = D.make_database(cfg, **kw)
    return scatter_keys(db) if name == "c2s" else db


def train_flops_per_row(dims):
    """forward + backward (dX and dW): 3x the forward's 2 * sum(in * out) multiply-adds"""
    return 3 * flops_per_row(dims)
METRIC = "joined rows scored/sec (query+MLP, whole box)"


def flops_per_row(dims):
    return 2 * sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))


def binding_roofline(flops_per_row, rows, alg_bytes, launch_ms, tf_peak, hbm_peak, tf_src="", hbm_src=""):
    """Both rooflines of one launch; the binding one (longer algorithmic time at peak) comes first."""
    s = launch_ms / 1e3
    tf = flops_per_row * rows / s / 1e12
    gb = alg_bytes / s / 1e9
    tensor_rf = {"bound": "tensor", "achieved": tf, "peak": tf_peak, "unit": "TFLOP/s", "frac": tf / tf_peak,
                 "flops_per_row": flops_per_row, "peak_source": tf_src}
    hbm_rf = {"bound": "hbm", "achieved": gb, "peak": hbm_peak, "unit": "GB/s", "frac": gb / hbm_peak,
              "alg_bytes_per_launch": alg_bytes, "peak_source": hbm_src}
    t_tensor = flops_per_row * rows / (tf_peak * 1e12)
    t_hbm = alg_bytes / (hbm_peak * 1e9)
    return (tensor_rf, hbm_rf) if t_tensor >= t_hbm else (hbm_rf, tensor_rf)


def workload_cfg(name, world):
    if name == "c2":
        base, sf1 = D.CONFIGS["c2"], 1.0
    elif name == "c1":
        base, sf1 = D.CONFIGS["c1"], 0.01
    elif name == "c1x":
        base, sf1 = D.CONFIGS["c1"], 10.0
    elif name == "c4p":
        base, sf1 = D.CONFIGS["c4p"], 10.0
    elif name == "c3":
        base, sf1 = D.CONFIGS["c3"], 10.0
    elif name == "c4":
        base, sf1 = D.CONFIGS["c4"], 10.0
    elif name == "c5":   # strong scaling: SF100 in total, SF100/N per GPU
        return D.CONFIGS["c5"], D.CONFIGS["c5"].sf / world
    elif name == "c2s":
        base, sf1 = D.CONFIGS["c2"], 1.0
    elif name == "train":
        base, sf1 = D.with_sf(D.CONFIGS["c2"], 1.0, dims=TRAIN_DIMS, sum_col=("fact", "l_quantity"), name="train"), 1.0
    else:
        raise SystemExit(f"unknown workload {name}")
    return D.with_sf(base, sf1 * world), sf1


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("bf16_tflops", 1590.0)), float(j.get("hbm_gbs", 6650.0)), "measured"
    # MEASURED_PEAKS.json is driver-written and git-ignored; when a box lacks it, use the values the
    # driver measured on this pool at the start of round 1 (SURVEY.md Appendix [PEAKS]) — higher,
    # i.e. stricter, than the profiling guide's generic fallback (1590 TF/s, 6650 GB/s).
    return 1677.0, 6552.0, "round-1 measured (SURVEY.md [PEAKS]; file absent)"


def sustained_peak():
    """bf16 peak for a kernel timed inside a long step (the profiling recipe's 'sustained' figure)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        if "bf16_tflops_sustained" in j:
            return float(j["bf16_tflops_sustained"]), "measured bf16_tflops_sustained"
    return 1413.9, "round-1 measured sustained (SURVEY.md [PEAKS]; file absent)"


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~2 ms while the timed region runs.

    In-process NVML starts in microseconds, so even a short timed region gets samples (a spawned
    `nvidia-smi -lms` needs far longer to start than a 20-step region lasts). The device is matched to
    the CUDA device by PCI bus id, so CUDA_VISIBLE_DEVICES remapping does not pick the wrong GPU.
    """

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, cuda_index):
        self.cuda_index = cuda_index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.h = None
        self.stop = threading.Event()

    def _handle(self):
        import pynvml as N
        import torch
        N.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return N, N.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            return N, N.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def __enter__(self):
        try:
            self.N, self.h = self._handle()
            self.max_mhz = float(self.N.nvmlDeviceGetMaxClockInfo(self.h, self.N.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def _sample(self):
        N = self.N
        self.samples.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
        r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for name, attr in self.REASONS:
            if r & getattr(N, attr, 0):
                self.reasons.add(name)

    def _run(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.stop.wait(0.002)

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": "nvml"}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def cpu_baseline(cfg, db, model, seconds=25.0):
    """The oracle, as it stands, on the host's cores: a bounded prefix of this workload.

    The sample is sized from a short first pass, which runs slower per row than the long one (thread
    start-up, cold caches), so a 25 s target lands at ~10-15 s of oracle work."""
    import oracle as O
    threads = os.cpu_count() or 1
    probe = min(db.fact_n, 2000 * threads)
    t0 = time.perf_counter()
    O.run(cfg, db, model, nthreads=threads, row_lo=0, row_hi=probe)
    dt = max(1e-3, time.perf_counter() - t0)
    rows = int(min(db.fact_n, max(probe, probe / dt * seconds)))
    t0 = time.perf_counter()
    r = O.run(cfg, db, model, nthreads=threads, row_lo=0, row_hi=rows)
    dt = time.perf_counter() - t0
    # plain single-core speed (BASELINE.md's CPU plan): one thread on a prefix sized for ~3 s
    one = int(min(db.fact_n, max(64, rows / max(dt, 1e-3) / threads * 3.0)))
    t1 = time.perf_counter()
    r1 = O.run(cfg, db, model, nthreads=1, row_lo=0, row_hi=one)
    dt1 = max(1e-6, time.perf_counter() - t1)
    return {"value": r.rows_joined / dt, "unit": "rows/s", "cores": threads, "kind": "oracle",
            "sample": f"first {rows} of {db.fact_n} lineitem rows of this rank's shard, full query "
                      f"(unordered_map join + scalar fp64 MLP + predicate + group-by), {dt:.1f} s",
            "single_core": {"value": r1.rows_joined / dt1, "unit": "rows/s", "cores": 1,
                            "sample": f"first {one} lineitem rows, one thread, {dt1:.1f} s"}}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def bench_model(name, cfg):
    """One model for every rank (replicated weights): normalisation from the first rows of the unsharded
    table; the training workload's regression output starts small (out_scale 0.05)."""
    prefix = make_db(name, cfg, max_slots=D.MODEL_SLOTS)
    return D.make_model(cfg, prefix, out_scale=0.05, out_shift=0.0) if name == "train" else D.make_model(cfg, prefix)


def timing_stats(ms):
    """Per-launch device times: median and the mean without the min and max (the paper averages runs after
    dropping the lowest and highest)."""
    s = sorted(ms)
    core = s[1:-1] if len(s) > 2 else s
    return {"median_ms": statistics.median(s), "trimmed_mean_ms": sum(core) / len(core), "min_ms": s[0],
            "max_ms": s[-1]}


def run_train(args, cfg, sf1, db, model, gq, fact_bytes, world, rank, local, stream):
    """--workload train: flern_train_step over the whole shard per step (NEXT-3). One GPU."""
    import torch
    from paper_2311_02781_b200 import flern as F
    if world > 1:
        raise SystemExit("--workload train runs on one GPU (no cross-rank gradient reduction)")
    q = gq.make_query(gq.fact_id)
    lr = 1e-7   # the step is timed, not the learning: a small rate keeps the weights in range
    for _ in range(args.warmup):
        F.flern_train_step(gq.ctx, q, 0, -1, lr)
    torch.cuda.synchronize()
    step_ms, rows = [], 0
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0e.record(stream)
        for _ in range(args.steps):
            r = F.flern_train_step(gq.ctx, q, 0, -1, lr)
            step_ms.append(r.elapsed_ms)
            rows += r.rows_joined
        t1e.record(stream)
        torch.cuda.synchronize()
    ms_per_step = t0e.elapsed_time(t1e) / args.steps
    value = rows / args.steps / (ms_per_step / 1e3)
    # e2e: every step copies the shard from pinned host memory into a table (flern_update_table) and trains
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in db.fact.items()}
    tid = F.flern_load_table(gq.ctx, "fact_e2e", pinned, F.FLERN_COPY_HOST)
    qe = gq.make_query(tid)
    t0 = time.perf_counter()
    for _ in range(max(1, args.e2e_steps)):
        F.flern_update_table(gq.ctx, tid, pinned, F.FLERN_COPY_HOST)
        F.flern_train_step(gq.ctx, qe, 0, -1, lr)
    e2e_s = (time.perf_counter() - t0) / max(1, args.e2e_steps)
    tf_peak, hbm_peak, peak_src = peaks()
    avg = sum(step_ms) / len(step_ms)
    rows_step = rows // args.steps
    primary, secondary = binding_roofline(train_flops_per_row(cfg.dims), rows_step, fact_bytes, avg, tf_peak, hbm_peak,
                                          f"{peak_src} (burst)", f"{peak_src} (copy bandwidth)")
    line = {"metric": TRAIN_METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOADS["train"], "sf_per_gpu": sf1, "rows_per_gpu": db.fact_n,
                       "rows_trained_per_step": rows_step, "lr": lr,
                       "l2": "no flush: inputs larger than L2 (fact columns %.0f MB/GPU > 126 MB)" % (fact_bytes / 1e6)},
            "roofline": {**primary, "traffic": None, "kernel": "flern_train_kernel + train_update_kernel",
                         "avg_launch_ms": avg, "timing": timing_stats(step_ms), "other": secondary},
            "e2e": {"value": rows_step / e2e_s, "unit": "rows/s", "h2d_bytes_per_step": fact_bytes,
                    "d2h_bytes_per_step": 24},
            "gpu_launches": args.steps * 2, "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        import oracle as O
        n = min(db.fact_n, 20000)
        t0 = time.perf_counter()
        ro = O.train_step(cfg, db, model, lr, 0, n)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": ro["batch"] / dt, "unit": "rows/s", "cores": 1, "kind": "oracle",
                                "sample": f"first {n} lineitem rows: batch export + fp64 SGD step, 1 thread, {dt:.1f} s"}
    print(json.dumps(line), flush=True)
    gq.close()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    cfg, sf1 = workload_cfg(args.workload, world)
    strong = args.workload in STRONG
    # C5 (SF100): a prefix of rank 0's shard (its orders rows restricted to the same slots give the same
    # join), so the host holds a bounded sample; the oracle's map build is over those orders only
    db = make_db(args.workload, cfg, rank=0, world=world, max_slots=2_000_000 if strong else None)
    model = bench_model(args.workload, cfg)
    threads = os.cpu_count() or 1
    if args.workload == "train":   # the oracle's training step (single-threaded fp64) on a bounded batch
        rows = min(db.fact_n, 20000)
        t_total, trained = 0.0, 0
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            r = O.train_step(cfg, db, model, 1e-6, 0, rows)
            if i >= args.warmup:
                t_total += time.perf_counter() - t0
                trained += r["batch"]
        value = trained / t_total
        print(json.dumps({
            "impl": "reference", "metric": TRAIN_METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS["train"], "sf_per_gpu": sf1, "rows_per_gpu": db.fact_n},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {rows} lineitem rows per step (batch export + fp64 SGD step, 1 thread)"},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    # bounded sample per step: ~ (budget / (W+K)) seconds of oracle work each
    probe = min(db.fact_n, 1000 * threads)
    t0 = time.perf_counter()
    O.run(cfg, db, model, nthreads=threads, row_lo=0, row_hi=probe)
    rate = probe / max(1e-3, time.perf_counter() - t0)
    per_step_s = min(20.0, 150.0 / max(1, args.steps + args.warmup))
    rows = int(min(db.fact_n, max(1000, rate * per_step_s)))
    for i in range(args.warmup):
        O.run(cfg, db, model, nthreads=threads, row_lo=0, row_hi=rows)
    scored, t_total = 0, 0.0
    for i in range(args.steps):
        lo = (i * rows) % max(1, db.fact_n - rows + 1)
        t0 = time.perf_counter()
        r = O.run(cfg, db, model, nthreads=threads, row_lo=lo, row_hi=lo + rows)
        t_total += time.perf_counter() - t0
        scored += r.rows_joined
    value = scored / t_total
    sample = f"{rows} consecutive lineitem rows per step of {db.fact_n} ({args.workload}), {threads} threads"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "sf_per_gpu": sf1, "rows_per_gpu": db.fact_n,
                   "parallelism": f"oracle on rank 0 host cores (N={world})"},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="flern", choices=["flern", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-model", action="store_true", help="diagnostic: FLERN_Q_NO_MODEL (scan/probe/gather/aggregate only)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2311_02781_b200 import dist as FD
    from paper_2311_02781_b200 import flern as F
    from paper_2311_02781_b200.session import GpuQuery

    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("run N>1 under torchrun (python -m torch.distributed.run --nproc-per-node N ...)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    cfg, sf1 = workload_cfg(args.workload, world)
    device = f"cuda:{local}"
    strong = args.workload in STRONG
    t_gen = time.perf_counter()
    if strong:
        # SF100: the shard is generated chunk by chunk straight into HBM; the orders table is drawn in
        # slot shares and assembled on every GPU by an NCCL all_gather (replicated build side)
        from datagen import device as DD
        slo, shi = D.shard_slots(cfg.sf, rank, world)
        n_fact, fact_dev = DD.fact_to_device(cfg, slo, shi, device)
        db = D.Database(cfg.sf, n_fact, fact_dev, DD.builds_to_device(cfg, device, rank, world))
        # host rows for the e2e leg and the cpu_baseline sample: a prefix of the shard (bounded host memory)
        host = D.make_database(cfg, rank=rank, world=world, max_slots=min(shi - slo, 10_000_000))
    else:
        db = host = make_db(args.workload, cfg, rank=rank, world=world)
        # fact shard resident in HBM (torch tensors borrowed by the library, no copy)
        fact_dev = {k: torch.from_numpy(v).to(device) for k, v in db.fact.items()}
    gen_s = time.perf_counter() - t_gen
    model = bench_model(args.workload, cfg)
    gq = GpuQuery(cfg, db, model, device=local, stream=stream.cuda_stream, load_fact=False)
    gq.set_fact(F.flern_load_table(gq.ctx, "fact", fact_dev, F.FLERN_BORROW_DEVICE))
    fact_bytes = sum(v.numel() * 4 for v in fact_dev.values())
    if args.workload == "train":
        return run_train(args, cfg, sf1, db, model, gq, fact_bytes, world, rank, local, stream)
    G = cfg.ngroups
    out_count = torch.zeros(G, dtype=torch.int64, device=device)
    out_sum = torch.zeros(G, dtype=torch.int64, device=device)
    counters = torch.zeros(4, dtype=torch.int64, device=device)
    partial = torch.zeros(2 * G, dtype=torch.int64, device=device)
    q_async = gq.make_query(gq.fact_id, flags=F.FLERN_Q_RESULT_DEVICE | F.FLERN_Q_ASYNC |
                            (F.FLERN_Q_NO_MODEL if args.no_model else 0))

    # rows scored by this rank (deterministic): one synchronous run
    r0 = gq.run(gq.make_query(gq.fact_id), count=np.zeros(G, np.int64), sum=np.zeros(G, np.int64))
    rows_scored_rank = int(r0.rows_scored)

    def step(ev_pair=None):
        if ev_pair:
            ev_pair[0].record(stream)
        F.flern_run_query(gq.ctx, q_async, count=out_count, sum=out_sum, counters=counters)
        if ev_pair:
            ev_pair[1].record(stream)
        if world > 1:   # the one exchange step: NCCL reduce of the int64 group partials
            FD.combine_partials(FD.pack_partials(out_count, out_sum, partial), dst=0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b in evs]
    t = torch.tensor([ms_total, float(rows_scored_rank)], dtype=torch.float64, device=device)
    if world > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        rows_all = t[1:].clone()
        dist.all_reduce(rows_all, op=dist.ReduceOp.SUM)
        ms_total, rows_total = float(tmax.item()), float(rows_all.item())
    else:
        rows_total = float(rows_scored_rank)
    ms_per_step = ms_total / args.steps
    value = rows_total / (ms_per_step / 1e3)

    # ---- end to end through the public API with host buffers (pinned), every step: H2D of the step's
    #      fact rows + query + D2H of the result. Rows: this rank's shard (C5: a prefix of it, so the host
    #      holds a bounded sample; the metric is a rate)
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in host.fact.items()}
    h2d = sum(v.numel() * 4 for v in pinned.values())
    host_count, host_sum = np.zeros(G, np.int64), np.zeros(G, np.int64)
    d2h = 2 * G * 8 + 4 * 8

    verbose = bool(os.environ.get("FLERN_E2E_VERBOSE"))
    # every step streams the shard from pinned host memory (the step's H2D) through the library's ring of
    # device chunk buffers, runs the query chunk by chunk and reads the result back (D2H); the e2e fact
    # table is a schema with no rows (flern_run_query_streamed)
    e2e_tid = F.flern_load_table(gq.ctx, "fact_e2e", {k: np.zeros(0, v.dtype) for k, v in host.fact.items()})
    e2e_q = gq.make_query(e2e_tid)

    # 8 chunks: each chunk's H2D copy (second stream) overlaps the previous chunk's query (the paper's §3.2)
    chunk = max(4, (host.fact_n + 7) // 8)

    def e2e_step():
        t0 = time.perf_counter()
        r = F.flern_run_query_streamed(gq.ctx, e2e_q, pinned, chunk, count=host_count, sum=host_sum)
        if verbose:
            print(f"e2e: streamed step {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr)
        return r

    for _ in range(2):
        e2e_rows = int(e2e_step().rows_scored)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    et = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    er = torch.tensor([float(e2e_rows)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dist.all_reduce(er, op=dist.ReduceOp.SUM)
    e2e_value = float(er.item()) / float(et.item())

    if rank == 0:
        tf_peak, hbm_peak, peak_src = peaks()
        peak_kind = "burst"
        fpr = 0 if args.no_model else flops_per_row(cfg.dims)   # --no-model runs no MLP
        avg_kernel_ms = sum(kernel_ms) / len(kernel_ms)
        tf_src = peak_src
        if avg_kernel_ms > 50.0:   # a launch this long runs under the power cap: the sustained figure
            tf_peak, tf_src = sustained_peak()
            peak_kind = "sustained"
        # algorithmic HBM bytes per launch: every staged fact column once; with a
        # pre-filter, the filter column for every row plus the other columns of the scored rows only
        # (build side and weights not counted: a lower bound, so `achieved` is conservative)
        if cfg.prefilter:
            pf_name = cfg.prefilter[0]
            other = sum(4 for k in db.fact if k != pf_name)
            alg_bytes = 4 * db.fact_n + other * rows_scored_rank
        else:
            alg_bytes = fact_bytes
        # + the build side touched once: the key and payload columns the query reads, for
        # the build rows this rank's shard references (orders: its slot share; other build tables: all rows;
        # with a pre-filter at most one per scored row)
        build_bytes = 0
        for pi, (bt, nb, cols) in enumerate(db.builds):
            touched = nb // world if pi == 0 else nb
            if cfg.prefilter:
                touched = min(touched, rows_scored_rank)
            build_bytes += 4 * len(cfg.build_cols(pi)) * touched
        alg_bytes += build_bytes
        primary, secondary = binding_roofline(fpr, rows_scored_rank, alg_bytes, avg_kernel_ms, tf_peak, hbm_peak,
                                              f"{tf_src} ({peak_kind})", f"{peak_src} (copy bandwidth)")
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(args.workload)
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "sf_per_gpu": sf1, "rows_per_gpu": db.fact_n,
                       "rows_scored_per_gpu": rows_scored_rank,
                       "l2": "no flush: inputs larger than L2 (fact columns %.0f MB/GPU > 126 MB)" % (fact_bytes / 1e6),
                       "parallelism": f"dp{world}: fact sharded by orderkey range, orders + weights replicated, "
                                      "NCCL reduce of int64 group partials",
                       "build_ms": gq.build_ms, "datagen_s": round(gen_s, 1),
                       "e2e_sample": f"{host.fact_n} of {db.fact_n} fact rows per GPU streamed per step"},
            "roofline": {**primary, "traffic": traffic,
                         "kernel": "flern_query_wide_kernel" if max(cfg.dims[1:-1]) > 256 else "flern_query_kernel",
                         "avg_launch_ms": avg_kernel_ms, "timing": timing_stats(kernel_ms), "other": secondary},
            "e2e": {"value": e2e_value, "unit": "rows/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps * F.flern_query_launches(),
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            # C5: a 2M-slot prefix, so the oracle's map build (part of its timed run) stays small
            line["cpu_baseline"] = cpu_baseline(cfg, D.make_database(cfg, max_slots=2_000_000) if strong else host,
                                                model)
        print(json.dumps(line), flush=True)
    gq.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
