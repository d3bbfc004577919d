"""a8 (cross-GPU combine) with the CUDA kernel on every rank (`-m gpu`).

Each rank runs flern_run_query (the fused kernel, through the C ABI) on its contiguous orderkey shard of
the fact table, with the orders table and the weights replicated, and paper_2311_02781_b200.dist sums the
int64 group partials across ranks. The combined aggregates must equal the single-process, unsharded GPU
result bit-exactly (every row's score is computed independently of the tile it lands in), and agree with
the oracle: exactly with the linear-threshold model (no row in the band), within the band bracket with the
random model.
  - two ranks sharing one GPU over gloo (runs on any box with one GPU);
  - one rank per GPU over NCCL (skipped with fewer than 2 GPUs)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg(kind):
    import datagen as D
    return D.with_sf(D.CONFIGS["c2"], 0.02, match_rate=0.9)


def _model(cfg, kind):
    import datagen as D
    from tests import helpers as H
    return H.linear_threshold_model(cfg) if kind == "linear" else D.make_model(cfg, D.make_database(cfg, max_slots=D.MODEL_SLOTS))


def _worker(rank, world, port, backend, kind, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import datagen as D
    from paper_2311_02781_b200 import dist as FD
    from paper_2311_02781_b200.session import GpuQuery
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg(kind)
        shard = D.make_database(cfg, rank=rank, world=world)
        gq = GpuQuery(cfg, shard, _model(cfg, kind), device=dev)
        G = cfg.ngroups
        cnt = torch.zeros(G, dtype=torch.int64, device=f"cuda:{dev}")
        sm = torch.zeros(G, dtype=torch.int64, device=f"cuda:{dev}")
        ctr = torch.zeros(4, dtype=torch.int64, device=f"cuda:{dev}")
        from paper_2311_02781_b200 import flern as F
        gq.run(gq.make_query(gq.fact_id, flags=F.FLERN_Q_RESULT_DEVICE), count=cnt, sum=sm, counters=ctr)
        buf = FD.pack_partials(cnt, sm)
        FD.combine_partials(buf, dst=None)
        c, s = FD.unpack_partials(buf)
        joined = torch.tensor([int(ctr[1].item())], dtype=torch.int64, device=f"cuda:{dev}")
        FD.combine_partials(joined, dst=None)
        gq.close()
        q.put((rank, c.cpu().tolist(), s.cpu().tolist(), int(joined.item()), shard.fact_n))
    finally:
        dist.destroy_process_group()


def _run(world, backend, kind):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out)


def _check(out, kind):
    import datagen as D
    import oracle as O
    from tests import parity
    cfg = _cfg(kind)
    full = D.make_database(cfg)
    model = _model(cfg, kind)
    assert sum(o[4] for o in out) == full.fact_n
    g = parity.run_gpu(cfg, full, model, debug=False)   # one process, unsharded
    o = O.run(cfg, full, model, band=parity.BAND)
    for rank, c, s, joined, _ in out:   # every rank holds the combined result (all_reduce)
        assert c == g["count"].tolist() and s == g["sum"].tolist(), rank
        assert joined == g["rows_joined"] == o.rows_joined
        assert np.all(o.count_hi <= c) and np.all(np.asarray(c) <= o.count_hi + o.count_band)
        assert np.all(o.sum_hi <= s) and np.all(np.asarray(s) <= o.sum_hi + o.sum_band)
        if kind == "linear":
            assert o.rows_band == 0 and c == o.count.tolist() and s == o.sum.tolist()


@pytest.mark.parametrize("kind", ["linear", "random"])
def test_two_ranks_one_gpu_gloo(kind):
    _check(_run(2, "gloo", kind), kind)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ranks_per_gpu_nccl(world):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    for kind in ("linear", "random"):
        _check(_run(world, "nccl", kind), kind)
