"""Multi-rank host logic on CPU (gloo, world size 2): each rank takes its contiguous orderkey
shard of the fact table (the sharding bench.py uses), computes its per-group partials with the
oracle (stand-in for the GPU kernel on this GPU-less box), and the partials are combined with
paper_2311_02781_b200.dist — the same calls bench.py makes over NCCL. The combined result must
equal the unsharded result bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import datagen as D
    import oracle as O
    from paper_2311_02781_b200 import dist as FD
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = D.with_sf(D.CONFIGS["c1"], 0.004, match_rate=0.9)
        model = D.make_model(cfg, D.make_database(cfg, max_slots=D.MODEL_SLOTS))   # replicated weights
        shard = D.make_database(cfg, rank=rank, world=world)
        r = O.run(cfg, shard, model, nthreads=2)
        buf = FD.pack_partials(torch.from_numpy(r.count), torch.from_numpy(r.sum))
        FD.combine_partials(buf, dst=None)
        c, s = FD.unpack_partials(buf)
        q.put((rank, c.tolist(), s.tolist(), shard.fact_n))
    finally:
        dist.destroy_process_group()


def test_sharded_partials_combine_to_unsharded_result():
    import datagen as D
    import oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = D.with_sf(D.CONFIGS["c1"], 0.004, match_rate=0.9)
    full = D.make_database(cfg)
    ref = O.run(cfg, full, D.make_model(cfg, full))
    assert sum(o[3] for o in out) == full.fact_n
    for rank, c, s, _ in out:
        assert c == ref.count.tolist() and s == ref.sum.tolist(), rank
