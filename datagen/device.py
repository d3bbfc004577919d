"""Chunked generation of a fact shard and the replicated build tables straight into device memory.

Input plumbing only (no method arithmetic), for databases too large to hold on the host at once:
config C5 is SF100, 600M lineitem rows (31 GB of fact columns) at one GPU. The host generates a
bounded chunk of order slots at a time (datagen's counter-based generator: any slot range is drawn
independently) and copies it into preallocated torch tensors on the device.

Replicated build tables (orders, customer) are generated once across a process group: each rank draws
its slot share and an all_gather over NCCL assembles the full table on every GPU (the bytes equal
a single-process draw of the whole table).
"""
from __future__ import annotations

import numpy as np
import torch

from . import (SEED, QueryConfig, col_dtype, gen_customer, gen_lineitem, gen_orders, lib, num_customers,
               num_order_slots, shard_slots)

CHUNK_SLOTS = 2_000_000   # order slots per host chunk (~8M lineitem rows, ~0.4 GB at 13 columns)


def _tdtype(name):
    return torch.float32 if col_dtype(name) == np.float32 else torch.int32


def lineitem_rows(sf: float, slot_lo: int, slot_hi: int, seed: int = SEED) -> int:
    return int(lib().fg_lineitem_rows(seed, sf, slot_lo, slot_hi))


def fact_to_device(cfg: QueryConfig, slot_lo: int, slot_hi: int, device, names=None, seed: int = SEED,
                   chunk_slots: int = CHUNK_SLOTS):
    """Lineitem rows of order slots [slot_lo, slot_hi) -> {col: device tensor}; returns (nrows, cols)."""
    names = list(names or cfg.fact_cols())
    n = lineitem_rows(cfg.sf, slot_lo, slot_hi, seed)
    out = {c: torch.empty(n, dtype=_tdtype(c), device=device) for c in names}
    off = 0
    for a in range(slot_lo, slot_hi, chunk_slots):
        b = min(slot_hi, a + chunk_slots)
        m, cols = gen_lineitem(cfg.sf, names, a, b, seed=seed)
        for c in names:
            out[c][off:off + m].copy_(torch.from_numpy(cols[c]))
        off += m
    assert off == n
    return n, out


def _gather_rows(part: dict, nrows_all: list, group):
    """all_gather of row-sharded columns (ranks hold consecutive row ranges of unequal length)."""
    import torch.distributed as dist
    world = len(nrows_all)
    mx = max(nrows_all)
    out = {}
    for c, t in part.items():
        buf = torch.zeros(mx, dtype=t.dtype, device=t.device)
        buf[:t.numel()].copy_(t)
        parts = [torch.empty(mx, dtype=t.dtype, device=t.device) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out[c] = torch.cat([p[:k] for p, k in zip(parts, nrows_all)])
    return out


def builds_to_device(cfg: QueryConfig, device, rank: int = 0, world: int = 1, group=None, seed: int = SEED):
    """The query's build tables, replicated on every rank's device: [(name, nrows, {col: tensor})].
    world > 1: each rank draws its share of the order slots and an all_gather assembles the table."""
    builds = []
    for p, (bt, src, key, bkey) in enumerate(cfg.probes):
        cols = cfg.build_cols(p)
        if bt == "orders":
            total = num_order_slots(cfg.sf)
            lo, hi = shard_slots(cfg.sf, rank, world)
            m, d = gen_orders(cfg.sf, cols, match_rate=cfg.match_rate, seed=seed, slot_lo=lo, slot_hi=hi)
            part = {c: torch.from_numpy(v).to(device) for c, v in d.items()}
            if world > 1:
                import torch.distributed as dist
                cnt = torch.tensor([m], dtype=torch.int64, device=device)
                cnts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
                dist.all_gather(cnts, cnt, group=group)
                nrows_all = [int(x.item()) for x in cnts]
                part = _gather_rows(part, nrows_all, group)
                m = sum(nrows_all)
            assert total > 0
            builds.append((bt, m, part))
        elif bt == "customer":
            m, d = gen_customer(cfg.sf, cols, seed=seed)
            assert m == num_customers(cfg.sf)
            builds.append((bt, m, {c: torch.from_numpy(v).to(device) for c, v in d.items()}))
        else:
            raise ValueError(bt)
    return builds
