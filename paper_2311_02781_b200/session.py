"""Wire a query configuration onto the C ABI: load tables, register the model UDF, build the
hash tables, marshal the query. Marshalling only — every step of the query runs in
libflern.so's kernels.

`cfg` is any object with the attributes of datagen.QueryConfig (probes, feats, group, ngroups,
sum_col, threshold, prefilter, build_cols(p)); `db` has .fact (dict of columns), .builds
([(name, nrows, {col: array})]); `model` has dims, W, b, shift, scale.
"""
from __future__ import annotations

import time

from . import flern as F


def _src(s):
    return -1 if s == "fact" else int(s)


class GpuQuery:
    def __init__(self, cfg, db, model, device: int = 0, stream: int | None = None,
                 fact_flags: int = F.FLERN_COPY_HOST, load_fact: bool = True):
        self.cfg = cfg
        self.ctx = F.flern_create(device, stream)
        self.fact_id = None
        if load_fact:
            self.fact_id = F.flern_load_table(self.ctx, "fact", db.fact, fact_flags)
        self.build_ids, self.ht_ids = [], []
        self.build_ms = 0.0   # flern_build_hashtable wall time (synchronous), all probes
        for p, (bt, src, key, bkey) in enumerate(cfg.probes):
            name, nrows, cols = db.builds[p]
            first = next(iter(cols.values()))
            on_dev = getattr(first, "is_cuda", False)   # device tensors (datagen.device) are borrowed in place
            tid = F.flern_load_table(self.ctx, f"{name}#{p}", cols, F.FLERN_BORROW_DEVICE if on_dev else F.FLERN_COPY_HOST)
            payload = [c for c in cfg.build_cols(p) if c != bkey]
            self.build_ids.append(tid)
            t0 = time.perf_counter()
            flags = F.FLERN_HT_MULTI if p in getattr(cfg, "multi", ()) else 0
            self.ht_ids.append(F.flern_build_hashtable_ex(self.ctx, tid, bkey, payload, flags))
            self.build_ms += 1e3 * (time.perf_counter() - t0)
        self.model_id = F.flern_load_model(self.ctx, "udf", model.dims, model.W, model.b, model.shift, model.scale)
        self.query = self.make_query(self.fact_id)

    def make_query(self, fact_id, threshold=None, flags=0):
        cfg = self.cfg
        probes = [(self.ht_ids[p], _src(src), key) for p, (bt, src, key, bkey) in enumerate(cfg.probes)]
        feats = [(_src(s), c) for s, c in cfg.feats]
        return F.Query(fact_id if fact_id is not None else -1, probes, self.model_id, feats,
                       (_src(cfg.group[0]), cfg.group[1]), cfg.ngroups, (_src(cfg.sum_col[0]), cfg.sum_col[1]),
                       threshold=cfg.threshold if threshold is None else threshold, prefilter=cfg.prefilter,
                       flags=flags)

    def set_fact(self, fact_id):
        self.fact_id = fact_id
        self.query.q.fact_table = fact_id

    def run(self, query=None, **kw):
        return F.flern_run_query(self.ctx, query or self.query, **kw)

    def close(self):
        if self.ctx:
            F.flern_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
