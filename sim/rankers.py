"""Rankers: the simulator asks one for the ranked order of the READY requests and the
handling label of every request, given the engine's pool state (lamps_pool_io
fields per slot, slot = id mod capacity)."""
from __future__ import annotations

import numpy as np


class PassRanker:
    """The CUDA pass (A0-A5 on the GPU) as the ranker: the engine's pool is imported,
    one lamps_schedule_step runs, the ranked keys and the per-slot strategy labels
    are read back.  The pass's own admission result is ignored by the unit engine
    (whose admission rule is the worked example's)."""

    def __init__(self, cfg: dict):
        from paper_2410_18248_b200 import Scheduler
        self.sched = Scheduler(cfg)
        self.cap = int(cfg["capacity"])

    def rank(self, fields: dict, id_base: int, next_id: int):
        s = self.sched
        s.import_pool(fields, id_base, next_id)
        r = s.step(kv_total=0)
        ids, _, _ = s.decode_keys(s.ranked_keys(), r["id_base"])
        e = s.export_pool()
        labels = {int(i): int(e["strategy"][int(i) % self.cap]) for i in np.asarray(fields["id"])[
            np.asarray(fields["state"]) != 0]}
        return [int(i) for i in ids], labels

    def close(self):
        self.sched.close()


class StaticRanker:
    """A fixed priority order over request ids (labels from an inner ranker)."""

    def __init__(self, order, inner):
        self.order = [int(x) for x in order]
        self.inner = inner

    def rank(self, fields: dict, id_base: int, next_id: int):
        ranked, labels = self.inner.rank(fields, id_base, next_id)
        live = set(ranked)
        return [i for i in self.order if i in live], labels
