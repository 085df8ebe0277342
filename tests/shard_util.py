"""Union pool <-> shards for the multi-GPU tests.

Shard r of `world` owns the global ids g with g % world == r; its local id is
g // world.  A union snapshot with ids starting at
world * B0 maps to shard snapshots with local ids starting at B0.
"""
import numpy as np

import gen
import oracle as O

FIELDS = ("state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem", "api_ticks",
          "resp_len", "post_len", "pending")


def union_and_shards(cname, world, cap_l, n_union, seed=0, B0=1000, **over):
    cfg_l = gen.lib_config(cname, **over)
    cfg_l["capacity"] = cap_l
    cfg_l["id_bits"] = max(cfg_l["id_bits"], (cap_l - 1).bit_length())
    cfg_u = dict(cfg_l)
    cfg_u["capacity"] = world * cap_l
    cfg_u["id_bits"] = max(cfg_l["id_bits"], (world * cap_l - 1).bit_length())
    u = gen.snapshot(cname, seed=seed, n=n_union, capacity=world * cap_l, id_base=world * B0)
    shards = []
    for r in range(world):
        f = {k: np.zeros(cap_l, np.int64) for k in ("id",) + FIELDS}
        f["strategy"][:] = O.NONE
        live = (u["state"] != 0) & (u["id"] % world == r)
        gids = u["id"][live]
        lids = gids // world
        for k in FIELDS:
            f[k][lids % cap_l] = u[k][live]
        f["id"][lids % cap_l] = lids
        nxt = int(lids.max()) + 1 if len(lids) else B0
        f.update(id_base=B0, next_id=nxt, capacity=cap_l)
        shards.append(f)
    return cfg_l, cfg_u, u, shards


def split_kv(kv_union, world):
    base = [kv_union // world] * world
    base[0] += kv_union - sum(base)
    return base


def restrict(ids, world, r):
    ids = np.asarray(ids, np.int64)
    return ids[ids % world == r] // world
