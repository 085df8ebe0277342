"""The multi-GPU exchange protocol, world_size 2 and 4
over torch.distributed gloo on CPU: every rank ranks its shard (oracle), sends
its head K as records + a header through one all-gather, merges the runs and
cuts against the global budget; the admitted sets must equal one oracle step
over the union pool.  This checks the decomposition the CUDA merge kernel
implements (the kernel itself is checked on a B200 in test_multigpu_gpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from shard_util import restrict, split_kv, union_and_shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _blk(n, B):
    return -(-n // B)


def _worker(rank, world, port, cname, cap_l, n_union, kv_union, K, q):
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    cfg_l, cfg_u, u, shards = union_and_shards(cname, world, cap_l, n_union, max_batch=K)
    kvs = split_kv(kv_union, world)
    o = O.OraclePool(cfg_l)
    sh = shards[rank]
    o.load(sh, sh["next_id"])
    B = cfg_l["block_tokens"]
    r = o.step(kv_total=kvs[rank])  # local ranking (its local admission is not used)
    slot_of = {int(i): k for k, i in enumerate(o.pool["id"])}
    head = []
    for i in range(min(len(r["ranked_id"]), K)):
        lid = int(r["ranked_id"][i])
        head.append((int(r["ranked_starving"][i]), int(r["ranked_score"][i]), lid * world + rank,
                     _blk(int(o.pool["ctx"][slot_of[lid]]) + 1, B)))
    hdr = (int(r["pinned"]), kvs[rank], len(head), int(r["n_eligible"]))
    gathered = [None] * world
    dist.all_gather_object(gathered, (hdr, head))
    budget = max(sum(h[1] for h, _ in gathered) - sum(h[0] for h, _ in gathered), 0)
    merged = sorted((rec for _, recs in gathered for rec in recs), key=lambda x: (-x[0], x[1], x[2]))[:K]
    used, adm = 0, []
    for rec in merged:
        if used + rec[3] > budget:
            break
        used += rec[3]
        adm.append(rec[2])
    q.put((rank, [g // world for g in adm if g % world == rank], budget, used))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cname,cap_l,n_union,kv_union,K", [
    (2, "C2", 2048, 1800, 3000, 256), (4, "C3", 1024, 3000, 640, 64), (2, "C4", 65536, 100000, 10000, 1024)])
def test_gloo_exchange_equals_union(world, cname, cap_l, n_union, kv_union, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cname, cap_l, n_union, kv_union, K, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, adm, budget, used = q.get(timeout=300)
        res[rank] = (adm, budget, used)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg_l, cfg_u, u, _ = union_and_shards(cname, world, cap_l, n_union, max_batch=K)
    ou = O.OraclePool(cfg_u)
    ou.load(u, u["next_id"])
    ro = ou.step(kv_total=kv_union)
    for r in range(world):
        adm, budget, used = res[r]
        assert adm == list(restrict(ro["admitted_id"], world, r))
        assert budget == ro["budget"] and used == ro["budget_used"]
