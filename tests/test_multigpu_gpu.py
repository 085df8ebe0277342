"""Multi-GPU global admission on one device through the loopback
transport: `world` shards step together (lamps_group_step); the exchange is a
device copy instead of the NCCL all-gather, the merge kernel is the one the
NCCL path runs.  Every shard must equal one oracle step over the union pool."""
import numpy as np
import pytest

import gen
import oracle as O
from shard_util import FIELDS, restrict, split_kv, union_and_shards

pytestmark = pytest.mark.gpu


def run(cname, world, cap_l, n_union, kv_union, steps=3, seed=0, p2p=False, head_only=False, **over):
    from paper_2410_18248_b200 import Scheduler
    from paper_2410_18248_b200.lamps import LAMPS_SHARE_DEVICE, LAMPS_XPORT_LOOPBACK, LAMPS_XPORT_P2P
    import torch
    cfg_l, cfg_u, u, shards = union_and_shards(cname, world, cap_l, n_union, seed=seed, **over)
    if p2p:  # peer-memory exchange inside the step kernel; ranks co-resident on this device
        S = [Scheduler(cfg_l, world=world, rank=r, transport=LAMPS_XPORT_P2P,
                       flags=LAMPS_SHARE_DEVICE | (64 if head_only else 0),  # 64 = LAMPS_HEAD_ONLY
                       stream=torch.cuda.Stream()) for r in range(world)]
        Scheduler.p2p_connect_local(S)
    else:
        stream = torch.cuda.current_stream()
        S = [Scheduler(cfg_l, world=world, rank=r, transport=LAMPS_XPORT_LOOPBACK, stream=stream)
             for r in range(world)]
    for r in range(world):
        S[r].import_pool(shards[r], shards[r]["id_base"], shards[r]["next_id"])
    o = O.OraclePool(cfg_u)
    o.load(u, u["next_id"])
    kvs = split_kv(kv_union, world)
    for t in range(steps):
        outs = Scheduler.group_step(S, None, kvs)
        ro = o.step(kv_total=kv_union)
        assert ro["rc"] == 0
        for r in range(world):
            g = outs[r]
            where = f"{cname} W={world} t={t} r={r}"
            assert list(g["admitted_id"]) == list(restrict(ro["admitted_id"], world, r)), where
            assert list(g["preempted_id"]) == list(restrict(ro["preempted_id"], world, r)), where
            assert g["budget"] == ro["budget"] and g["budget_used"] == ro["budget_used"], where
            assert g["blocked_head"] == ro["blocked_head"], where
            # local ranked order == global order restricted to the shard (a prefix of it when
            # only the head is ranked)
            ids, score, starv = S[r].decode_keys(S[r].ranked_keys(), g["id_base"])
            mine = ro["ranked_id"] % world == r
            m = len(ids)
            assert head_only or m == int(mine.sum()), where
            assert np.array_equal(ids, (ro["ranked_id"][mine] // world)[:m]), where
            assert np.array_equal(score, ro["ranked_score"][mine][:m]), where
            assert np.array_equal(starv, ro["ranked_starving"][mine][:m]), where
            # whole shard state == union state restricted
            e = S[r].export_pool()
            P = o.pool
            live = (P["state"] != 0) & (P["id"].astype(np.int64) % world == r)
            lids = P["id"][live].astype(np.int64) // world
            for f in FIELDS:
                assert np.array_equal(e[f][lids % cap_l], P[f][live].astype(np.uint32)), (where, f)
        assert sum(x["n_admitted"] for x in outs) == ro["n_admitted"]
    for s in S:
        s.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_loopback_merge_c2(world):
    run("C2", world, 2048, 1800, 3000, max_batch=256)


@pytest.mark.parametrize("world,cap_l", [(2, 65536), (8, 16384)])
def test_loopback_merge_c4(world, cap_l):
    run("C4", world, cap_l, 100000, 10000, max_batch=1024)


@pytest.mark.parametrize("world,cap_l,K", [(4, 32768, 4096), (8, 16384, 8192)])
def test_loopback_merge_large_k(world, cap_l, K):
    # world * K records beyond one CTA's shared memory (global max_batch 8192
    # over 8 shards): the grid-wide merge by rank (k_merge_count / k_merge_place / k_merge_cut)
    run("C4", world, cap_l, 100000, 1_000_000, max_batch=K)


def test_loopback_merge_tight_budget_and_small_k():
    run("C3", 4, 1024, 3000, 80, max_batch=7)


def test_loopback_merge_empty_shard():
    # a union of 3 requests over 4 shards: one shard has nothing
    run("C1", 4, 16, 3, 292, max_batch=16)


def test_nccl_one_rank_merge_path():
    """LAMPS_MERGE at world 1: the NCCL exchange (dlopen'd libnccl, a 1-rank
    communicator, ncclAllGather) + merge kernel, stepped with events, against the oracle."""
    import torch
    from paper_2410_18248_b200 import LAMPS_MERGE, Scheduler
    cfg = gen.lib_config("C2")
    snap = gen.snapshot("C2", seed=3, id_base=77)
    s = Scheduler(cfg, flags=LAMPS_MERGE, world=1, rank=0, nccl_id=Scheduler.nccl_unique_id(),
                  stream=torch.cuda.current_stream())
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    o = O.OraclePool(cfg)
    o.load(snap, snap["next_id"])
    kv = gen.CONFIGS["C2"]["kv_total"]
    prev = np.zeros(0, np.int64)
    from paper_2410_18248_b200.lamps import EVENT_DTYPE
    for t in range(4):
        ev = np.zeros(min(3, len(prev)), EVENT_DTYPE)
        for j in range(len(ev)):
            ev[j]["id"], ev[j]["kind"] = prev[j], 2 if j == 0 else 1
        g = s.step(ev, kv)
        oev = np.zeros(len(ev), O.EVENT_DTYPE)
        oev["id"], oev["kind"] = ev["id"], ev["kind"]
        ro = o.step(oev, kv_total=kv)
        assert list(g["admitted_id"]) == list(ro["admitted_id"]), t
        assert list(g["preempted_id"]) == list(ro["preempted_id"]), t
        assert g["budget"] == ro["budget"] and g["budget_used"] == ro["budget_used"], t
        prev = np.asarray(g["admitted_id"], np.int64)
    assert s.stats()[0] == 1 + 1  # fused (events in its prologue) + merge
    s.close()


# ---- peer-memory transport: records stored into every rank's buffer, flags, merge and
# admission inside the fused step kernel (one kernel per rank per step)
@pytest.mark.parametrize("world", [2, 4])
def test_p2p_merge_c2(world):
    run("C2", world, 2048, 1800, 3000, max_batch=256, p2p=True, steps=4)


def test_p2p_merge_c4():
    run("C4", 2, 65536, 100000, 10000, max_batch=1024, p2p=True)


def test_p2p_merge_w4_k2048():
    # 4 ranks x 2048 records: the largest exchange the in-kernel merge stages on chip
    run("C4", 4, 32768, 100000, 200000, max_batch=2048, p2p=True)


def test_p2p_merge_tight_budget_and_small_k():
    run("C3", 4, 1024, 3000, 80, max_batch=7, p2p=True, steps=5)


def test_p2p_self_exchange_world1():
    """world 1 over the peer-memory path: identical to the plain single-shard step."""
    from paper_2410_18248_b200 import Scheduler
    from paper_2410_18248_b200.lamps import LAMPS_XPORT_P2P
    cfg = gen.lib_config("C3")
    snap = gen.snapshot("C3", seed=2, id_base=77)
    a = Scheduler(cfg)
    b = Scheduler(cfg, transport=LAMPS_XPORT_P2P, flags=32)  # LAMPS_MERGE
    for s in (a, b):
        s.import_pool(snap, snap["id_base"], snap["next_id"])
    for t in range(4):
        ga, gb = a.step(kv_total=640), b.step(kv_total=640)
        for k in ("n_eligible", "budget", "budget_used", "n_admitted", "n_preempted", "blocked_head"):
            assert ga[k] == gb[k], (t, k)
        assert np.array_equal(ga["admitted_id"], gb["admitted_id"])
        assert np.array_equal(ga["preempted_id"], gb["preempted_id"])
    assert b.stats()[0] == 1  # one kernel: exchange and merge inside k_fused
    a.close(); b.close()


def test_p2p_merge_head_only():
    """F3 head-only ranking on every rank + the peer-memory exchange: the same global batch."""
    run("C2", 2, 2048, 1800, 3000, max_batch=256, p2p=True, head_only=True, steps=4)


def _p2p_group(cfg, world):
    import torch
    from paper_2410_18248_b200 import Scheduler
    from paper_2410_18248_b200.lamps import LAMPS_SHARE_DEVICE, LAMPS_XPORT_P2P
    S = [Scheduler(cfg, world=world, rank=r, transport=LAMPS_XPORT_P2P, flags=LAMPS_SHARE_DEVICE,
                   stream=torch.cuda.Stream()) for r in range(world)]
    Scheduler.p2p_connect_local(S)
    return S


def test_shared_device_rank_iterate_refused_before_staging():
    """lamps_iterate on a world>1 LAMPS_SHARE_DEVICE rank is refused before any
    return / arrival is staged -- pool, id window and the next group step are unchanged."""
    from paper_2410_18248_b200.lamps import LAMPS_EINVAL
    cfg_l, cfg_u, u, shards = union_and_shards("C2", 2, 2048, 1800)
    S, T = _p2p_group(cfg_l, 2), _p2p_group(cfg_l, 2)
    for G in (S, T):
        for r in range(2):
            G[r].import_pool(shards[r], shards[r]["id_base"], shards[r]["next_id"])
    kvs = split_kv(3000, 2)
    before = S[0].export_pool()
    arr = S[0].segments([dict(prompt_len=50, pre_len=10, resp_len=5, post_len=7, api_seconds=0.5,
                              has_api=1)] * 3)
    rc, out, ids = S[0].iterate_rc(arrivals=arr, kv_total=kvs[0])
    assert rc == LAMPS_EINVAL and out is None
    after = S[0].export_pool()
    for f in FIELDS:
        assert np.array_equal(before[f], after[f]), f
    a = type(S[0]).group_step(S, None, kvs)
    b = type(S[0]).group_step(T, None, kvs)
    for r in range(2):
        assert np.array_equal(a[r]["admitted_id"], b[r]["admitted_id"])
    # the id window did not move: the next arrivals get the same ids on both groups
    sa = S[0].submit(arr)
    sb = T[0].submit(arr)
    assert np.array_equal(sa, sb)
    for s in S + T:
        s.close()


def test_group_step_refused_shard_stages_nothing():
    """a group step in which one shard's events are invalid is refused before any
    shard is staged; the same group then steps exactly like a twin that never saw the call."""
    from paper_2410_18248_b200 import Scheduler
    from paper_2410_18248_b200.lamps import EVENT_DTYPE, LampsError, LAMPS_XPORT_LOOPBACK
    import torch
    cfg_l, cfg_u, u, shards = union_and_shards("C2", 2, 2048, 1800)
    stream = torch.cuda.current_stream()
    G = [[Scheduler(cfg_l, world=2, rank=r, transport=LAMPS_XPORT_LOOPBACK, stream=stream) for r in range(2)]
         for _ in range(2)]
    for S in G:
        for r in range(2):
            S[r].import_pool(shards[r], shards[r]["id_base"], shards[r]["next_id"])
    kvs = split_kv(3000, 2)
    first = [Scheduler.group_step(S, None, kvs) for S in G]
    ev = []
    for r in range(2):
        e = np.zeros(2, EVENT_DTYPE)
        e["id"], e["kind"] = first[0][r]["admitted_id"][:2], 2  # FINISHED
        ev.append(e)
    bad = [ev[0], ev[1].copy()]
    bad[1]["id"][0] = 1 << 40  # not admitted by shard 1's previous step
    with pytest.raises(LampsError):
        Scheduler.group_step(G[0], bad, kvs)
    for S in G:  # shard 0's FINISHED events must not have been half-applied
        out = Scheduler.group_step(S, ev, kvs)
        S.append(out)
    for r in range(2):
        assert np.array_equal(G[0][2][r]["admitted_id"], G[1][2][r]["admitted_id"])
        e0, e1 = G[0][r].export_pool(), G[1][r].export_pool()
        for f in FIELDS:
            assert np.array_equal(e0[f], e1[f]), (r, f)
    for S in G:
        for s in S[:2]:
            s.close()
