"""The peer-memory transport across PROCESSES (LAMPS_XPORT_P2P as bench.py uses it at
N > 1): two ranks exchange their CUDA IPC handles over torch.distributed (gloo), map each
other's exchange buffers (lamps_p2p_connect) and step; the in-kernel exchange, flags and
merge must give every rank its share of one oracle step over the union pool.  On a
single-GPU box both processes share the device and their step kernels are time-sliced
(each waits for the other's flag), which exercises the system-scope protocol; on a
multi-GPU box the same code runs over NVLink."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        import oracle as O
        from paper_2410_18248_b200 import Scheduler
        from paper_2410_18248_b200.lamps import LAMPS_XPORT_P2P
        from shard_util import restrict, split_kv, union_and_shards

        dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
        dev = rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        cfg_l, cfg_u, u, shards = union_and_shards("C2", world, 2048, 1800, max_batch=256)
        s = Scheduler(cfg_l, world=world, rank=rank, transport=LAMPS_XPORT_P2P)
        hs = [None] * world
        dist.all_gather_object(hs, s.p2p_handle())
        s.p2p_connect(hs)
        s.import_pool(shards[rank], shards[rank]["id_base"], shards[rank]["next_id"])
        o = O.OraclePool(cfg_u)
        o.load(u, u["next_id"])
        kvs = split_kv(3000, world)
        for t in range(3):
            g = s.step(kv_total=kvs[rank])
            ro = o.step(kv_total=3000)
            assert list(g["admitted_id"]) == list(restrict(ro["admitted_id"], world, rank)), (rank, t)
            assert list(g["preempted_id"]) == list(restrict(ro["preempted_id"], world, rank)), (rank, t)
            assert g["budget"] == ro["budget"] and g["budget_used"] == ro["budget_used"], (rank, t)
        assert s.stats()[0] == 1
        s.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))


@pytest.mark.timeout(300)
def test_p2p_two_processes():
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), os.environ.get("PYTHONPATH", "")])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=280) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res


def _worker_dead_peer(rank, world, port, q):
    """Rank 1 connects but never steps: rank 0's step must end (bounded wait) with
    LAMPS_ENCCL instead of hanging the GPU."""
    try:
        import time

        import torch
        import torch.distributed as dist

        os.environ["LAMPS_P2P_TIMEOUT_MS"] = "300"
        from paper_2410_18248_b200 import Scheduler
        from paper_2410_18248_b200.lamps import LAMPS_ENCCL, LAMPS_XPORT_P2P
        from shard_util import union_and_shards

        dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
        torch.cuda.set_device(rank % torch.cuda.device_count())
        cfg_l, _, _, shards = union_and_shards("C2", world, 2048, 1800, max_batch=256)
        s = Scheduler(cfg_l, world=world, rank=rank, transport=LAMPS_XPORT_P2P)
        hs = [None] * world
        dist.all_gather_object(hs, s.p2p_handle())
        s.p2p_connect(hs)
        s.import_pool(shards[rank], shards[rank]["id_base"], shards[rank]["next_id"])
        if rank == 0:
            t0 = time.time()
            rc = s.step_rc(kv_total=1500)
            dt = time.time() - t0
            assert rc == LAMPS_ENCCL, rc
            assert dt < 30, dt
        dist.barrier()
        s.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))


@pytest.mark.timeout(300)
def test_p2p_dead_peer_times_out():
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), os.environ.get("PYTHONPATH", "")])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_dead_peer, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=280) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res
