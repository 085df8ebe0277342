"""Benchmark of the LAMPS scheduling pass (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5]

One step = one lamps_schedule_step over the whole request pool: A0 events,
A1 strategy argmin, A2 memory-over-time score, A3 starvation + keys, A4 radix
sort, A5 admission.  Workload (N=1): config C5, the 1M-request
pool (2^20 slots, GPT-J profile) BASELINE.json's metric is quoted on.  Metric:
scheduling decisions/s = eligible (READY) requests decided per step / device
time per step.  Inputs are resident in HBM; L2 (126 MB) is flushed before
every timed step by writing a 256 MiB buffer (outside the timed events).

For N > 1 (torchrun) every rank owns its own 1M-request shard (weak scaling)
and the ranks admit ONE global batch: each ranks its shard, one NCCL
all-gather of the top-K records, an identical merge + cut on every rank
(DESIGN.md section 8); time is the max over ranks.

--impl reference times the CPU oracle (oracle/, plain C, one core) as it
stands on the same workload: the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# A4 (the sort) in the fused kernel: the keys to their ranges, the barrier, the range sorts
SORT_SEGS = ("range_assign", "run_offsets", "run_place", "run_store", "barrier", "l_prep", "range_sort", "store_grid")
METRIC = "scheduling decisions/s and µs per step at 1M-request pool; % HBM peak"
UNIT = "decisions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-variants", action="store_true", help="skip the policy / selective-update variants")
    ap.add_argument("--merge", action="store_true",
                    help="N=1: run the multi-shard exchange + merge path with one rank")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-shard exchange: p2p = peer stores + merge inside the step kernel "
                         "(CUDA IPC over NVLink), nccl = ncclAllGather + merge kernel")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: one 1M-request shard per GPU; strong: the 1M-request pool as --shards "
                         "shards (8 x 131072) spread over the GPUs, all shards of a GPU co-resident")
    ap.add_argument("--shards", type=int, default=8, help="strong scaling: shards of the 1M pool")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N ranks on this node (rank r -> cuda:r), rendezvous on
    127.0.0.1; rank 0 prints the JSON line.  NCCL_DEBUG=INFO unless set, so the
    communicator's rank count is in the log."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def cpu_info():
    """(host cores, CPU model) for the oracle baseline's "1 core of N"."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count(), model


class PinnedCore:
    """Run the oracle on one host core (the `taskset -c <core>` of BASELINE.md 4, applied to
    this process with sched_setaffinity; the oracle is single-threaded C called in-process)."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def n_ready(snap):
    return int((snap["state"] == 1).sum())  # READY (gen.pools)


def config_dict(cname, cfg, kv, n_elig, world, parallelism):
    """The workload description; identical in both arms (same pool, same keys)."""
    return {"workload": f"{cname}: 1M-request pool (2^20 slots), GPT-J profile, {n_elig} READY per shard"
                        if cname == "C5" else f"{cname}: {cfg['capacity']}-slot pool, {n_elig} READY per shard",
            "slots_per_gpu": cfg["capacity"], "eligible_per_gpu": n_elig, "kv_total_blocks": kv,
            "max_batch": cfg["max_batch"], "key_bits": 1 + cfg["score_bits"] + cfg["id_bits"],
            "l2": "flushed before every timed step (256 MiB write)", "parallelism": parallelism,
            "n_shards": world,
            "timed": "steady-state steps from the pool snapshot; its first step after the import, which "
                     "builds the range grid (cold, once per imported pool), runs untimed"}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import gen
    import oracle as O
    cname = args.config
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)
    kv = gen.CONFIGS[cname]["kv_total"]
    full = args.steps + args.warmup <= 60
    if not full:  # bounded sample: a 2^18-slot pool of the same workload
        cfg["capacity"] = 1 << 18
        snap = gen.snapshot(cname, seed=0, n=1 << 18, capacity=1 << 18)
    merged = world > 1 or args.merge
    conf = config_dict(cname, gen.lib_config(cname), kv, n_ready(gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)),
                       world, parallelism(world, merged, args.transport if merged else None, gen.lib_config(cname)))
    p = O.OraclePool(cfg)
    p.load(snap, snap["next_id"])
    ncores, model = cpu_info()
    with PinnedCore() as pc:
        for _ in range(args.warmup):
            p.step(kv_total=kv)
        t0 = time.perf_counter()
        ne = 0
        for _ in range(args.steps):
            r = p.step(kv_total=kv)
            ne += r["n_eligible"]
        dt = time.perf_counter() - t0
    v = ne / dt
    sample = (f"full {cname} pool ({cfg['capacity']} slots)" if full else
              f"{cname} workload, 2^18-slot sample") + f", {args.steps} oracle steps, pinned to core {pc.core}"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": conf,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "cores_total": ncores,
                             "cores_desc": f"1 core of {ncores}", "cpu_model": model, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def cpu_baseline(cname, seconds=12.0):
    import gen
    import oracle as O
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)
    p = O.OraclePool(cfg)
    p.load(snap, snap["next_id"])
    kv = gen.CONFIGS[cname]["kv_total"]
    ncores, model = cpu_info()
    with PinnedCore() as pc:
        t0 = time.perf_counter()
        n, ne = 0, 0
        while True:
            r = p.step(kv_total=kv)
            n += 1
            ne += r["n_eligible"]
            if time.perf_counter() - t0 > seconds:
                break
        dt = time.perf_counter() - t0
    return {"value": ne / dt, "unit": UNIT, "cores": 1, "cores_total": ncores, "cores_desc": f"1 core of {ncores}",
            "cpu_model": model, "kind": "oracle",
            "sample": f"{n} oracle steps over the full {cname} pool ({cfg['capacity']} slots), "
                      f"{1e3 * dt / n:.0f} ms/step, single-threaded C pinned to core {pc.core}"}


def parallelism(world, merged, transport, cfg):
    xdesc = ("peer stores into every rank's buffer + merge inside the step kernel" if transport == "p2p"
             else "NCCL all-gather + merge kernel")
    if world > 1:
        return (f"{world} shards x 1M, one exchange of the top-{cfg['max_batch']} per step for the global "
                f"admission ({xdesc})")
    return f"1 shard, exchange + merge with one rank ({xdesc})" if merged else "1 shard"


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    from paper_2410_18248_b200 import LAMPS_TIMING, Scheduler
    from paper_2410_18248_b200.lamps import EVENT_DTYPE, SEGMENT_DTYPE

    # LAMPS_BENCH_OVERSUBSCRIBE=1 (testing the N > 1 code path on a one-GPU box): ranks share
    # the devices and talk over gloo; the ranks' kernels are time-sliced, so times are not
    # meaningful
    oversub = os.environ.get("LAMPS_BENCH_OVERSUBSCRIBE") == "1"
    if oversub:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cname = args.config
    cfg = gen.lib_config(cname)
    kv = gen.CONFIGS[cname]["kv_total"]
    cap = cfg["capacity"]
    id_base = (1 << 20) * 7 + 99
    snap = gen.snapshot(cname, seed=rank, id_base=id_base)
    stream = torch.cuda.current_stream()

    from paper_2410_18248_b200.lamps import LAMPS_XPORT_NCCL, LAMPS_XPORT_P2P
    nccl_id, mflags = None, 0
    merged = world > 1 or args.merge
    transport = args.transport if merged else None
    if merged and world == 1:
        from paper_2410_18248_b200 import LAMPS_MERGE
        mflags = LAMPS_MERGE
    s = None
    if merged and transport == "p2p":
        # peer-memory exchange: every rank maps every rank's exchange buffer (CUDA IPC);
        # falls back to NCCL if the mapping is not possible on this machine
        try:
            s = Scheduler(cfg, flags=mflags, stream=stream, world=world, rank=rank, transport=LAMPS_XPORT_P2P)
            if world > 1:
                hs = [None] * world
                dist.all_gather_object(hs, s.p2p_handle())
                s.p2p_connect(hs)
                # one trial exchange (empty pool): the peers' stores must arrive (bounded
                # wait in the kernel, LAMPS_ENCCL on timeout)
                rc = s.step_rc(kv_total=0)
                if rc != 0:
                    raise RuntimeError(f"trial exchange failed ({rc})")
        except Exception as e:  # noqa: BLE001
            print(f"p2p transport unavailable ({e}); using NCCL", file=sys.stderr)
            if s is not None:
                s.close()
            s, transport = None, "nccl"
        if world > 1:  # every rank must agree on the transport
            flag = torch.tensor([1 if transport == "p2p" else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if transport == "p2p" and int(flag.item()) == 0:
                s.close()
                s, transport = None, "nccl"
    if merged and transport == "nccl":
        if world > 1:
            obj = [Scheduler.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        else:
            nccl_id = Scheduler.nccl_unique_id()
    if s is None:
        s = Scheduler(cfg, flags=mflags, stream=stream, world=world, rank=rank, nccl_id=nccl_id,
                      transport=LAMPS_XPORT_NCCL)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-only timing (value): async steps, inputs resident, L2 flushed
    clk = ClockSampler(local).__enter__()  # samples clocks during warm-up and the timed steps
    for _ in range(args.warmup):
        flush.zero_()
        s.step_async(kv)
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.4:  # let the sampler start and the clocks settle
        for _ in range(20):
            flush.zero_()
            s.step_async(kv)
        torch.cuda.synchronize()
    r0 = s.result()
    # timed steps start from the snapshot again, so the measured state is snapshot + k steps
    # (the warm-up / burn steps would otherwise age the pool: starvation counters grow).  The
    # first step after a pool import builds the range grid from a bucket histogram (a cold
    # step, ~110 us, once per imported pool); it runs untimed, the timed steps are steady state
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    flush.zero_()
    s.step_async(kv)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        flush.zero_()
        starts[k].record(stream)
        s.step_async(kv)
        ends[k].record(stream)
    barrier()
    per_step_ms = sorted(a.elapsed_time(b) for a, b in zip(starts, ends))
    ms = sum(per_step_ms) / args.steps
    # the clock sampler (an nvidia-smi process) covered warm-up and the timed steps; it is
    # stopped here because its driver queries stall host-side CUDA calls, which the
    # host-timed e2e loop below would otherwise absorb
    clk.__exit__(None, None, None)
    res = s.result()
    n_elig = res["n_eligible"]
    # the P/D/S mix of the eligible requests after the timed steps (Table 2's API
    # classes), from the pool's state words
    ex = s.export_pool()
    rd = ex["state"] == 1
    mix = {"P": int(((ex["strategy"] == 0) & rd).sum()), "D": int(((ex["strategy"] == 1) & rd).sum()),
           "S": int(((ex["strategy"] == 2) & rd).sum()), "none": int(((ex["strategy"] == 3) & rd).sum())}
    kernels, passes = s.stats()
    fused = kernels == (2 if merged and transport == "nccl" else 1)
    ms_t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    ne_t = torch.tensor([float(n_elig)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ne_t, op=dist.ReduceOp.SUM)
    ms_max, ne_sum = float(ms_t.item()), float(ne_t.item())
    value = ne_sum / (ms_max / 1e3)

    # ---- per-kernel breakdown (separate handle with CUDA events between kernels, plus
    # the fused kernel's per-phase SM-clock trace)
    from paper_2410_18248_b200 import LAMPS_TRACE
    phase, trace_us, sp_passes = None, None, passes
    sp = Scheduler(cfg, flags=LAMPS_TIMING | LAMPS_TRACE, stream=stream) if not merged else None
    if sp is not None:
      sp.import_pool(snap, snap["id_base"], snap["next_id"])
      for _ in range(max(args.warmup, 100)):  # burn-in: the range weights settle
          flush.zero_()
          sp.step_async(kv)
      sp.timing()
      sp.import_pool(snap, snap["id_base"], snap["next_id"])  # same states as the timed steps above
      flush.zero_()
      sp.step_async(kv)  # the cold step after the import (untimed, as above)
      sp.timing()
      traces = []
      for _ in range(args.steps):
          flush.zero_()
          sp.step_async(kv)
          if fused and len(traces) < 10:
              traces.append(sp.trace().astype(np.int64))
      phase_ms, nst = sp.timing()
      sp_kernels, sp_passes = sp.stats()
      sp.close()
      phase = [x / nst for x in phase_ms]  # ms per step: [events, score or fused, sort, admit]
      trace_us = None
      if fused and traces:
          t = np.stack(traces)
          # warm-step phase boundaries of k_fused (kernels_fused.cu TRACE points)
          segs = [("score", 0, 1), ("range_assign", 1, 4), ("run_offsets", 4, 5), ("run_place", 5, 12),
                  ("run_store", 12, 6), ("barrier", 6, 7), ("l_prep", 7, 13), ("range_sort", 13, 14),
                  ("store_grid", 14, 8)]
          mhz = float(clk.summary().get("sm_mhz") or 1965.0)  # sampled during the timed steps
          trace_us = {nm: round(float(np.median((t[:, :, b1] - t[:, :, a1]).max(axis=1))) / mhz, 2)
                      for nm, a1, b1 in segs}
          trace_us["admission_cta0"] = round(float(np.median(t[:, 0, 9] - t[:, 0, 8])) / mhz, 2)

    # ---- end to end through the public API (host events in, host result out)
    e2e_steps = args.e2e_steps or max(args.steps, 200)
    # leave 8192 free slots in the id window so arrivals can be submitted
    snap_e = gen.snapshot(cname, seed=rank, id_base=id_base, n=cap - 8192)
    s.import_pool(snap_e, snap_e["id_base"], snap_e["next_id"])
    prev = s.step(kv_total=kv)["admitted_id"]
    paused, h2d, d2h = [], 0, 0
    barrier()
    t0 = time.perf_counter()
    ne_e2e = 0
    # the engine's buffers, reused every iteration (as a serving engine would)
    ev_buf = np.zeros(4, EVENT_DTYPE)
    ev_buf["kind"] = [2, 2, 1, 1]
    ids_buf = np.zeros(2, np.uint64)
    nxt = np.zeros(2, SEGMENT_DTYPE)
    nxt["pre_len"], nxt["has_api"] = 50, 0
    resp = np.full(2, 16, np.uint32)
    segs = np.zeros(2, SEGMENT_DTYPE)
    segs["prompt_len"], segs["pre_len"], segs["has_api"], segs["api_seconds"] = 300, 100, 1, 1.5
    segs["resp_len"], segs["post_len"] = 64, 50
    for k in range(e2e_steps):
        # one engine iteration through lamps_iterate: API returns of requests paused earlier,
        # 2 new arrivals, and the step with the engine's report on the previous batch (2
        # finish, 2 call their API) -- staging in the kernel's parameter block, one kernel,
        # one host synchronisation
        ne = min(4, len(prev))
        ev = ev_buf[:ne]
        ev["id"] = prev[:ne]
        nr = min(2, len(paused))
        ids = ids_buf[:nr]
        ids[:] = paused[:nr]
        paused = paused[nr:]
        rc, out, _ = s.iterate_rc(events=ev, ret_ids=ids, ret_resp=resp[:nr], ret_next=nxt[:nr], arrivals=segs,
                                  kv_total=kv)
        if rc != 0:
            raise RuntimeError(f"lamps_iterate failed ({rc})")
        h2d += ev.nbytes + ids.nbytes + resp[:nr].nbytes + nxt[:nr].nbytes + segs.nbytes
        paused += [int(x) for x in ev["id"][2:]]
        d2h += 64 + 9 * out["n_admitted"] + 8 * out["n_preempted"]
        ne_e2e += out["n_eligible"]
        prev = out["admitted_id"]
    torch.cuda.synchronize()
    dt_e2e = time.perf_counter() - t0
    e2e_t = torch.tensor([dt_e2e, float(ne_e2e)], device="cuda", dtype=torch.float64)
    if world > 1:
        mx = e2e_t[:1].clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = e2e_t[1:].clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dt_e2e, ne_e2e = float(mx.item()), float(sm.item())
    e2e_value = ne_e2e / dt_e2e

    # ---- variants: the same pool and timing under the selective score
    # update (interval 10, the paper's ToolBench setting) and the baseline keys
    variants = []
    if world == 1 and not args.no_variants:
        from paper_2410_18248_b200.lamps import LAMPS_POLICY_FCFS, LAMPS_POLICY_SJF, LAMPS_POLICY_SJF_TOTAL
        from paper_2410_18248_b200 import LAMPS_HEAD_ONLY, LAMPS_MERGE
        for name, over in (("p2p_exchange_merge_world1", dict(flags=LAMPS_MERGE, transport=LAMPS_XPORT_P2P)),
                           ("head_only", dict(flags=LAMPS_HEAD_ONLY)),
                           ("head_only_interval_10", dict(flags=LAMPS_HEAD_ONLY, score_interval=10)),
                           ("lamps_interval_10", dict(score_interval=10)),
                           ("sjf", dict(policy=LAMPS_POLICY_SJF)),
                           ("sjf_total", dict(policy=LAMPS_POLICY_SJF_TOTAL)),
                           ("fcfs", dict(policy=LAMPS_POLICY_FCFS))):
            vcfg = dict(cfg); vcfg.update({k: v for k, v in over.items() if k not in ("flags", "transport")})
            sv = Scheduler(vcfg, flags=over.get("flags", 0), stream=stream,
                           transport=over.get("transport", LAMPS_XPORT_NCCL))
            sv.import_pool(snap, snap["id_base"], snap["next_id"])
            for _ in range(max(args.warmup, 100)):  # the range weights settle (burn-in)
                flush.zero_()
                sv.step_async(kv)
            sv.import_pool(snap, snap["id_base"], snap["next_id"])
            flush.zero_()
            sv.step_async(kv)  # the cold step after the import (untimed)
            nsteps = max(args.steps, 10)
            ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(nsteps)]
            ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(nsteps)]
            torch.cuda.synchronize()
            for k in range(nsteps):
                flush.zero_()
                ev0[k].record(stream)
                sv.step_async(kv)
                ev1[k].record(stream)
            torch.cuda.synchronize()
            vms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1)) / nsteps
            vres = sv.result()
            variants.append({"name": name, **over, "us_per_step": vms * 1e3,
                             "decisions_per_s": vres["n_eligible"] / (vms / 1e3), "steps": nsteps})
            sv.close()

    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        # algorithmic bytes of one step: the SoA is read once (28 B/slot),
        # the state word written once (4 B/slot), and the keys written and read once (16 B/key)
        step_bytes = 32 * cap + 16 * n_elig
        if phase is None:  # multi-GPU: whole step (fused kernel + all-gather + merge), max over ranks
            dom = "k_fused+merge" if transport == "nccl" else "k_fused"
            kernels_tbl = {dom: {"ms": ms_max, "bytes": step_bytes, "GBps": step_bytes / (ms_max * 1e6)}}
        elif fused:
            dom = "k_fused"
            kernels_tbl = {"k_fused": {"ms": phase[1], "bytes": step_bytes, "GBps": step_bytes / (phase[1] * 1e6),
                                       "phase_us": trace_us},
                           "k0_events": {"ms": phase[0], "launched": False}}
        else:
            k1_bytes = 32 * cap + 8 * n_elig
            sort_bytes = 16 * n_elig * sp_passes
            kernels_tbl = {
                "k1_score": {"ms": phase[1], "bytes": k1_bytes, "GBps": k1_bytes / (phase[1] * 1e6)},
                "k2_sort": {"ms": phase[2], "passes": sp_passes, "bytes": sort_bytes,
                            "GBps": sort_bytes / (phase[2] * 1e6) if phase[2] else None},
                "k3_admit": {"ms": phase[3]}, "k0_events": {"ms": phase[0]},
            }
            dom = "k2_sort" if phase[2] >= phase[1] else "k1_score"
        ach = kernels_tbl[dom]["GBps"]
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(dom)
            except Exception:
                traffic = None
        xdesc = ("peer stores into every rank's buffer + merge inside the step kernel" if transport == "p2p"
                 else "NCCL all-gather + merge kernel")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "us_per_step": ms_max * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": config_dict(cname, cfg, kv, n_ready(snap), world, parallelism(world, merged, transport, cfg)),
            "transport": transport if merged else None, "ranks_connected": world,
            "strategy_mix": mix,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak if ach else None, "traffic": traffic,
                         "peak_source": peak_src},
            "kernels": kernels_tbl,
            # A4 alone (SURVEY 8(d) "keys/s per sort"): eligible keys over the fused kernel's sort
            # phases (keys to their ranges, the barrier, the range sorts; slowest CTA of each)
            "sort": ({"keys_per_s": n_elig / (1e-6 * sum(trace_us[k] for k in SORT_SEGS)),
                      "us": round(sum(trace_us[k] for k in SORT_SEGS), 2),
                      "phases": list(SORT_SEGS)} if trace_us else None),
            "pool_slots_per_s": world * cap / (ms_max / 1e3),
            # this rank's per-step distribution (median and p99 of the step time)
            "step_us": {"min": round(per_step_ms[0] * 1e3, 2),
                        "median": round(per_step_ms[len(per_step_ms) // 2] * 1e3, 2),
                        "p99": round(per_step_ms[min(len(per_step_ms) - 1, int(0.99 * len(per_step_ms)))] * 1e3, 2),
                        "max": round(per_step_ms[-1] * 1e3, 2)},
            "path": ("fused cooperative step kernel" + (f" ({xdesc})" if merged else "")) if fused else "3-kernel path",
            "sort_passes": passes,
            "gpu_launches": kernels * args.steps,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                    "d2h_bytes_per_step": d2h / e2e_steps,
                    "ms_per_step": 1e3 * dt_e2e / e2e_steps,
                    "path": "lamps_iterate per engine iteration: API returns + arrivals + events + step "
                            "(host buffers; results by mapped memory)"},
        }
        if variants:
            line["variants"] = variants
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cname)
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_strong(args, rank, world, local):
    """Strong scaling: the 1M-request pool as `shards` shards of 2^20 / shards
    slots, shard g on GPU g // (shards / N); the shards of one GPU are co-resident step kernels
    (#SM / S CTAs each, one stream each, launched together), every shard exchanges its top-K
    records with all others by peer stores (same GPU: device memory; other GPUs: CUDA IPC over
    NVLink) and admits its share of ONE global batch.  Time per step = device time from before
    the first to after the last of this GPU's kernels, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    from paper_2410_18248_b200 import Scheduler
    from paper_2410_18248_b200.lamps import EVENT_DTYPE, LAMPS_SHARE_DEVICE, LAMPS_XPORT_P2P
    W = args.shards
    if W % world:
        raise SystemExit(f"--shards {W} must be a multiple of the rank count {world}")
    S = W // world
    oversub = os.environ.get("LAMPS_BENCH_OVERSUBSCRIBE") == "1"
    if oversub:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cname = args.config
    cfg = gen.lib_config(cname)
    cap = cfg["capacity"] // W
    cfg["capacity"] = cap
    kv_all = gen.CONFIGS[cname]["kv_total"]
    kvs_all = [kv_all // W + (kv_all - W * (kv_all // W) if g == 0 else 0) for g in range(W)]
    mine = [rank * S + j for j in range(S)]
    kvs = [kvs_all[g] for g in mine]
    id_base = (1 << 17) * 7 + 99
    streams = [torch.cuda.Stream() for _ in mine]
    shards = [Scheduler(cfg, flags=LAMPS_SHARE_DEVICE, stream=streams[j], world=W, rank=g,
                        transport=LAMPS_XPORT_P2P, local_ranks=S) for j, g in enumerate(mine)]
    # each shard is 1/W of the 1M pool: its Preserve-paused KV is capped at 40% of ITS budget share
    snaps = [gen.snapshot(cname, seed=g, n=cap, capacity=cap, id_base=id_base, kv_total=kvs_all[g]) for g in mine]
    handles = [s.p2p_handle() for s in shards]
    if world > 1:
        allh = [None] * world
        dist.all_gather_object(allh, handles)
        flat = [h for hs in allh for h in hs]
    else:
        flat = handles
    for s in shards:
        s.p2p_connect(flat)
    main = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def load():
        for s, sn in zip(shards, snaps):
            s.import_pool(sn, sn["id_base"], sn["next_id"])
        barrier()

    def enqueue(start=None, end=None):
        # the GPU idles ~100 us (after the L2 flush) while the host enqueues the S launches, so
        # the shards start together and the host's launch latency is not device time (as the
        # flush hides it for the one launch of the single-shard step); e2e below includes it
        torch.cuda._sleep(200_000)
        e0 = torch.cuda.Event()
        e0.record(main)
        if start is not None:
            start.record(main)
        for st in streams:
            st.wait_event(e0)
        Scheduler.group_step_async(shards, kvs)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)
        if end is not None:
            end.record(main)

    load()
    Scheduler.group_step_async(shards, [0] * S)  # trial exchange: every shard's records arrive
    for s in shards:
        s.result()
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device="cuda")
    clk = ClockSampler(local).__enter__()
    load()
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        enqueue()
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.4:  # let the clock sampler start
        flush.zero_()
        enqueue()
        torch.cuda.synchronize()
    barrier()
    load()
    flush.zero_()
    enqueue()  # the cold step after the import (builds the shards' range grids), untimed
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        enqueue(starts[k], ends[k])
    barrier()
    clk.__exit__(None, None, None)
    per = sorted(a.elapsed_time(b) for a, b in zip(starts, ends))
    ms = sum(per) / args.steps
    res = [s.result() for s in shards]
    ne_local = sum(r["n_eligible"] for r in res)
    adm_local = sum(r["n_admitted"] for r in res)
    t = torch.tensor([ms, float(ne_local), float(adm_local)], device="cuda", dtype=torch.float64)
    if world > 1:
        mx = t[:1].clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm_ = t[1:].clone(); dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
        ms_max, ne_all, adm_all = float(mx.item()), float(sm_[0].item()), float(sm_[1].item())
    else:
        ms_max, ne_all, adm_all = ms, float(ne_local), float(adm_local)
    value = ne_all / (ms_max / 1e3)
    # end to end: the engine's iteration through the public API (lamps_group_step with each
    # shard's events about its previous batch: 2 finish), results to the host
    load()
    prev = [np.zeros(0, np.uint64) for _ in shards]
    h2d = d2h = 0
    e2e_steps = args.e2e_steps or max(args.steps, 100)
    barrier()
    t0 = time.perf_counter()
    ne_e2e = 0
    for k in range(e2e_steps):
        evs = []
        for p in prev:
            e = np.zeros(min(2, len(p)), EVENT_DTYPE)
            e["id"], e["kind"] = p[:len(e)], 2
            evs.append(e)
            h2d += e.nbytes
        outs = Scheduler.group_step(shards, evs, kvs)
        prev = [np.asarray(o["admitted_id"], np.uint64) for o in outs]
        for o in outs:
            d2h += 64 + 9 * o["n_admitted"] + 8 * o["n_preempted"]
            ne_e2e += o["n_eligible"]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt, float(ne_e2e)], device="cuda", dtype=torch.float64)
    if world > 1:
        mx = t[:1].clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm_ = t[1:].clone(); dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
        dt, ne_e2e = float(mx.item()), float(sm_.item())
    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        n_elig_gpu = ne_all / world
        gpu_bytes = 32 * cap * S + 16 * n_elig_gpu  # this GPU's shards
        ach = gpu_bytes / (ms_max * 1e6)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "us_per_step": ms_max * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{cname}: 1M-request pool as {W} shards x {cap} slots, {int(ne_all)} READY in all",
                       "shards": W, "shards_per_gpu": S, "slots_per_shard": cap, "kv_total_blocks": kv_all,
                       "max_batch": cfg["max_batch"], "l2": "flushed before every timed step (256 MiB write)",
                       "parallelism": f"{W} shards over {world} GPU(s), {S} co-resident step kernels per GPU "
                                      f"(#SM/{S} CTAs each); top-{cfg['max_batch']} records of every shard "
                                      f"stored into every shard's buffer, merge + global cut in each kernel"},
            "transport": "p2p", "ranks_connected": world, "admitted_per_step": adm_all,
            "roofline": {"bound": "hbm", "kernel": f"k_fused x {S} (co-resident)", "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak, "traffic": None, "peak_source": peak_src},
            "step_us": {"min": round(per[0] * 1e3, 2), "median": round(per[len(per) // 2] * 1e3, 2),
                        "max": round(per[-1] * 1e3, 2)},
            "gpu_launches": S * args.steps, "clocks": clk.summary(),
            "e2e": {"value": ne_e2e / dt, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                    "d2h_bytes_per_step": d2h / e2e_steps, "ms_per_step": 1e3 * dt / e2e_steps,
                    "path": "lamps_group_step per engine iteration (events in, results by mapped memory)"},
        }
        print(json.dumps(line), flush=True)
    for s in shards:
        s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; using {world} ranks", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.scaling == "strong":
        return run_strong(args, rank, world, local)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
