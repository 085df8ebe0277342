"""Test-side rankers for the simulators (sim/): the CPU oracle as the ranker, so the
same engine run can be produced by the oracle and by the CUDA pass and compared."""
import numpy as np

import oracle as O


class OracleRanker:
    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        self.cap = int(cfg["capacity"])

    def rank(self, fields: dict, id_base: int, next_id: int):
        o = O.OraclePool(self.cfg)
        f = {k: np.asarray(v) for k, v in fields.items()}
        o.load(f, next_id)
        r = o.step(kv_total=0, debug=True)
        assert r["rc"] == O.OK
        live = f["state"] != 0
        labels = {int(i): int(r["strategy"][int(i) % self.cap]) if f["state"][int(i) % self.cap] == O.READY
                  else int(f["strategy"][int(i) % self.cap]) for i in f["id"][live]}
        return [int(i) for i in r["ranked_id"]], labels


def table1_cfg(golden, fx="a", policy=0):
    """Scheduler config of the worked example: B = 1 token, fixture costs (R17)."""
    t1 = golden["table1"]
    f, cm = t1["fixtures"][fx], t1["common"]
    return dict(capacity=16, block_tokens=cm["block_tokens"], tau=f["tau"], A1=cm["A1"], A2=f["A2"],
                S0=cm["S0"], S1=f["S1"], SH=cm["SH"], c_other=cm["c_other"], ticks_per_second=1.0,
                starvation_threshold=10_000, max_batch=16, kv_capacity_blocks=1 << 20, score_bits=40,
                id_bits=23, policy=policy, score_interval=0)


def table1_specs(golden):
    return [(r["api_after"], r["api_iters"], r["post"]) for r in golden["table1"]["requests"].values()]


class OracleBackend:
    """The CPU oracle behind the scale engine's scheduler interface (sim/engine.py)."""

    def __init__(self, cfg: dict):
        self.o = O.OraclePool(cfg)
        self.tps = float(cfg["ticks_per_second"])

    def predict(self, truth, seed, len_ppm, api_ppm):
        t = np.ascontiguousarray(truth, O.TRUTH_DTYPE)
        rc, p = O.predict(t, seed=seed, len_error_ppm=len_ppm, api_error_ppm=api_ppm)
        assert rc == O.OK
        segs = np.zeros(len(t), O.SEG_DTYPE)
        segs["prompt_len"] = t["prompt_len"]
        segs["pre_len"] = p["pre_len"]
        segs["resp_len"] = p["resp_len"]
        segs["post_len"] = p["post_len"]
        segs["api_seconds"] = p["api_ticks"].astype(np.float64) / self.tps
        segs["has_api"] = t["has_api"]
        return segs

    def submit(self, segs):
        rc, ids = self.o.submit(segs)
        assert rc == O.OK
        return ids

    def api_return(self, ids, resp, segs):
        assert self.o.api_return(ids, resp, segs) == O.OK

    def step(self, ev, kv_total):
        r = self.o.step(ev, kv_total)
        assert r["rc"] == O.OK
        return {"admitted_id": r["admitted_id"], "n_admitted": r["n_admitted"], "n_preempted": r["n_preempted"]}

    def close(self):
        pass
