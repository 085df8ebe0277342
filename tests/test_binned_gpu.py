"""GPU <-> oracle parity (bit-exact) on pools that stress the binned R and the shared-memory range
sort of the fused kernel (items 2-3):

* slots laid out by context length, so each CTA's keys fall into a few ranges: most keys go to the
  per-range overflow list instead of the 48-key bins;
* every READY request one step short of the starvation threshold, so the whole order flips to the
  starving group at once: every range hint misses (more misses than the miss queue holds: the
  search runs inline), every key lands in range 0, the range overflows and the step takes the
  grid-wide fallback, compacting the keys from the bins and the overflow list.
Measured on a B200 (`scripts/r02/binned_stress_stats.py`, `profiles/r02/binned_stress_stats.txt`):
the sorted C4 layout puts up to ~125 keys per CTA on the overflow list and ~200 hint misses per
CTA; the C5 flip step has 6266 misses in one CTA (past the 5344-entry miss queue), 6261 overflow
keys and takes the 7-pass global LSD.
"""
import numpy as np
import pytest

import gen
from parity_util import compare_outputs, compare_state, load_both, make_pair

CONTENT = ("state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem", "api_ticks", "resp_len",
           "post_len", "pending")


def run(cname, snap, steps, cfg=None, kv=None):
    cfg = cfg or gen.lib_config(cname)
    s, o = make_pair(cfg, path="fused")
    load_both(s, o, snap)
    kv = kv if kv is not None else gen.CONFIGS[cname]["kv_total"]
    for t in range(steps):
        g = s.step(kv_total=kv)
        r = o.step(kv_total=kv, debug=True)
        compare_outputs(s, g, r, where=f"{cname} step {t}")
        compare_state(s, o, r, where=f"{cname} step {t}")
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 3])
def test_sorted_layout_overflows_bins(seed):
    """C4 pool with the requests ordered by context length across the slots."""
    snap = gen.snapshot("C4", seed=seed, id_base=0)
    live = np.flatnonzero(snap["state"] != 0)  # the live slots keep their ids; their requests move
    order = live[np.argsort((snap["ctx"] + snap["pre_rem"])[live], kind="stable")]
    for f in CONTENT:
        v = snap[f].copy()
        v[live] = snap[f][order]
        snap[f] = v
    run("C4", snap, steps=5)


@pytest.mark.gpu
@pytest.mark.slow
def test_mass_starvation_flip_c5():
    """C5 pool (2^20 slots) whose READY requests all turn starving on the same step."""
    cfg = gen.lib_config("C5")
    T = int(cfg.get("starvation_threshold", gen.CONFIGS["C5"].get("starvation_threshold", 100)))
    snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99)
    ready = snap["state"] == 1
    snap["cnt"] = np.where(ready, max(T - 2, 0), snap["cnt"])
    snap["starving"] = np.where(ready, 0, snap["starving"])
    run("C5", snap, steps=4, cfg=cfg)
