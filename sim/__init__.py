"""Discrete-event simulators that drive the LAMPS pass in a closed loop.

They play the ENGINE: time, KV residency of running / preempted / paused requests,
Preserve / Discard / Swap physics, recomputation and swap timing, API durations,
arrivals and completions.  They hold none of the method's arithmetic: the ranked
order (A1-A4: strategy argmin, memory-over-time score, starvation, sort) and the
handling label chosen at API entry come from a *ranker*:

  * ``PassRanker`` -- the CUDA pass through the C ABI (paper_2410_18248_b200);
  * any object with the same ``rank`` method (tests plug the CPU oracle in, so the
    same schedule can be produced by both and compared);
  * ``StaticRanker`` -- a fixed priority order (the paper's hand-made "Preferred*"
    schedule).

``unit``   -- the worked example's unit model (Table 1).
``engine`` -- the iteration-level engine at workload scale, admission by the pass
              itself (A5), with prediction error injection (row F4) for the paper's
              starvation and misprediction studies.
"""
from .rankers import PassRanker, StaticRanker  # noqa: F401
from .unit import UnitRequest, simulate_unit, average_jct  # noqa: F401
