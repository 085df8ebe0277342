"""Host-side costs around one synchronous step on the C5 pool (no L2 flush): the ctypes
call of a trivial entry point, the launch call (lamps_schedule_step_async), the time from
the launch call's return to the end of the synchronisation, and the same with the kernel
alone timed by CUDA events."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2410_18248_b200 import Scheduler
from paper_2410_18248_b200.lamps import lib

cfg = gen.lib_config("C5")
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99, n=cfg["capacity"] - 8192)
kv = gen.CONFIGS["C5"]["kv_total"]
STREAM = os.environ.get("STREAM", "default")
s = Scheduler(cfg, stream=torch.cuda.Stream() if STREAM == "own" else None)
s.import_pool(snap, snap["id_base"], snap["next_id"])
for _ in range(300):
    s.step(kv_total=kv)
N = 300
L = lib()
t0 = time.perf_counter()
for _ in range(N):
    L.lamps_version() if hasattr(L, "lamps_version") else L.lamps_last_error(s.h)
t_ctypes = (time.perf_counter() - t0) / N * 1e6
la, sy, ev = [], [], []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(N):
    torch.cuda.synchronize()
    a = time.perf_counter()
    s.step_async(kv)
    b = time.perf_counter()
    torch.cuda.synchronize()
    c = time.perf_counter()
    la.append(b - a); sy.append(c - b)
st = []
for _ in range(N):
    a = time.perf_counter()
    s.step(kv_total=kv)
    st.append(time.perf_counter() - a)
for _ in range(N // 3):
    e0.record(); s.step_async(kv); e1.record(); torch.cuda.synchronize()
    ev.append(e0.elapsed_time(e1) * 1e3)
m = lambda x: float(np.median(x)) * 1e6
print(f"stream={STREAM}: ctypes trivial call {t_ctypes:.1f} us; launch call {m(la):.1f} us; launch return -> synced {m(sy):.1f} us; "
      f"step() sync total {m(st):.1f} us; kernel by events (idle GPU) {float(np.median(ev)):.1f} us")
