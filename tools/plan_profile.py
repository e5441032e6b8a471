"""Host planning cost of the C2 query (spq_plan_create through the binding) on a GPU ctx: median
of 30 plans, each after evict_all and a 5 ms pause (pool workers asleep, as between bench steps).
With SPANQ_PROFILE=1 and the profiling build (SPANQ_LIB=.../libspanq_prof.so) the library also
prints its per-stage laps. Usage: python tools/plan_profile.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_02749_b200 import inputs, spanq

w = inputs.c2(seed=2)
dev = 0 if torch.cuda.is_available() else -1
ctx = spanq.Context(w.shape, 512, device=dev, max_position=1 << 15)
ts = []
for i in range(30):
    ctx.evict_all()
    if dev >= 0:
        torch.cuda.synchronize()
    time.sleep(0.005)
    t0 = time.perf_counter()
    p = ctx.plan(w.queries)
    t1 = time.perf_counter()
    p.release()
    ts.append((t1 - t0) * 1e3)
ts.sort()
print(f"plan_create C2 ({'GPU' if dev >= 0 else 'host-only'} ctx): p10 {ts[3]:.3f} median {ts[15]:.3f} p90 {ts[27]:.3f} ms; "
      f"{os.cpu_count()} host threads")
