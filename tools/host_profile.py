"""Host-side cost of one C2 step through the Python binding (planning + launches), GPU ctx."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

w = inputs.c2(seed=2)
s = w.shape
dev = torch.device("cuda:0")
ctx = spanq.Context(s, 512, device=0, max_position=1 << 15, out_dtype="fp32")
tab = runner.device_tables(s, 0, w.seed, dev)
p0 = ctx.plan(w.queries)
view = p0.view()
ptok, jtok = runner.prefill_tokens(view, w.queries), runner.join_tokens(view, w.queries)
qp, kp, vp = runner.gather(tab, ptok, dev)
qj, kj, vj = runner.gather(tab, jtok, dev)
op = torch.empty((len(ptok), s.hq, s.d), dtype=torch.float32, device=dev)
oj = torch.empty((len(jtok), s.hq, s.d), dtype=torch.float32, device=dev)
p0.release()
torch.cuda.synchronize()
for i in range(8):
    ctx.evict_all()
    t0 = time.perf_counter()
    plan = ctx.plan(w.queries)
    t1 = time.perf_counter()
    plan.prefill(0, qp, kp, vp, op)
    t2 = time.perf_counter()
    plan.join(0, qj, kj, vj, oj)
    t3 = time.perf_counter()
    plan.release()
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"plan {1e6*(t1-t0):7.1f} us  prefill call {1e6*(t2-t1):6.1f}  join call {1e6*(t3-t2):6.1f}  release {1e6*(t4-t3):6.1f}",
          flush=True)
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
