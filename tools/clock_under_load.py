"""SM clock under the bench's own load: C2 steps of 40 back-to-back (prefill, join) layers (the
same layer's inputs, bf16 O) for ~8 s while nvidia-smi samples clocks.sm / power every ~100 ms;
prints the clock distribution and the last layer's prefill / join kernel times (ABI timing events)
of each step — evidence for which MEASURED_PEAKS figure (burst or sustained) a kernel timed inside
a long step should be held against. Usage: python tools/clock_under_load.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2511_02749_b200 import inputs, runner, spanq

w = inputs.c2(seed=2)
dev = torch.device("cuda:0")
ctx = spanq.Context(w.shape, 512, device=0, max_position=1 << 15, out_dtype="bf16")
tab = runner.device_tables(w.shape, 0, w.seed, dev)
p0 = ctx.plan(w.queries)
v = p0.view()
pt, jt = runner.prefill_tokens(v, w.queries), runner.join_tokens(v, w.queries)
qp, kp, vp = runner.gather(tab, pt, dev)
qj, kj, vj = runner.gather(tab, jt, dev)
op = torch.empty((len(pt), 32, 128), dtype=torch.bfloat16, device=dev)
oj = torch.empty((len(jt), 32, 128), dtype=torch.bfloat16, device=dev)
p0.release()
ctx.set_timing(True)
pre, join = [], []
with bench.ClockSampler(0) as clk:
    t_end = time.time() + 8.0
    while time.time() < t_end:
        ctx.evict_all()
        plan = ctx.plan(w.queries)
        for _ in range(40):
            plan.prefill(0, qp, kp, vp, op)
            plan.join(0, qj, kj, vj, oj)
        torch.cuda.synchronize()
        a, b = ctx.last_attn_ms()
        pre.append(a)
        join.append(b)
        plan.release()
s = clk.summary()
sm = sorted(float(r[0]) for r in clk.rows if r[0].replace(".", "").isdigit())
pw = sorted(float(r[2]) for r in clk.rows if r[2].replace(".", "").isdigit())
print(f"samples {len(sm)}: SM MHz min {sm[0]:.0f} p10 {sm[len(sm) // 10]:.0f} median {statistics.median(sm):.0f} "
      f"max {sm[-1]:.0f}; power median {statistics.median(pw):.0f} W max {pw[-1]:.0f} W; reasons {s['reasons']}")
print(f"passes {len(pre)}: prefill kernel median {statistics.median(pre):.4f} ms (first 5 {statistics.median(pre[:5]):.4f}, "
      f"last 5 {statistics.median(pre[-5:]):.4f}); join median {statistics.median(join):.4f} ms")
print("MEASURED_PEAKS:", bench.peaks())
