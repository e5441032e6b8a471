"""Profiling only: CTA-0 event timeline of the span_attn_tc kernel for one C2 prefill launch.
Usage: python tools/trace_step.py [dbg_mode] > gpurun_out/trace.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

mode = sys.argv[1] if len(sys.argv) > 1 else "0"
os.environ["SPANQ_DBG_MODE"] = mode
dev = torch.device("cuda:0")
w = inputs.c2()
ctx = spanq.Context(w.shape, 1024, device=0, max_position=1 << 15, out_dtype="fp32")
tabs = [runner.device_tables(w.shape, 0, w.seed, dev)]
for _ in range(2):
    ctx.evict_all()
    runner.run_pass(ctx, w.queries, tabs, dev, release=True)
buf = torch.zeros(5 * 1024 * 2, dtype=torch.int64, device=dev)
os.environ["SPANQ_TRACE"] = str(buf.data_ptr())
ctx.evict_all()
plan = ctx.plan(w.queries)
view = plan.view()
ptok = runner.prefill_tokens(view, w.queries)
q, k, v = runner.gather(tabs[0], ptok, dev)
o = torch.empty((len(ptok), 32, 128), dtype=torch.float32, device=dev)
plan.prefill(0, q, k, v, o)
torch.cuda.synchronize()
del os.environ["SPANQ_TRACE"]
t = buf.view(5, 1024, 2).cpu().numpy()
names = {10: "K issue", 11: "V issue", 20: "P_A rdy", 21: "Q rdy", 22: "S_A issue", 23: "P_B rdy", 24: "drain P_A",
         30: "S rdy", 31: "P done", 32: "O rdy", 33: "epi done", 40: "slotA free", 41: "slotB free", 42: "QA done",
         43: "QB done", 34: "max done", 35: "exp start"}
roles = ["tma", "mma", "smxA", "smxB", "qprep"]
t0 = min(t[r][0][1] for r in range(5) if t[r][0][1] > 0)
ev = []
for r in range(5):
    for e, c in t[r]:
        if c > 0:
            ev.append((c - t0, roles[r], names.get(int(e), str(e))))
ev.sort()
for c, r, n in ev[:700]:
    print(f"{c:9d} {r:6s} {n}")
