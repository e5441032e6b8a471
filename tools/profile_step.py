"""Run a few C2 steps (plan -> prefill -> join) for ncu / compute-sanitizer captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
dev = torch.device("cuda:0")
w = inputs.CONFIGS[cfg]()
ctx = spanq.Context(w.shape, 4096, device=0, max_position=1 << 15, out_dtype="fp32")
tabs = [runner.device_tables(w.shape, 0, w.seed, dev)]
for q in w.warmup_queries:
    runner.run_pass(ctx, [q], tabs, dev, release=True)
for i in range(steps):
    if cfg != "C3":
        ctx.evict_all()
    runner.run_pass(ctx, w.queries, tabs, dev, release=True)
torch.cuda.synchronize()
print("ok", ctx.launch_count())
