"""Run a few steps (plan -> prefill -> join [-> decode]) for ncu / compute-sanitizer captures.
Usage: python tools/profile_step.py [steps] [config: C1 C2 C2s C3 C4] [out dtype] [decode steps]
(C2s = C2 shrunk to 1/8: the sanitizer-sized bf16 case)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
out = (sys.argv[3] or None) if len(sys.argv) > 3 else None
n_dec = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device("cuda:0")
w = inputs.c2(scale=0.125) if cfg == "C2s" else inputs.CONFIGS[cfg]()
out = out or ("fp32" if w.shape.dtype == "fp32" else "bf16")
ctx = spanq.Context(w.shape, 4096, device=0, max_position=1 << 15, out_dtype=out)
if os.environ.get("PROFILE_PDL") == "0":  # sanitizer A/B: attention/combine not launched as PDL dependents
    ctx.set_option(spanq.OPT_PDL, 0)
tabs = [runner.device_tables(w.shape, 0, w.seed, dev)]
for q in w.warmup_queries:
    runner.run_pass(ctx, [q], tabs, dev, release=True)
for i in range(steps):
    if cfg != "C3":
        ctx.evict_all()
    res = runner.run_pass(ctx, w.queries, tabs, dev, release=n_dec == 0)
    if n_dec:
        res.plan.decode_reserve(n_dec)
        g = np.random.default_rng(i)
        B = len(w.queries)
        for t in range(n_dec):
            q, k, v = runner.gather(tabs[0], g.integers(0, w.shape.vocab, B), dev)
            o = torch.empty((B, w.shape.hq, w.shape.d), dtype=torch.bfloat16 if out == "bf16" else torch.float32,
                            device=dev)
            res.plan.decode_step(0, t, q, k, v, o)
        res.plan.release()
torch.cuda.synchronize()
print("ok", ctx.launch_count())
