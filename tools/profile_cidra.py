"""CIDRA (K8) capture for ncu: the bench's reposition workload (a random permutation of C2's 268
blocks, random shifts in [-8192, 8192]) on a 40-layer 8B-shape pool. Usage: python tools/profile_cidra.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, spanq

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = inputs.Shape(**{**inputs.SHAPE_8B, "block_size": 64, "layers": 40})
ctx = spanq.Context(s, 512, device=0, max_position=1 << 15)
g = np.random.default_rng(7)
n = 268
dst = g.permutation(n).astype(np.int32)
src = np.arange(n, dtype=np.int32)
delta = g.integers(-8192, 8193, size=n).astype(np.int32)
for _ in range(reps):
    st = ctx.reposition(src, dst, delta)
torch.cuda.synchronize()
print("ok", st)
