"""CIDRA (K8) at one layer and at 40 layers, C2's block count: event time per call (host schedule
+ H2D + kernel, as bench.py `reposition`) and the host time of the call alone, so the kernel's
share of the one-layer case is visible. Usage: python tools/cidra_l1.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, spanq

w = inputs.c2()
s = inputs.Shape(**{**w.shape.__dict__, "layers": 40})
ctx = spanq.Context(s, 512, device=0, max_position=1 << 15)
stream = torch.cuda.Stream()
n = 268
g = np.random.default_rng(7)
dst = g.permutation(n).astype(np.int32)
src = np.arange(n, dtype=np.int32)
delta = g.integers(-8192, 8193, size=n).astype(np.int32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for layers in ((0, 1), (0, 40)):
    ctx.reposition(src, dst, delta, layers=layers, stream=stream)
    ev, host = [], []
    for _ in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        ctx.reposition(src, dst, delta, layers=layers, stream=stream)
        host.append((time.perf_counter() - t0) * 1e3)
        b.record(stream)
        stream.synchronize()
        ev.append(a.elapsed_time(b))
    nbytes = 2 * 2 * n * (layers[1] - layers[0]) * s.hkv * s.block_size * s.d * 2
    med = float(np.median(ev))
    print(f"layers {layers}: event {med:.4f} ms ({nbytes / med / 1e6:.0f} GB/s), host call {np.median(host):.4f} ms")
