"""Per-call GPU time and host-induced gaps over a 40-layer C2 step (one plan): events around each
ABI call on the launching stream. Usage: python tools/layer_gaps.py > gpurun_out/gaps.txt"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

L = 40
w = inputs.c2(seed=2)
s = inputs.Shape(**{**w.shape.__dict__, "layers": L})
dev = torch.device("cuda:0")
ctx = spanq.Context(s, 512, device=0, max_position=1 << 15, out_dtype="fp32")
tab = runner.device_tables(s, 0, w.seed, dev)
st = torch.cuda.Stream(dev)
p0 = ctx.plan(w.queries, stream=st)
v = p0.view()
ptok, jtok = runner.prefill_tokens(v, w.queries), runner.join_tokens(v, w.queries)
qp, kp, vp = runner.gather(tab, ptok, dev)
qj, kj, vj = runner.gather(tab, jtok, dev)
op = torch.empty((len(ptok), s.hq, s.d), dtype=torch.float32, device=dev)
oj = torch.empty((len(jtok), s.hq, s.d), dtype=torch.float32, device=dev)
p0.release(stream=st)
torch.cuda.synchronize()
with torch.cuda.stream(st):
    for rep in range(3):
        ctx.evict_all()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4 * L + 2)]
        t0 = time.perf_counter()
        evs[0].record(st)
        plan = ctx.plan(w.queries, stream=st)
        evs[1].record(st)
        host = []
        for l in range(L):
            h0 = time.perf_counter()
            evs[2 + 4 * l].record(st)
            plan.prefill(l, qp, kp, vp, op, stream=st)
            evs[3 + 4 * l].record(st)
            evs[4 + 4 * l].record(st)
            plan.join(l, qj, kj, vj, oj, stream=st)
            evs[5 + 4 * l].record(st)
            host.append(time.perf_counter() - h0)
        plan.release(stream=st)
        st.synchronize()
        tot = evs[0].elapsed_time(evs[-1 - 1 + 1 - 1]) if False else evs[0].elapsed_time(evs[5 + 4 * (L - 1)])
        pre = [evs[2 + 4 * l].elapsed_time(evs[3 + 4 * l]) for l in range(L)]
        jn = [evs[4 + 4 * l].elapsed_time(evs[5 + 4 * l]) for l in range(L)]
        gap_pj = [evs[3 + 4 * l].elapsed_time(evs[4 + 4 * l]) for l in range(L)]
        gap_jp = [evs[5 + 4 * l].elapsed_time(evs[2 + 4 * (l + 1)]) for l in range(L - 1)]
        print(f"rep {rep}: total {tot:.3f} ms; plan(gpu) {evs[0].elapsed_time(evs[1]):.3f}; "
              f"prefill call med {np.median(pre):.4f} join call med {np.median(jn):.4f}; "
              f"gaps p->j sum {sum(gap_pj):.3f} j->p sum {sum(gap_jp):.3f} ms; host per layer med "
              f"{1e3 * np.median(host):.3f} ms; first layer prefill {pre[0]:.4f} join {jn[0]:.4f}")
