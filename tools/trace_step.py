"""Profiling only: CTA-0 event timeline of the span_attn_tc kernel for one C2 prefill launch.
Needs the profiling build (python -m paper_2511_02749_b200.build --profiling); uses it unless
SPANQ_LIB points elsewhere.
Usage: python tools/trace_step.py [dbg_mode] [prefill|join] [fp32|bf16] [C2|C4] > gpurun_out/trace.txt"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SPANQ_LIB", os.path.join(ROOT, "paper_2511_02749_b200", "lib", "libspanq_prof.so"))
import numpy as np
import torch

from paper_2511_02749_b200 import inputs, runner, spanq

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
out_dtype = sys.argv[3] if len(sys.argv) > 3 else "fp32"
dev = torch.device("cuda:0")
cfg = sys.argv[4] if len(sys.argv) > 4 else "C2"
w = inputs.c2() if cfg == "C2" else inputs.CONFIGS[cfg]()
ctx = spanq.Context(w.shape, 1024, device=0, max_position=1 << 15, out_dtype=out_dtype)
ctx.set_trace(None, mode)
tabs = [runner.device_tables(w.shape, 0, w.seed, dev)]
for _ in range(2):
    ctx.evict_all()
    runner.run_pass(ctx, w.queries, tabs, dev, release=True)
NW = 16
buf = torch.zeros(NW * 1024 * 2 + 2 * 1024, dtype=torch.int64, device=dev)
which = sys.argv[2] if len(sys.argv) > 2 else "prefill"
ctx.evict_all()
plan = ctx.plan(w.queries)
view = plan.view()
ptok = runner.prefill_tokens(view, w.queries)
q, k, v = runner.gather(tabs[0], ptok, dev)
o = torch.empty((len(ptok), w.shape.hq, w.shape.d), dtype=torch.float32 if out_dtype == "fp32" else torch.bfloat16, device=dev)
if which == "prefill":
    ctx.set_trace(buf, mode)
plan.prefill(0, q, k, v, o)
if which == "join":
    jtok = runner.join_tokens(view, w.queries)
    qj, kj, vj = runner.gather(tabs[0], jtok, dev)
    oj = torch.empty((len(jtok), w.shape.hq, w.shape.d), dtype=torch.float32 if out_dtype == "fp32" else torch.bfloat16, device=dev)
    ctx.set_trace(buf, mode)
    plan.join(0, qj, kj, vj, oj)
torch.cuda.synchronize()
ctx.set_trace(None, 0)
allb = buf.cpu().numpy()
t = allb[:NW * 2048].reshape(NW, 1024, 2)
spans = allb[NW * 2048:].reshape(-1, 2)
spans = spans[spans[:, 0] > 0]
g0 = spans[:, 0].min()
st, en = (spans[:, 0] - g0) / 1e3, (spans[:, 1] - g0) / 1e3
busy = en - st
print(f"# CTAs {len(spans)}: start max {st.max():.1f} us; end min/p50/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f} us;"
      f" busy min/p50/max {busy.min():.1f}/{np.median(busy):.1f}/{busy.max():.1f} us")
order = np.argsort(en)
print("# slowest CTAs:", [(int(i), round(float(en[i]), 1)) for i in order[-6:]])
print("# fastest CTAs:", [(int(i), round(float(en[i]), 1)) for i in order[:6]])
print("# end_us_by_cta:", " ".join(f"{float(e):.0f}" for e in en))
names = {10: "K issue", 11: "V issue", 12: "K want", 13: "V want", 20: "P_A rdy", 21: "Q rdy", 22: "K rdy", 23: "P_B rdy", 24: "V rdy", 25: "S issued", 27: "PV issued", 38: "item setup",
         30: "S rdy", 31: "P done", 32: "O rdy", 33: "epi done", 36: "stg free", 37: "stg stored", 40: "slotA free", 41: "slotB free", 42: "QA done",
         43: "QB done", 46: "rot fast", 47: "rot slow", 48: "rot table", 44: "QA loaded", 45: "QB loaded", 34: "max done", 35: "exp start", 50: "stg0", 51: "stg1", 52: "stg2", 53: "stg3",
         26: "O free", 60: "finA", 61: "O_A rdy", 62: "O_A drained", 64: "finB", 65: "O_B rdy", 66: "O_B drained"}
roles = ["tma", "mma", "w2", "w3", "smxA0", "smxA1", "smxA2", "smxA3", "smxB0", "smxB1", "smxB2", "smxB3",
         "qp0", "qp1", "qp2", "qp3"]
t0 = min(t[r][0][1] for r in range(NW) if t[r][0][1] > 0)
ev = []
for r in range(NW):
    for e, c in t[r]:
        if c > 0:
            # events 10-13 / 22 / 24 / 30 / 31 carry the sub-tile index in bits 8+
            ev.append((c - t0, roles[r], names.get(int(e) & 255, str(e)) + (f" #{int(e) >> 8}" if e >= 256 else "")))
ev.sort()
for c, r, n in ev[:3000]:
    print(f"{c:9d} {r:6s} {n}")
