"""Kernel-level A/B (profiling aid, run under gpurun): prefill / join attention kernel times of C2
(d = 128) and C4 (d = 64), cold cache, bf16 O, for several library builds and runtime options,
interleaved so box drift hits every variant alike.

  python tools/kab.py [reps] VARIANT [VARIANT ...]
  VARIANT = <lib file in paper_2511_02749_b200/lib or "-">[:key=value,...]   (keys: spq_set_option ids)
  e.g.  python tools/kab.py 5 - -:1=1 libspanq_b.so

Each variant runs in its own process (a library is loaded once per process); the median of `reps`
cold passes is printed per kernel.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2511_02749_b200 import inputs, runner, spanq
opts, reps = json.loads(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
out = {}
for name, w in (("C2", inputs.c2()), ("C4", inputs.CONFIGS["C4"]())):
    ctx = spanq.Context(w.shape, 2048, device=0, max_position=1 << 15, out_dtype="bf16")
    for k, v in opts.items():
        ctx.set_option(int(k), float(v))
    ctx.set_timing(True)
    tabs = [runner.device_tables(w.shape, 0, w.seed, dev)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    pre, jn = [], []
    for i in range(reps + 2):
        ctx.evict_all()
        flush.zero_()
        runner.run_pass(ctx, w.queries, tabs, dev, release=True)
        torch.cuda.synchronize()
        p, j = ctx.last_attn_ms()
        if i >= 2:
            pre.append(p); jn.append(j)
    out[name] = (float(np.median(pre)), float(np.median(jn)))
    ctx.close()
print("RESULT", json.dumps(out))
'''.replace("ROOT", repr(ROOT))


def run(variant, reps):
    lib, _, optstr = variant.partition(":")
    env = dict(os.environ)
    if lib and lib != "-":
        env["SPANQ_LIB"] = os.path.join(ROOT, "paper_2511_02749_b200", "lib", lib)
    opts = dict(kv.split("=") for kv in optstr.split(",") if kv)
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(opts), str(reps)], env=env, capture_output=True,
                       text=True, timeout=600)
    for line in r.stdout.splitlines():
        if line.startswith("RESULT"):
            return json.loads(line[6:])
    sys.stderr.write(r.stderr[-3000:])
    return None


def main():
    reps = int(sys.argv[1])
    variants = sys.argv[2:]
    rounds = 2
    res = {v: [] for v in variants}
    for _ in range(rounds):
        for v in variants:
            res[v].append(run(v, reps))
    for v in variants:
        rs = [r for r in res[v] if r]
        if not rs:
            print(f"{v:40s} FAILED")
            continue
        c2p = min(r["C2"][0] for r in rs)
        c2j = min(r["C2"][1] for r in rs)
        c4p = min(r["C4"][0] for r in rs)
        c4j = min(r["C4"][1] for r in rs)
        print(f"{v:40s} C2 pre {c2p:.4f} join {c2j:.4f} | C4 pre {c4p:.4f} join {c4j:.4f}  "
              f"(C2 pre frac {139.72484915e9 / (c2p / 1e3) / 1e12 / 1630.0:.3f}, join {71.41e9 / (c2j / 1e3) / 1e12 / 1630.0:.3f})")


if __name__ == "__main__":
    main()
