"""Run single bench.py sections (for iteration): python tools/bench_extras.py decode judge bulk c5"""
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
args = types.SimpleNamespace(out_dtype="bf16", warmup=3, steps=5, layers=1)
fns = {"decode": bench.measure_decode, "judge": bench.measure_judge_tree, "bulk": bench.measure_bulk,
       "c5": bench.measure_c5}
with torch.cuda.stream(stream):
    for name in sys.argv[1:]:
        print(name, json.dumps(fns[name](dev, stream, args)), flush=True)
