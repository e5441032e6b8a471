#!/bin/bash
# Quick GPU iteration (run under gpurun): build, parity tests, 1-layer + 40-layer bench, traces.
# Usage: bash tools/gpu_quick.sh [tag] [pytest -k expr]
tag=${1:-q}
mkdir -p gpurun_out
python -m paper_2511_02749_b200.build > /dev/null || exit 1
if [ -n "$2" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/${tag}_tests.log 2>&1
else
  timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1
fi
tail -3 gpurun_out/${tag}_tests.log
timeout 300 python bench.py --layers 1 --no-cpu-baseline > gpurun_out/${tag}_bench1.json 2> gpurun_out/${tag}_bench1.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench40.json 2> gpurun_out/${tag}_bench40.err
timeout 120 python tools/trace_step.py 0 prefill > gpurun_out/${tag}_trace_pre.txt 2>&1
timeout 120 python tools/trace_step.py 0 join > gpurun_out/${tag}_trace_join.txt 2>&1
python - <<PY
import json
for f in ["gpurun_out/${tag}_bench1.json", "gpurun_out/${tag}_bench40.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, "value %.1f ms %.3f pre %.3f ms frac %.3f join %.3f ms frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], d["join_kernel"]["ms"], d["join_kernel"]["frac"]))
    except Exception as e:
        print(f, "failed", e)
PY
head -3 gpurun_out/${tag}_trace_pre.txt gpurun_out/${tag}_trace_join.txt
