#!/bin/bash
# GPU iteration (run under gpurun): GPU tests, kernel A/B of library builds, CTA-0 traces.
#   bash tools/ab_run.sh TAG "pytest -k expr or empty" "kab variants"
tag=$1; mkdir -p gpurun_out
if [ -n "$2" ]; then k=(-k "$2"); else k=(); fi
timeout 900 python -m pytest tests -m gpu -x -q "${k[@]}" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 600 python tools/kab.py 5 $3 > gpurun_out/${tag}_kab.txt 2>&1; cat gpurun_out/${tag}_kab.txt
for m in prefill join; do timeout 120 python tools/trace_step.py 0 $m bf16 > gpurun_out/${tag}_t_$m.txt 2>&1; python tools/trace_items.py gpurun_out/${tag}_t_$m.txt | tail -1; done
