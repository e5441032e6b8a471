python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for m in 0 1 3 5; do python tools/trace_step.py $m prefill > gpurun_out/m${m}_pre.txt 2>&1; head -1 gpurun_out/m${m}_pre.txt; done
