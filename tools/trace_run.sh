mkdir -p gpurun_out
for m in prefill join; do timeout 120 python tools/trace_step.py 0 $m bf16 > gpurun_out/t_$m.txt 2>&1; python tools/trace_items.py gpurun_out/t_$m.txt > gpurun_out/t_${m}_items.txt 2>&1; done
timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 20 > gpurun_out/b1.json 2> gpurun_out/b1.err
tail -c 600 gpurun_out/b1.err
