#!/bin/bash
# Profiling pass for profiles/ (run under gpurun): launch list of bench-like steps, one full ncu
# capture per hot kernel, the bench JSON, and nvidia-smi clocks.
#   bash tools/profile_round.sh            (then: python tools/ncu_summary.py r02)
set -x
python -m paper_2511_02749_b200.build > /dev/null
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/prof/gpu.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-locality --no-c5 > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:span_attn_tc -s 2 -c 2 \
  -o gpurun_out/prof/attn python tools/profile_step.py 2 > gpurun_out/prof/ncu_attn.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:rope_kv_write -s 2 -c 1 \
  -o gpurun_out/prof/kvwrite python tools/profile_step.py 2 > gpurun_out/prof/ncu_kv.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:combine -s 1 -c 1 \
  -o gpurun_out/prof/combine python tools/profile_step.py 2 > gpurun_out/prof/ncu_comb.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cidra -s 1 -c 1 \
  -o gpurun_out/prof/cidra python tools/profile_cidra.py 2 > gpurun_out/prof/ncu_cidra.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 8 -c 1 \
  -o gpurun_out/prof/decode python tools/profile_step.py 1 C2 bf16 16 > gpurun_out/prof/ncu_decode.log 2>&1
# (compute-sanitizer is closed on the GPU pool from round 2 on: the r02 logs in profiles/ are the
# last sanitizer evidence)
timeout 900 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err
