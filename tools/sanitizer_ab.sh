#!/bin/bash
# compute-sanitizer A/B (run under gpurun): the probe kernels (tools/sanitizer_probe.cu) under
# racecheck / synccheck, and the C2s step (bf16 and fp32 O).
python -m paper_2511_02749_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/sanitizer_probe tools/sanitizer_probe.cu
O=gpurun_out/san; mkdir -p $O; rm -f $O/summary.txt
for tool in racecheck synccheck; do
  for m in ${PROBE_MODES:-0 1 2 3 4 5 6 7}; do
    timeout 120 compute-sanitizer --tool $tool --print-limit 5 tools/sanitizer_probe $m > $O/probe_${tool}_$m.log 2>&1
    echo "probe $tool mode $m rc=$?: $(grep -E 'SUMMARY|^ok' $O/probe_${tool}_$m.log | tr '\n' ' ')" >> $O/summary.txt
  done
done
for out in ${C2S_OUTS-bf16 fp32}; do
  for tool in synccheck racecheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 10 python tools/profile_step.py 1 C2s $out 4 \
      > $O/${tool}_C2s_$out.log 2>&1
    echo "$tool C2s $out rc=$?: $(grep -E 'SUMMARY|^ok' $O/${tool}_C2s_$out.log | tr '\n' ' ')" >> $O/summary.txt
  done
done
cat $O/summary.txt
