# usage: bash tools/knob_sweep.sh VAR "v1 v2 ..."  (run under gpurun)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for v in $2; do
  env $1=$v timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 10 > gpurun_out/knob_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/knob_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1=$v', 'step %.3f ms pre %.3f ms frac %.3f join %.3f ms frac %.3f' % (d['ms_per_step'], r['kernel_ms'], r['frac'], d['join_kernel']['ms'], d['join_kernel']['frac']))"
  env $1=$v timeout 120 python tools/trace_step.py 0 prefill > gpurun_out/knob_${v}_trace.txt 2>&1
done
