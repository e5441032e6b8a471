# A/B in one box: bash tools/ab.sh VAR "valA valB" [reps] [extra bench args]  (run under gpurun)
# prints C2 (d=128) and C4 (d=64) prefill / join kernel times for each value of the env knob VAR
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
nvidia-smi --query-gpu=serial --format=csv,noheader
for rep in $(seq ${3:-2}); do
for v in $2; do
  env $1=$v timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 20 $4 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); r=d['roofline']; j=d.get('judge', {})
print('$1=$v', 'step %.3f pre %.4f join %.4f | C4 pre %.4f join %.4f' % (d['ms_per_step'], r['kernel_ms'], d['join_kernel']['ms'], j.get('prefill_kernel_ms', 0), j.get('join_kernel_ms', 0)))"
done; done
