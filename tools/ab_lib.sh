# A/B of two builds in one box: bash tools/ab_lib.sh libA.so libB.so [reps] (run under gpurun; no rebuild)
nvidia-smi --query-gpu=serial --format=csv,noheader
for rep in $(seq ${3:-2}); do
for L in $1 $2; do
  SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/$L timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 20 > gpurun_out/ablib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ablib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$L', 'step %.3f pre %.3f join %.3f' % (d['ms_per_step'], r['kernel_ms'], d['join_kernel']['ms']))"
done; done
