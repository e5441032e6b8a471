# A/B of two builds in one box: bash tools/ab_lib.sh libA.so libB.so [reps] [extra bench args]
# (run under gpurun; no rebuild). Prints C2 (d=128) and C4 (d=64) prefill / join kernel times.
nvidia-smi --query-gpu=serial --format=csv,noheader
for rep in $(seq ${3:-2}); do
for L in $1 $2; do
  SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/$L timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 20 $4 > gpurun_out/ablib.json 2>gpurun_out/ablib.err
  python -c "
import json; d=json.loads(open('gpurun_out/ablib.json').read().strip().splitlines()[-1]); r=d['roofline']; j=d.get('judge', {})
print('$L', 'step %.3f pre %.4f join %.4f | C4 pre %.4f join %.4f' % (d['ms_per_step'], r['kernel_ms'], d['join_kernel']['ms'], j.get('prefill_kernel_ms', 0), j.get('join_kernel_ms', 0)))" || tail -5 gpurun_out/ablib.err
done; done
