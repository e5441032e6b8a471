python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for pm in 0 1 2 3; do
  SPANQ_POLY_EXP=$pm timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 10 > gpurun_out/pm${pm}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pm${pm}.json').read().strip().splitlines()[-1]); r=d['roofline']
print('pm ${pm}', 'pre %.3f ms frac %.3f join %.3f ms frac %.3f' % (r['kernel_ms'], r['frac'], d['join_kernel']['ms'], d['join_kernel']['frac']))"
done
