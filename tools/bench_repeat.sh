python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,serial,clocks.sm,temperature.gpu,power.draw --format=csv,noheader
for i in 1 2 3; do
  timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 20 > gpurun_out/rep_$i.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/rep_$i.json').read().strip().splitlines()[-1]); r=d['roofline']
print('rep $i', 'step %.3f pre %.3f join %.3f' % (d['ms_per_step'], r['kernel_ms'], d['join_kernel']['ms']), d['clocks'])"
done
