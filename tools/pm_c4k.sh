# A/B of the FMA-pipe exp2 share on the d=64 C4 attention kernels (judge line kernel times)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for rep in 1 2; do for pm in 0 1 2; do
  SPANQ_POLY_EXP=$pm timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 10 > gpurun_out/pmk.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pmk.json').read().strip().splitlines()[-1]); j=d['judge']
print('pm $pm c4 prefill %.4f join %.4f | c2 pre %.4f join %.4f' % (j['prefill_kernel_ms'], j['join_kernel_ms'], d['roofline']['kernel_ms'], d['join_kernel']['ms']))"
done; done
