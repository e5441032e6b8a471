# A/B of the FMA-pipe exp2 share on the 2B-shape (d=64) judge workload (run under gpurun)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for rep in 1 2; do for pm in 0 1 2; do
  SPANQ_POLY_EXP=$pm timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 10 > gpurun_out/pmc4.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pmc4.json').read().strip().splitlines()[-1]); j=d['judge']
print('pm $pm c4 cold %.3f warm %.3f | c2 pre %.4f join %.4f' % (j['cold_ttft_l1_ms'], j['warm_ttft_l1_ms'], d['roofline']['kernel_ms'], d['join_kernel']['ms']))"
done; done
