python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 120 python tools/trace_step.py 0 prefill > gpurun_out/t_pre5.txt 2>&1
for e in 0 0.75 1.5; do for so in 2 3 5; do
  SPANQ_EPOCH_COST=$e SPANQ_SUB_OVERHEAD=$so timeout 300 python bench.py --layers 1 --no-cpu-baseline --no-locality --steps 20 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1])
print('epoch $e sub $so join %.4f pre %.4f' % (d['join_kernel']['ms'], d['roofline']['kernel_ms']))"
done; done
