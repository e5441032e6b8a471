# A/B of the K/V ring depths at d=64 on the C4 judge line (two prebuilt libraries; run under gpurun)
mkdir -p gpurun_out
SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/libspanq_d64b.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "d64 or c4 or tiny" 2>&1 | tail -1
for rep in 1 2 3; do for L in libspanq_d64b.so libspanq_d64a.so; do
  SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/$L timeout 300 python bench.py --layers 1 --no-cpu-baseline --steps 10 > gpurun_out/r64.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r64.json').read().strip().splitlines()[-1]); j=d['judge']
print('$L c4 pre %.4f join %.4f | c2 pre %.4f join %.4f' % (j['prefill_kernel_ms'], j['join_kernel_ms'], d['roofline']['kernel_ms'], d['join_kernel']['ms']))"
done; done
