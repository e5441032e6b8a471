python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cidra.py -m gpu -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-locality --steps 5 > gpurun_out/cr.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/cr.json').read().strip().splitlines()[-1]); r=d['reposition']; print('cidra ms %.4f frac %.3f' % (r['ms'], r['frac']))"; done
