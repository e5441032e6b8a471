mkdir -p gpurun_out
python -m paper_2511_02749_b200.build > /dev/null || exit 1
nvidia-smi --query-gpu=serial,clocks.sm --format=csv,noheader
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s2_tests.log 2>&1; tail -3 gpurun_out/s2_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/s2_smoke.log 2>&1; tail -4 gpurun_out/s2_smoke.log
timeout 300 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; tail -c 600 gpurun_out/s2_bench.json
for od in fp32 bf16 fp32 bf16; do
timeout 300 python bench.py --layers 1 --no-cpu-baseline --no-locality --out-dtype $od > gpurun_out/s2_b1_$od.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/s2_b1_$od.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$od', 'step %.3f pre %.3f join %.3f' % (d['ms_per_step'], r['kernel_ms'], d['join_kernel']['ms']))"
done
