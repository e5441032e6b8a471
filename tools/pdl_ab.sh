# programmatic dependent launch: full GPU tests (PDL on by default) + A/B of a 40-layer step
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_tests.log
for rep in 1 2; do for v in 1 0; do echo "PDL=$v"; SPANQ_PDL=$v timeout 120 python tools/layer_gaps.py 2>&1 | tail -2; done; done
for v in 1 0; do SPANQ_PDL=$v timeout 300 python bench.py --no-cpu-baseline --no-locality --steps 10 > gpurun_out/pdlb.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/pdlb.json').read().strip().splitlines()[-1]); print('PDL=$v value %.1f step %.3f e2e %.1f (%.3f ms)' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step']))"; done
