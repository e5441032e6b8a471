python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pdl2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl2_tests.log
for rep in 1 2; do for v in 1 0; do echo "PDL=$v"; SPANQ_PDL=$v timeout 120 python tools/layer_gaps.py 2>&1 | tail -2; done; done
