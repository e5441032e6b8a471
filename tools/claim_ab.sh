# A/B of the prefill claim-ahead limit (run under gpurun)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
SPANQ_CLAIM_AHEAD=1 timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/ab.sh SPANQ_CLAIM_AHEAD "1 0" 3
