# A/B of the paired-chunk epilogue (run under gpurun)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
SPANQ_EPI_PAIRS=1 timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/ab.sh SPANQ_EPI_PAIRS "1 0" 3
