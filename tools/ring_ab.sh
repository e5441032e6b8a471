# A/B of the K/V ring depths at d=128 (two prebuilt libraries; run under gpurun)
mkdir -p gpurun_out
SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/libspanq_k3v3.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_rag or full_size_c2 or multi_query" 2>&1 | tail -1
bash tools/ab_lib.sh libspanq_k3v3.so libspanq_k4v2.so 3
