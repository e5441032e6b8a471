python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_partition.py tests/test_gpu_cidra.py -m gpu -v 2>&1 | tail -18
timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -c 600 gpurun_out/c5.json; tail -3 gpurun_out/c5.err
