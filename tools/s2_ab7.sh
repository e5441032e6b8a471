mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/ab_lib.sh libspanq_new.so libspanq_old.so 3
timeout 300 python bench.py --layers 1 --no-cpu-baseline > gpurun_out/j1.json 2> gpurun_out/j1.err; tail -c 1200 gpurun_out/j1.json; tail -3 gpurun_out/j1.err
