python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 400 python -m pytest tests -m gpu -v > gpurun_out/t6_$i.log 2>&1; echo "run $i rc=$?"; tail -2 gpurun_out/t6_$i.log
done
timeout 300 python bench.py --layers 1 --no-cpu-baseline --no-locality > gpurun_out/t6_b1.json 2> gpurun_out/t6_b1.err; tail -c 1500 gpurun_out/t6_b1.json
