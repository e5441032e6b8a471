# A/B of the K1 (rope_kv_write) layouts: parity with the new build, ncu kernel times of both
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for L in libspanq_k1new.so libspanq_k1old.so libspanq_k1new.so libspanq_k1old.so; do
SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rope_kv_write --csv python tools/profile_step.py 3 2>/dev/null | grep rope_kv_write | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo " $L"
done
