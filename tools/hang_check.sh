# The unpaired-launch stress that hung before the slot-B fix (commit message of the fix): lib/libspanq_epi.so
# was a build with the paired-chunk epilogue variant (SPANQ_EPI_PAIRS), which shifts the Q-prep timing.
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
for i in $(seq 6); do
  SPANQ_EPI_PAIRS=1 SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/libspanq_epi.so timeout 150 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c1_fp32 or small_rag or ragged_gqa1" > gpurun_out/hc_$i.log 2>&1; echo "epi-variant seq $i rc=$?"
done
timeout 500 python -m pytest tests -m gpu -q > gpurun_out/hc_all.log 2>&1; echo "all rc=$?"; tail -2 gpurun_out/hc_all.log
