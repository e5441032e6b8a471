mkdir -p gpurun_out
for L in libspanq_new.so libspanq_old.so libspanq_new.so libspanq_old.so; do
SPANQ_LIB=$PWD/paper_2511_02749_b200/lib/$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rope_kv_write --csv python tools/profile_step.py 3 2>/dev/null | grep rope_kv_write | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo " $L"
done
bash tools/ab_lib.sh libspanq_new.so libspanq_old.so 2
