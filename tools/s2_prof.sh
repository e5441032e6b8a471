python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/p_smoke.log 2>&1; echo "smoke rc=$?"; tail -6 gpurun_out/p_smoke.log
bash tools/profile_round.sh > gpurun_out/p_round.log 2>&1
tail -c 3000 gpurun_out/prof/bench.json; echo; tail -c 600 gpurun_out/prof/bench_ref.json
