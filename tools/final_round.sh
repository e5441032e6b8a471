# Final validation + profiling pass of a round (run under gpurun): GPU tests, smoke, ncu captures,
# launch list, bench (default) and the reference arm
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/fr_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fr_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/fr_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/fr_smoke.log
bash tools/profile_round.sh > gpurun_out/p_round.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/prof/bench.json').read().strip().splitlines()[-1])
print('value %.1f step %.3f l1 %.3f plan %.3f pre %.4f (%.3f) join %.4f (%.3f)' % (d['value'], d['ms_per_step'], d['ttft_l1_ms'], d['plan_host_ms'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['join_kernel']['ms'], d['join_kernel']['frac']))
print(d['judge']); print(d['reposition']['ms'], d['reposition']['frac'])"
