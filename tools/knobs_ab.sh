# A/B of several runtime knobs on the current build (run under gpurun)
python -m paper_2511_02749_b200.build > /dev/null; mkdir -p gpurun_out
bash tools/ab.sh SPANQ_QROT_TABLE "1 0" 2
bash tools/ab.sh SPANQ_QRING2 "2 1" 2
bash tools/ab.sh SPANQ_RESCALE_THRESHOLD "12 8" 2
