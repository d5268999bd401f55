# ncu evidence for profiles/r01 (run under gpurun; one GPU).  Plain run first, then the launch
# list, then one full-set capture of a C2 main-round k_sample launch (the 76 ms one).
set -x
B="python bench.py --rows-per-step 16384 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/prof_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv $B > gpurun_out/prof_ncu1.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sample --launch-skip ${SKIP:-38} --launch-count 1 -f -o gpurun_out/k_sample_r1g $B > gpurun_out/prof_ncu2.log 2>&1; echo "full rc=$?"
