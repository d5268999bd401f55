# One full capture of the longest level-0 launch of a 16,384-component C2 step, report kept.
set -x
B="python bench.py --config c2 --rows-per-step 16384 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:RefPolicy0 --launch-skip 2 --launch-count 1 -f -o gpurun_out/k_l0 $B > gpurun_out/cap_l0.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/k_l0.ncu-rep
python scripts/ncu_keys.py gpurun_out/k_l0.ncu-rep gpurun_out/k_sample_c2_key_metrics.json > /dev/null; echo "keys rc=$?"
