# A/B of the event sampler's closed-form first hold on C3/C4 (run under gpurun; one GPU).
set -x
timeout 600 python -m pytest tests/test_gpu_ed.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"
for c in c3 c4; do
  for m in "" "--full-hold"; do
    timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $m > gpurun_out/ab_${c}${m}.log 2>&1
    echo "$c $m rc=$?"; tail -1 gpurun_out/ab_${c}${m}.log | cut -c1-600
  done
done
