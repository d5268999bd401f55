# A/B of the event sampler's closed-form first hold on C3/C4 (run under gpurun; one GPU).
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"
for c in ${CFGS:-c3 c4}; do
  for m in "" "--full-hold"; do
    timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $m > gpurun_out/ab_${c}${m}.log 2>&1
    echo "$c $m rc=$?"
  done
done
