# Session 3 run 2: split-invariant geometric screen + one-block-per-event level-0 stream (EV0).
# Event-sampler tests, parity suite, level-0 SHA A/B (EV0 vs queue), C2 A/B, C3 scale diagnostic.
set -x
V=paper_1904_12754_b200/_lib/variants
timeout 1200 python -m pytest tests/test_gpu_ed.py tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_gpu_edges.py tests/test_alias.py -m gpu -q -rs > gpurun_out/s3b_pytest.log 2>&1; echo "pytest rc=$?"
for v in default noev0; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/ev_$v.sha > gpurun_out/ev_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/ev_l0_$v.log
done
cat gpurun_out/ev_*.sha
for rep in 1 2; do
  for v in default noev0; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ev_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/ev_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
timeout 1500 python scripts/scale_diag.py c3 > gpurun_out/diag_c3.log 2>&1; echo "diag rc=$?"
