# Level-0 walker A/B: t2 = the holding test on the 2^64 scale (no 64-bit shift / subtract) and the
# sample loop ending on a count instead of a vote, vs the in-tree build.  Level-0 SHA check, C2
# jobs, then the parity tests on the variant.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default t2; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/t2_$v.sha > gpurun_out/t2_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/t2_l0_$v.log
done
cat gpurun_out/t2_*.sha
for rep in 1 2; do
  for v in default t2; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/t2_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/t2_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
EXPMC_LIB=$PWD/$V/t2.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t2_pytest.log
