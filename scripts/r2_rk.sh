# Round keys in shared memory for the level-0 walker (variants/rk.so) vs the default: level-0
# pass (bitwise check by SHA-256) and C2 job A/B, twice each.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default rk; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/rk_$v.sha > gpurun_out/rk_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/rk_l0_$v.log
done
cat gpurun_out/rk_*.sha
for rep in 1 2; do
  for v in default rk; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/rk_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/rk_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
