# Level-0 kernel at 3 blocks/SM (variants/b0m3.so) vs the default (4): C2 job A/B, twice each.
set -x
V=paper_1904_12754_b200/_lib/variants
for rep in 1 2; do
  for v in default b0m3; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/m3_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/m3_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
