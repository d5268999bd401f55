# C2 A/B of the deferred finish (variants/defer.so) against the default build, twice each.
set -x
V=paper_1904_12754_b200/_lib/variants
for rep in 1 2; do
for v in default defer; do
  if [ $v = default ]; then L=""; else L="EXPMC_LIB=$PWD/$V/$v.so"; fi
  env $L timeout 600 python bench.py --rows-per-step 131072 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/df_${v}_$rep.log 2>&1; echo "$v rc=$?"
  python - gpurun_out/df_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
r = d["roofline"]
print(f"  value {d['value']:.4g} kernel_ms {r['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
done
done
EXPMC_LIB=$PWD/$V/defer.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_gpu_scale_parity.py -k "not graph_full_size" -m gpu -q -x > gpurun_out/df_pytest.log 2>&1; echo "defer pytest rc=$?"
