# Keyless-stream event walker in the grouped kernel (variants/gk.so) vs the in-tree build: C4 / C3.
set -x
V=paper_1904_12754_b200/_lib/variants
for cfg in c4 c3; do
  for v in default gk; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 900 python bench.py --config $cfg --rows-per-step 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/gk_${cfg}_$v.log 2>&1; echo "$cfg $v rc=$?"
    python - gpurun_out/gk_${cfg}_$v.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
EXPMC_LIB=$PWD/$V/gk.so timeout 900 python -m pytest tests/test_gpu_ed.py tests/test_gpu_configs.py tests/test_gpu_shard.py tests/test_alias.py -m gpu -q > gpurun_out/gk_pytest.log 2>&1; echo "gk pytest rc=$?"
