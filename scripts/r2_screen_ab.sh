# Round 2: geometric screen (event sampler) -- GPU tests of the event sampler, then C4 / C3 A/B of
# the round-1 kernel (head.so), the geometric screen at 4 blocks/SM (default build) and at 3 (skip3.so).
set -x
timeout 900 python -m pytest tests/test_gpu_ed.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"
V=paper_1904_12754_b200/_lib/variants
for cfg in c4 c3; do
  for v in head default skip3; do
    if [ $v = default ]; then L=""; else L="EXPMC_LIB=$PWD/$V/$v.so"; fi
    env $L timeout 900 python bench.py --config $cfg --rows-per-step 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab_${cfg}_$v.log 2>&1; echo "$cfg $v rc=$?"
    python - gpurun_out/ab_${cfg}_$v.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
r = d["roofline"]
print(f"  value {d['value']:.4g} rows/s {d['rows_per_s']:.0f} kernel_ms {r['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f} conv {d['completeness']['converged']} over {d['completeness']['over_budget']}")
PY
  done
done
