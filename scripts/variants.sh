#!/bin/bash
# usage: bash scripts_variants.sh <rows> <names...>   -- bench each library variant (experiments only)
rows=$1; shift
for m in "$@"; do
  EXPMC_LIB=$PWD/paper_1904_12754_b200/_lib/variants/$m.so timeout 300 python bench.py --rows-per-step $rows --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$m.log 2>&1
  echo "$m rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/var_$m.log').read().splitlines()[-1]);print('  value %.4g rows/s %.0f kernel_ms %.1f ms/step %.1f share %.3f' % (d['value'],d['rows_per_s'],d['roofline']['kernel_ms'],d['ms_per_step'],d['roofline']['step_share']))"
done
