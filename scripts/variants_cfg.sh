#!/bin/bash
# usage: bash scripts/variants_cfg.sh <config> <names...> -- bench library variants on a config (experiments only)
cfg=$1; shift
for m in "$@"; do
  EXPMC_LIB=$PWD/paper_1904_12754_b200/_lib/variants/$m.so timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/var_${cfg}_$m.log 2>&1
  echo "$cfg $m rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/var_${cfg}_$m.log').read().splitlines()[-1]);print('  value %.4g rows/s %.0f kernel_ms %.1f ms/step %.1f' % (d['value'],d['rows_per_s'],d['roofline']['kernel_ms'],d['ms_per_step']))"
done
