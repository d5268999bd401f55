# Level-0 kernel occupancy A/B after the event tuning (48 registers fit without loop spills):
# default (4 blocks/SM, 64 registers), b0m5 (5 blocks, 48 registers), b0m6 (6 blocks, 40 registers,
# 6 spill accesses per trip); then C4 / C3 with the 32-bit index helpers against the build before
# them (half), then the R-MAT scale-20 parity test.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default b0m5 b0m6; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/oc_$v.sha > gpurun_out/oc_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/oc_l0_$v.log
done
cat gpurun_out/oc_*.sha
show() { python - $1 <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
}
for rep in 1 2; do
  for v in default b0m5 b0m6; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/oc_${v}_$rep.log 2>&1; echo "$v rc=$?"; show gpurun_out/oc_${v}_$rep.log
  done
done
for cfg in c4 c3; do
  for v in default half; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 900 python bench.py --config $cfg --rows-per-step 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/oc_${cfg}_$v.log 2>&1; echo "$cfg $v rc=$?"; show gpurun_out/oc_${cfg}_$v.log
  done
done
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -m gpu -q -s -k "c4-20" > gpurun_out/oc_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/oc_pytest.log
