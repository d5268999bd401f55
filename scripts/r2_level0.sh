# Level-0 kernel experiment (RefPolicy0): level-0 run_level over every C2 component with the
# default build, b0 (Walker0, 4 blocks/SM) and b0m5 (5 blocks/SM); results must be bitwise equal.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default b0 b0m5; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/l0_$v.sha > gpurun_out/l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/l0_$v.log
done
cat gpurun_out/l0_*.sha
