# Event-walker stream A/B (grouped kernel): default (queued keyless stream), edev (one Philox block
# per event, no queue), edevpf (+ prefetch of the landing row's u), edevpf4 (the same at 4 blocks
# per SM, 64 registers).  Bitwise check of run_level batches on C3, then C4 / C3 steps.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default edev edevpf edevpf4; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/ed_ab.py gpurun_out/ed_$v.sha > gpurun_out/ed_ab_$v.log 2>&1; echo "$v rc=$?"; tail -3 gpurun_out/ed_ab_$v.log
done
cat gpurun_out/ed_*.sha
show() { python - $1 <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
}
for cfg in c4 c3; do
  for v in default edev edevpf edevpf4; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 900 python bench.py --config $cfg --rows-per-step 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ed_${cfg}_$v.log 2>&1; echo "$cfg $v rc=$?"; show gpurun_out/ed_${cfg}_$v.log
  done
done
