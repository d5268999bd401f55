# Round 2 session 4 run 1: the runs of session 3b whose results were lost with the container:
# full GPU suite at HEAD, EV0 vs queue level-0 SHA + C2 A/B, default bench + reference arm, smoke.
set -x
V=paper_1904_12754_b200/_lib/variants
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=12 > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_pytest.log
for v in default noev0; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/ev_$v.sha > gpurun_out/ev_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/ev_l0_$v.log
done
cat gpurun_out/ev_*.sha
for rep in 1 2; do
  for v in default noev0; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/ev_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
timeout 900 python bench.py > gpurun_out/s4_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s4_bench.log | cut -c1-600
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s4_smoke.log
