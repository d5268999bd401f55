# C2 A/B: default (in-tree build), prep (item constants prepared once per run of an item's
# chunks), qend (prep + the word queue advanced once per event); level-0 SHA check, C2 jobs.
set -x
V=paper_1904_12754_b200/_lib/variants
for v in default prep qend; do
  L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
  env $L timeout 600 python scripts/level0_ab.py gpurun_out/pq_$v.sha > gpurun_out/pq_l0_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/pq_l0_$v.log
done
cat gpurun_out/pq_*.sha
for rep in 1 2; do
  for v in default prep qend; do
    L=""; [ $v != default ] && L="EXPMC_LIB=$PWD/$V/$v.so"
    env $L timeout 600 python bench.py --rows-per-step 262144 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/pq_${v}_$rep.log 2>&1; echo "$v rc=$?"
    python - gpurun_out/pq_${v}_$rep.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"  value {d['value']:.4g} kernel_ms {d['roofline']['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
  done
done
EXPMC_LIB=$PWD/$V/qend.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_fem.py tests/test_forward.py tests/test_gpu_edges.py tests/test_gpu_scale_parity.py -k "not graph_full_size" -m gpu -q > gpurun_out/pq_pytest.log 2>&1; echo "qend pytest rc=$?"
