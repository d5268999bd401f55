# Round 2: per-edge records (EdgeRec) A/B on C4 / C3 (runtime flag --row-gather), product-form
# S-mode (variants/prod.so) A/B on C2 and its parity suite.
set -x
timeout 900 python -m pytest tests/test_gpu_ed.py tests/test_alias.py -m gpu -q -x > gpurun_out/ep_pytest.log 2>&1; echo "pytest rc=$?"
show() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
r = d["roofline"]
print(f"  value {d['value']:.4g} kernel_ms {r['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f}")
PY
}
for cfg in c4 c3; do
  for v in erec rowgather; do
    F=""; [ $v = rowgather ] && F="--row-gather"
    timeout 900 python bench.py --config $cfg --rows-per-step 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $F > gpurun_out/ep_${cfg}_$v.log 2>&1; echo "$cfg $v rc=$?"; show gpurun_out/ep_${cfg}_$v.log
  done
done
V=paper_1904_12754_b200/_lib/variants
for rep in 1 2; do
  for v in default prod; do
    L=""; [ $v = prod ] && L="EXPMC_LIB=$PWD/$V/prod.so"
    env $L timeout 600 python bench.py --rows-per-step 131072 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ep_c2_${v}_$rep.log 2>&1; echo "c2 $v rc=$?"; show gpurun_out/ep_c2_${v}_$rep.log
  done
done
EXPMC_LIB=$PWD/$V/prod.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_fem.py tests/test_forward.py tests/test_gpu_scale_parity.py -k "not graph_full_size" -m gpu -q > gpurun_out/ep_prod_pytest.log 2>&1; echo "prod pytest rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/ep_cfg_pytest.log 2>&1; echo "cfg pytest rc=$?"
timeout 1800 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/ep_c4_line.log 2>&1; echo "c4 line rc=$?"
