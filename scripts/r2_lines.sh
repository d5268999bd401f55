# Round 2: GPU tests touched since the last pass, then bench lines (C2 default, C4 whole job,
# C3 whole job) and a C3 capture.
set -x
timeout 900 python -m pytest tests/test_alias.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/ln_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/ln_c2.log 2>&1; echo "c2 rc=$?"
timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/ln_c4.log 2>&1; echo "c4 rc=$?"
timeout 1500 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e > gpurun_out/ln_c3.log 2>&1; echo "c3 rc=$?"
CFG=c3 ROWS=65536 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c3.ncu-rep gpurun_out/k_sample_c3_key_metrics.json > /dev/null; echo "keys rc=$?"
