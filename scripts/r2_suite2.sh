# Full GPU suite on the current default build (graph scale fixtures pending), then the C4
# capture of the current event-sampler kernel (edge records).
set -x
timeout 1800 python -m pytest tests -m gpu -q -rs -k "not graph_full_size" --durations=8 > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?"
CFG=c4 ROWS=65536 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c4.ncu-rep gpurun_out/k_sample_c4_key_metrics.json > /dev/null; echo "keys rc=$?"
rm -f gpurun_out/k_sample_c4.ncu-rep
