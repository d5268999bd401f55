# Captures on the final build: C2 (launch list, level-0 and general walker kernels) and C3 (grouped
# event kernel).
set -x
bash scripts/prof_c2_r2.sh
CFG=c3 ROWS=65536 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c3.ncu-rep gpurun_out/k_sample_c3_key_metrics.json > /dev/null; echo "keys rc=$?"
rm -f gpurun_out/k_sample_c3.ncu-rep
