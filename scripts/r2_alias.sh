# Round 2: full GPU suite (graph scale fixtures pending), C5 reference-order vs event+alias,
# then the C4 launch list and a full capture of its longest k_sample_grouped launch.
set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -k "not graph_full_size" --durations=10 > gpurun_out/al_pytest.log 2>&1; echo "pytest rc=$?"
for s in reference event; do
  timeout 900 python bench.py --config c5 --sampler $s --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/al_c5_$s.log 2>&1; echo "c5 $s rc=$?"
  python - gpurun_out/al_c5_$s.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
r = d["roofline"]
print(f"  value {d['value']:.4g} rows/s {d['rows_per_s']:.0f} kernel_ms {r['kernel_ms']:.1f} ms/step {d['ms_per_step']:.1f} conv {d['completeness']['converged']} over {d['completeness']['over_budget']}")
PY
done
CFG=c4 ROWS=65536 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c4.ncu-rep gpurun_out/k_sample_c4_key_metrics.json > /dev/null; echo "keys rc=$?"
