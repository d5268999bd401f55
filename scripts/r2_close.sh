# Closing run on the final build: smoke, the full GPU suite, both C2 bench arms.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cl_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/cl_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/cl_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cl_pytest.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cl_c2_ref.jsonl 2> gpurun_out/cl_c2_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/cl_c2.jsonl 2> gpurun_out/cl_c2.err; echo "c2 rc=$?"
python - gpurun_out/cl_c2.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(f"value {d['value']:.4g} ms/step {d['ms_per_step']:.1f} e2e {d['e2e']['ms_per_step']:.1f} kernel_ms/step {d['roofline']['kernel_ms'] / d['steps']:.1f} cpu {d['cpu_baseline']['value']:.3g}")
PY
