# Round-2 closing evidence on the current build: the full GPU suite and smoke, the C2 / C4 / C3
# whole-job lines, the C5 line, and the C4 capture of the current grouped kernel.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fl_smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/fl_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fl_pytest.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fl_c2_ref.jsonl 2> gpurun_out/fl_c2_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/fl_c2.jsonl 2> gpurun_out/fl_c2.err; echo "c2 rc=$?"
timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/fl_c4.jsonl 2> gpurun_out/fl_c4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e > gpurun_out/fl_c3.jsonl 2> gpurun_out/fl_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-e2e > gpurun_out/fl_c5.jsonl 2> gpurun_out/fl_c5.err; echo "c5 rc=$?"
for f in c2 c4 c3 c5; do python - gpurun_out/fl_$f.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(sys.argv[1], f"value {d['value']:.4g} ms/step {d['ms_per_step']:.1f} e2e {d['e2e'] and d['e2e'].get('ms_per_step')} kernel_ms/step {d['roofline']['kernel_ms'] / d['steps']:.1f}")
PY
done
CFG=c4 ROWS=65536 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c4.ncu-rep gpurun_out/k_sample_c4_key_metrics.json > /dev/null; echo "keys rc=$?"
rm -f gpurun_out/k_sample_c4.ncu-rep
