# State check of HEAD on a fresh box: smoke, the full GPU suite, then both bench arms (C2).
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/h_pytest.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/h_bench_ref.jsonl 2> gpurun_out/h_bench_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/h_bench_c2.jsonl 2> gpurun_out/h_bench_c2.err; echo "bench rc=$?"
cat gpurun_out/h_bench_c2.jsonl | cut -c1-600
