# Round 2: the full GPU suite on the current default build, then the default bench line.
set -x
timeout 1800 python -m pytest tests -m gpu -q -rs ${PYTEST_K:+-k "$PYTEST_K"} --durations=12 > gpurun_out/su_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/su_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/su_smoke.log 2>&1; echo "smoke rc=$?"
