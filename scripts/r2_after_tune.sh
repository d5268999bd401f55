# After the level-0 event tuning: C3 scale parity with the reseed null, the full C2 job line,
# then the C2 launch list and captures of the current kernels.
set -x
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py -m gpu -q -s -k "c3" > gpurun_out/at_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/at_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/at_bench_c2.jsonl 2> gpurun_out/at_bench_c2.err; echo "bench rc=$?"
cut -c1-330 gpurun_out/at_bench_c2.jsonl
bash scripts/prof_c2_r2.sh
