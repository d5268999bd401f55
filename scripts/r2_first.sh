# Round-2 first GPU pass: gpu tests, default bench (short), reference arm, N=2 shared-device self-launch,
# then the C2 launch list and one full-set capture of the longest k_sample launch.
set -x
mkdir -p gpurun_out
nproc
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2_ref.log 2>&1; echo "ref rc=$?"
EXPMC_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_n2.log 2>&1; echo "n2 rc=$?"
CFG=c2 ROWS=16384 bash scripts/prof_c4.sh
python scripts/ncu_keys.py gpurun_out/k_sample_c2.ncu-rep gpurun_out/k_sample_c2_key_metrics.json > /dev/null; echo "keys rc=$?"
