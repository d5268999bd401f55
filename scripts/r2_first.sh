# Round-2 first GPU pass: gpu tests, default bench (short), reference arm, N=2 shared-device self-launch.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2_ref.log 2>&1; echo "ref rc=$?"
EXPMC_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_n2.log 2>&1; echo "n2 rc=$?"
nproc
