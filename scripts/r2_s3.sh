# Round 2 session 3: GPU suite on the rebuilt tree (C3 scale fixture in; R-MAT-20 pending),
# default bench line, reference arm, smoke, and the self-launching two-rank bench on one device.
set -x
timeout 2400 python -m pytest tests -m gpu -q -rs -k "not c4-20" --durations=12 > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/s3_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/s3_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc=$?"
EXPMC_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/s3_g2.log 2>&1; echo "g2 rc=$?"
