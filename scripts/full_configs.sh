# Full-size C3 / C4 / C5 bench lines (run under gpurun; one GPU).
set -x
timeout 900 python bench.py --config c3 --rows-per-step 1000000 --steps 1 --warmup 1 --no-e2e > gpurun_out/full_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --rows-per-step 1048576 --steps 1 --warmup 1 --no-e2e > gpurun_out/full_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-e2e > gpurun_out/full_c5.log 2>&1; echo "c5 rc=$?"
