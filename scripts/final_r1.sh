# Round-1 closing measurements (one GPU): C2 ncu capture of the final kernel, full-size C3/C4.
set -x
CFG=c2 ROWS=16384 bash scripts/prof_c4.sh
timeout 900 python bench.py --config c3 --rows-per-step 1000000 --steps 1 --warmup 1 --no-e2e > gpurun_out/full_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --rows-per-step 1048576 --steps 1 --warmup 1 --no-e2e > gpurun_out/full_c4.log 2>&1; echo "c4 rc=$?"
