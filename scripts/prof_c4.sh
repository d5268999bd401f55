# ncu evidence for the event-driven sampler on C4 (run under gpurun; one GPU): plain run,
# launch list, then one full-set capture of the longest k_sample launch.
set -x
C=${CFG:-c4}
B="python bench.py --config $C --rows-per-step ${ROWS:-16384} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/prof_${C}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${C}.csv $B > gpurun_out/prof_${C}_ncu1.log 2>&1; echo "launch rc=$?"
SKIP=$(python - "$C" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")) if len(r) > 14 and "k_sample" in r[4]]
t = [float(r[14]) for r in rows]
print(max(range(len(t)), key=t.__getitem__))
PY
)
echo "skip=$SKIP"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sample --launch-skip $SKIP --launch-count 1 -f -o gpurun_out/k_sample_${C} $B > gpurun_out/prof_${C}_ncu2.log 2>&1; echo "full rc=$?"
