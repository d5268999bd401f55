# C2 ncu evidence for round 2 (one GPU): plain run, launch list, then one full capture of the
# longest level-0 launch (k_sample<RefPolicy0>) and of the longest general launch
# (k_sample<RefPolicy<false>>), with their key metrics and SASS source pages.
set -x
B="python bench.py --config c2 --rows-per-step 16384 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/p2_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r2.csv $B > gpurun_out/p2_ncu1.log 2>&1; echo "launch rc=$?"
for K in RefPolicy0 9RefPolicyILb0EEELb0E; do
  SKIP=$(python - "$K" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/launches_c2_r2.csv")) if len(r) > 14 and "k_sample" in r[4]]
key = "RefPolicy0" if sys.argv[1] == "RefPolicy0" else "RefPolicy<"
sel = [float(r[14]) for r in rows if key in r[4]]
print(max(range(len(sel)), key=sel.__getitem__))
PY
)
  echo "$K skip=$SKIP"
  timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$K --launch-skip $SKIP --launch-count 1 -f -o gpurun_out/k_sample_c2_$K $B > gpurun_out/p2_ncu_$K.log 2>&1; echo "full $K rc=$?"
  python scripts/ncu_keys.py gpurun_out/k_sample_c2_$K.ncu-rep gpurun_out/k_sample_c2_${K}_key_metrics.json > /dev/null; echo "keys rc=$?"
  ncu -i gpurun_out/k_sample_c2_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/k_sample_c2_${K}_sass.csv 2>/dev/null; echo "sass rc=$?"
  rm -f gpurun_out/k_sample_c2_$K.ncu-rep
done
