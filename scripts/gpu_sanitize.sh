CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_run.py c1 c3_small c5_small > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok \(" gpurun_out/sanitize_$tool.log | tail -4
done
