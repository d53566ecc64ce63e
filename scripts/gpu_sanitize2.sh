CS=/usr/local/cuda/bin/compute-sanitizer
python __graft_entry__.py build
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_next.py > gpurun_out/sanitize2_$tool.log 2>&1; echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/sanitize2_$tool.log | tail -5
done
