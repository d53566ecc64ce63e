# Final code: memcheck + initcheck over every entry point (original driver, c1 / c3_small / c5_small,
# single GPU and LOCAL ranks) and the NEXT-row driver.
CS=/usr/local/cuda/bin/compute-sanitizer
python __graft_entry__.py build
for tool in memcheck initcheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_run.py c1 c3_small c5_small > gpurun_out/sanitize3_$tool.log 2>&1; echo "main $tool rc=$?"
  grep -E "ERROR SUMMARY" gpurun_out/sanitize3_$tool.log | tail -2
done
timeout 1500 $CS --tool memcheck --error-exitcode 9 python scripts/sanitize_next.py > gpurun_out/sanitize3_next.log 2>&1; echo "next memcheck rc=$?"
grep -E "ERROR SUMMARY" gpurun_out/sanitize3_next.log | tail -2
