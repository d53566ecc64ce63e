python __graft_entry__.py build
CS=/usr/local/cuda/bin/compute-sanitizer
for mode in ns ch; do
timeout 600 $CS --tool initcheck --print-limit 3 python scripts/initcheck_probe.py $mode > gpurun_out/initprobe_$mode.log 2>&1; echo "$mode rc=$?"
grep -E "SUMMARY" gpurun_out/initprobe_$mode.log
head -40 gpurun_out/initprobe_$mode.log
done
