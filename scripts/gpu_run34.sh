python __graft_entry__.py build
python scripts/initcheck_probe.py ns; echo "plain ns rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
for args in "ns" "ns graphs" "ch graphs"; do
timeout 600 $CS --tool initcheck --print-limit 2 python scripts/initcheck_probe.py $args > gpurun_out/initprobe.log 2>&1; echo "initcheck $args rc=$?"
grep -E "SUMMARY" gpurun_out/initprobe.log; grep -A12 -m1 "Uninitialized\|Invalid" gpurun_out/initprobe.log
done
timeout 600 $CS --tool memcheck python scripts/initcheck_probe.py ns graphs 2>&1 | grep SUMMARY; echo "memcheck ns graphs"
timeout 1500 python -m pytest tests/test_gpu_ns.py tests/test_gpu_vanka.py tests/test_gpu_newton.py -q > gpurun_out/gpu_t34.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_t34.log
