python __graft_entry__.py build
timeout 1200 python scripts/ns_long_run.py --steps 40000 --sample 5000 --vanka > gpurun_out/ns_long_vanka.jsonl 2> gpurun_out/ns_long_vanka.err; echo "vanka rc=$?"
tail -3 gpurun_out/ns_long_vanka.jsonl; tail -3 gpurun_out/ns_long_vanka.err
timeout 1500 python scripts/ns_long_run.py --steps 40000 --sample 10000 > gpurun_out/ns_long_jacobi.jsonl 2> gpurun_out/ns_long_jacobi.err; echo "jacobi rc=$?"
tail -2 gpurun_out/ns_long_jacobi.jsonl; tail -3 gpurun_out/ns_long_jacobi.err
