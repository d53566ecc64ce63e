cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dcgs2.py tests/test_gpu_parity.py -x -q > gpurun_out/p4_pytest.log 2>&1; tail -2 gpurun_out/p4_pytest.log
M="--metrics gpu__time_duration.sum --cache-control none --clock-control none --profile-from-start off --csv"
MGB200_GMRES_LOOP=host timeout 900 ncu $M --kernel-name regex:"dcgs_(dots|update)|prolong_csr|k_tsell|k_reduce" --log-file gpurun_out/p4_c3_kernels.csv python scripts/profile_ops.py step --config c3 --orth dcgs2 > gpurun_out/p4_1.log 2>&1; echo "ncu rc=$?"
bash scripts/gpu_ab.sh p4 "c3 e6" "MGB200_DCGS_TMA=0"
