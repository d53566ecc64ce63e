cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dcgs2.py -x -q > gpurun_out/ob_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ob_pytest.log
bash scripts/gpu_orth_ab.sh ob "c3 c2" "auto reg"
MGB200_GMRES_LOOP=host timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --profile-from-start off --csv --kernel-name regex:"dcgs|k_reduce|scale_div" --log-file gpurun_out/ob_c3_dcgs2_warm.csv python scripts/profile_ops.py step --config c3 --orth dcgs2 > gpurun_out/ob_ncu.log 2>&1; echo "ncu rc=$?"
