cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum --cache-control none --clock-control none --profile-from-start off --csv"
for tma in 1 0; do
MGB200_DCGS_TMA=$tma MGB200_GMRES_LOOP=host timeout 900 ncu $M --kernel-name regex:"dcgs_(dots|update)" --log-file gpurun_out/p3_dcgs_tma$tma.csv python scripts/profile_ops.py step --config c3 --orth dcgs2 > gpurun_out/p3_$tma.log 2>&1; echo "tma$tma rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name regex:"prolong_csr|k_tsell" -o gpurun_out/p3_c3_transfers python scripts/profile_ops.py kernels --config c3 > gpurun_out/p3_tr.log 2>&1; echo "tr rc=$?"
