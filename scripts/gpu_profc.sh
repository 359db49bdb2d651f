cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/profc
python scripts/profile_iterate.py > gpurun_out/profc/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/profc/r02c_iterate_launches.csv python scripts/profile_iterate.py > gpurun_out/profc/ncu_list.log 2>&1; echo "list rc=$?"
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_tc_mlp -s 20 -c 1 -o gpurun_out/profc/r02c_k_tc_mlp_march python scripts/profile_iterate.py > gpurun_out/profc/ncu_mlp.log 2>&1; echo "mlp rc=$?"
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_tc_heads -s 0 -c 2 -o gpurun_out/profc/r02c_k_tc_heads python scripts/profile_iterate.py > gpurun_out/profc/ncu_heads.log 2>&1; echo "heads rc=$?"
tail -3 gpurun_out/profc/plain.log
ls -la gpurun_out/profc
