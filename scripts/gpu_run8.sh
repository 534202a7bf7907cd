cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/profile_cfg4_jac.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_rows' -c 4 -o gpurun_out/prof_cfg4_v7 -f python scripts/profile_cfg4_jac.py > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
