cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_seg' -c 4 -o gpurun_out/prof_seg2 -f python scripts/profile_cfg4_jac.py > gpurun_out/ncu_seg.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_seg.log
