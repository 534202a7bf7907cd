cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
timeout 300 python scripts/rows_sweep.py cfg4 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
timeout 300 python scripts/rows_sweep.py cfg3 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_seg' -c 5 -o gpurun_out/prof_seg -f python scripts/rows_sweep.py cfg4 > gpurun_out/ncu_seg.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_seg.log
