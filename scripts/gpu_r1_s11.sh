cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
timeout 300 python scripts/rows_sweep.py cfg4 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
EGFEM_CELLS_CFG=16,2 timeout 300 python scripts/rows_sweep.py cfg4 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
EGFEM_CELLS_CFG=16,2 timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
EGFEM_CELLS_CFG=16,2 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$' -c 4 -o gpurun_out/prof_cell -f python scripts/profile_cfg4_jac.py > gpurun_out/ncu_cell.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_cell.log
