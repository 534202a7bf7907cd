cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
for cc in 2,3 4,4 16,3; do EGFEM_CELLS_CFG=$cc timeout 300 python scripts/rows_sweep.py cfg3 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
EGFEM_PATH=rows timeout 300 python scripts/rows_sweep.py cfg3 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
