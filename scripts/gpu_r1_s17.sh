cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
EGFEM_CELLS_STAGE=bulk timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "small or fused or cfg4 or partition or fp32" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
for st in cp bulk; do for c in cfg4 cfg3; do EGFEM_CELLS_STAGE=$st timeout 300 python scripts/rows_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done; done
EGFEM_CELLS_STAGE=bulk timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
