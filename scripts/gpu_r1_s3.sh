cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
for impl in seg rows; do
  for c in cfg4 cfg3 cfg2; do
    EGFEM_ROWS_IMPL=$impl timeout 300 python scripts/rows_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
  done
done
for rc in 32,3 32,4 16,6; do
  EGFEM_ROWS_CFG=$rc timeout 300 python scripts/rows_sweep.py cfg4 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
done
EGFEM_ROWS_CFG=32,3 timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
for rc in 16,4 8,4; do
  EGFEM_ROWS_CFG=$rc timeout 300 python scripts/rows_sweep.py cfg3 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
done
