# Quick GPU check during development: the -m gpu tests, then per-kernel times of the hot path on
# cfg4 (fp64, fp32) and cfg3 (scripts/rows_sweep.py).  Usage: gpurun -- 'bash scripts/gpu_quick.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
for c in cfg4 cfg3; do timeout 300 python scripts/rows_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
