cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "small or interp or cfg4 or full or partition or minsurf or quad or f2" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
for c in cfg4 cfg3; do timeout 300 python scripts/rows_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
