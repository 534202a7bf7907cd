cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
for c in cfg4 cfg3; do timeout 300 python scripts/rows_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; done
timeout 300 python scripts/rows_sweep.py cfg4 f32 >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$' -c 4 -o gpurun_out/prof_cell -f python scripts/profile_cfg4_jac.py > gpurun_out/ncu_cell.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_cell.log
