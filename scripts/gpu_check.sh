# Development check: selected -m gpu tests (PYTEST_K) and short bench lines.  Usage:
#   gpurun -- 'PYTEST_K="overlap or partition" bash scripts/gpu_check.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for c in ${BENCH_CFGS:-cfg1}; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err; done
