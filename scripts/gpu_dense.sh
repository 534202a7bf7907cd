cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "batched or cfg5 or paths" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg5 --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2>&1
