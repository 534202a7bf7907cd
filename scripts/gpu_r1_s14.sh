cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "batched or cfg5 or paths" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg5 --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_dense -c 30 --csv python bench.py --config cfg5 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ncu_dense.csv 2>&1
