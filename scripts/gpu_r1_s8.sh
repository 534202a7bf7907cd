cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg5 --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2>&1
EGFEM_BATCHED=csf timeout 600 python bench.py --config cfg5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_cfg5_csf.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_dense' -c 1 -o gpurun_out/prof_dense -f python bench.py --config cfg5 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ncu_dense.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_dense.log
