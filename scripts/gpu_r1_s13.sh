cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in quadratic_i4 biochem_i2 plap_i1 plap3d_i2; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/bench_$c.json 2>&1; done
