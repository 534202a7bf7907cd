# Round-1 evidence run: tests, smoke, bench lines (all configs), reference arm, launch list,
# ncu --set full of the step's kernels, FP64 peak.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.log 2>&1
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in cfg1 cfg2 cfg3 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1; done
timeout 600 python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench_f32.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$|k_interp' -c 5 -o gpurun_out/prof_cfg4 -f python scripts/profile_cfg4_jac.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
