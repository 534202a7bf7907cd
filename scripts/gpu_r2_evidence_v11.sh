#!/bin/bash
# Round-2 evidence run: smoke, tests, bench lines (all configs), reference arm, launch lists,
# ncu --set full of the hot kernels (cfg4 fp64/fp32, cfg5).  Outputs under gpurun_out/r2/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2v11; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.log 2>&1
lscpu > $O/lscpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --config cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>&1; done
timeout 600 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32.json 2>&1
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$|k_interp' -c 5 -o $O/prof_cfg4 -f python scripts/profile_cfg4_jac.py > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$|k_interp' -c 5 -o $O/prof_cfg4_f32 -f python scripts/profile_cfg4_jac.py f32 > $O/ncu_full32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:egfem_grp_0' -c 1 -o $O/prof_cfg5 -f python scripts/profile_cfg5.py > $O/ncu_full5.log 2>&1
# summaries on the box (gpurun copies back at most 64 MiB): text summaries, SASS stall tables,
# traffic.json; the full reports of cfg4 are dropped after summarising
for r in prof_cfg4 prof_cfg4_f32 prof_cfg5; do python scripts/ncu_summary.py $O/$r.ncu-rep > $O/$r.txt 2>&1; done
ncu -i $O/prof_cfg4.ncu-rep --page source --csv --print-source sass > $O/sass_cfg4.csv 2>/dev/null
python scripts/sass_stalls.py $O/sass_cfg4.csv 30 > $O/sass_cfg4_stalls.txt 2>&1
ncu -i $O/prof_cfg5.ncu-rep --page source --csv --print-source sass > $O/sass_cfg5.csv 2>/dev/null
python scripts/sass_stalls.py $O/sass_cfg5.csv 30 > $O/sass_cfg5_stalls.txt 2>&1
python scripts/make_traffic.py $O/prof_cfg4.ncu-rep $O/prof_cfg4_f32.ncu-rep $O/prof_cfg5.ncu-rep r2 $O/traffic.json  v11 > /dev/null 2>&1
rm -f $O/prof_cfg4.ncu-rep $O/prof_cfg4_f32.ncu-rep $O/sass_cfg4.csv $O/sass_cfg5.csv
fi
du -sh gpurun_out
ls -la $O
timeout 600 python scripts/geo_ab.py > $O/geo_ab.json 2> $O/geo_ab.err
