#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/geo4; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python scripts/geo_ab.py > $O/geo_ab.json 2> $O/geo_ab.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$|k_interp' -c 5 -o $O/prof_cfg4_f32 -f python scripts/profile_cfg4_jac.py f32 > $O/ncu_full32.log 2>&1
python scripts/ncu_summary.py $O/prof_cfg4_f32.ncu-rep > $O/prof_cfg4_f32.txt 2>&1
rm -f $O/prof_cfg4_f32.ncu-rep
