#!/bin/bash
# Geometry-class interp: tests, A/B timing, bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/geo; mkdir -p $O
timeout 900 python -m pytest tests/test_geo_gpu.py tests/test_step_gpu.py -q --timeout 600 > $O/pytest_geo.log 2>&1; echo "rc=$?" >> $O/pytest_geo.log
timeout 600 python scripts/geo_ab.py > $O/geo_ab.json 2> $O/geo_ab.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
