#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/lean; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32.json 2>> $O/bench.err
