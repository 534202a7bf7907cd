#!/bin/bash
# single-pass step: GPU tests, then single pass vs two launches (cfg4 fp64 / fp32, cfg3, minsurf3d)
cd $GRAFT_REPO_ROOT
O=gpurun_out/step; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q -x --timeout 300 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 1
: > $O/step_sweep.jsonl
timeout 600 python scripts/step_sweep.py cfg4 f64 30 32,64,2048 32,64,2048,1 32,64,2048,2 >> $O/step_sweep.jsonl 2> $O/sweep.err
timeout 300 python scripts/step_sweep.py cfg4 f32 30 32,64,2048 >> $O/step_sweep.jsonl 2>> $O/sweep.err
timeout 300 python scripts/step_sweep.py cfg3 f64 30 32,64,2048 >> $O/step_sweep.jsonl 2>> $O/sweep.err
timeout 300 python scripts/step_sweep.py minsurf3d f64 30 32,64,2048 >> $O/step_sweep.jsonl 2>> $O/sweep.err
