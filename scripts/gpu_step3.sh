#!/bin/bash
# single-pass step with the packed row words (and w = NULL) vs the two launches; its GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/step3; mkdir -p $O
timeout 900 python -m pytest tests/test_step_gpu.py -q --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python scripts/step_sweep.py cfg4 f64 30 32,64,2048 32,64,2048,1 32,64,2048,2 > $O/sweep_f64.jsonl 2> $O/sweep_f64.err
EGFEM_CELLS_WORDS=0 timeout 600 python scripts/step_sweep.py cfg4 f64 30 32,64,2048 > $O/sweep_f64_w0.jsonl 2>> $O/sweep_f64.err
timeout 600 python scripts/step_sweep.py cfg4 f32 30 32,64,2048 > $O/sweep_f32.jsonl 2> $O/sweep_f32.err
timeout 600 python scripts/step_sweep.py cfg3 f64 30 32,64,2048 > $O/sweep_cfg3.jsonl 2> $O/sweep_cfg3.err
