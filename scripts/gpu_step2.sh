#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/step; mkdir -p $O
timeout 600 python scripts/step_sweep.py cfg4 f64 30 32,64,2048 32,64,2048,1 32,64,2048,2 32,256,2048,2 64,64,2048,1 > $O/sweep3_f64.jsonl 2> $O/sweep3_f64.err
EGFEM_STEP_NC=1 timeout 600 python scripts/step_sweep.py cfg4 f64 30 32,64,2048 32,64,2048,2 32,256,2048,2 > $O/sweep3nc_f64.jsonl 2> $O/sweep3nc_f64.err
