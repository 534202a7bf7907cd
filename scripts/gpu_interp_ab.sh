#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/interp; mkdir -p $O; : > $O/ab.jsonl
for rep in 1 2; do for ch in 0 1; do for c in "cfg4" "cfg4 f32" "cfg3"; do
EGFEM_INTERP_CHUNK=$ch timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"chunk\": $ch, /" >> $O/ab.jsonl 2>> $O/err
done; done; done
