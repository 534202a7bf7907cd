#!/bin/bash
# cell-kernel configurations (G, CPL) on cfg4 fp64 / fp32 with the packed words
cd $GRAFT_REPO_ROOT
O=gpurun_out/cfgsweep; mkdir -p $O; : > $O/ab.jsonl
for rep in 1 2; do for c in "8,3" "16,3" "16,4" "4,6"; do for dt in f64 f32; do
EGFEM_CELLS_CFG=$c timeout 300 python scripts/rows_sweep.py cfg4 $dt | sed "s/^{/{\"G_CPL\": \"$c\", /" >> $O/ab.jsonl 2>> $O/err
done; done; done
