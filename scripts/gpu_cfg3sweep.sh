#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/cfg3sw; mkdir -p $O; : > $O/ab.jsonl
for rep in 1 2; do for c in "2,3" "4,2" "8,1"; do for dt in f64 f32; do
EGFEM_CELLS_CFG=$c timeout 300 python scripts/rows_sweep.py cfg3 $dt | sed "s/^{/{\"G_CPL\": \"$c\", /" >> $O/ab.jsonl 2>> $O/err
done; done; done
