#!/bin/bash
# A/B of the cell kernels: packed words vs staged slices, two repeats (rows_sweep cfg4 f64/f32, cfg3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/abw; mkdir -p $O; : > $O/ab.jsonl
for rep in 1 2; do for wv in 1 0; do
for c in "cfg4" "cfg4 f32" "cfg3"; do EGFEM_CELLS_WORDS=$wv timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"words\": $wv, /" >> $O/ab.jsonl 2>> $O/err; done
done; done
