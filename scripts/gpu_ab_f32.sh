#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/abf; mkdir -p $O; : > $O/ab.jsonl
L=paper_2005_06193_b200/lib
for rep in 1 2; do for v in "$@"; do
cp $L/variants/$v.so $L/libegfem.so
for c in "cfg4 f32" "cfg3 f32"; do timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"lib\": \"$v\", /" >> $O/ab.jsonl 2>> $O/err; done
done; done
