#!/bin/bash
# A/B of library variants (lib/variants/*.so copied over lib/libegfem.so in turn): rows_sweep cfg4
# f64 / f32 and cfg3, two rounds.  usage: gpurun -- 'bash scripts/gpu_ab_libs.sh v1 v2 ...'
cd $GRAFT_REPO_ROOT
O=gpurun_out/ablibs; mkdir -p $O; : > $O/ab.jsonl
L=paper_2005_06193_b200/lib
for rep in 1 2; do for v in "$@"; do
cp $L/variants/$v.so $L/libegfem.so
for c in "cfg4" "cfg4 f32" "cfg3"; do timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"lib\": \"$v\", /" >> $O/ab.jsonl 2>> $O/err; done
done; done
