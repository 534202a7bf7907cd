#!/bin/bash
# interp occupancy variants (lib/variants/ib*.so) on cfg4 f64 / f32, then the default bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out/abi; mkdir -p $O; : > $O/ab.jsonl
L=paper_2005_06193_b200/lib
cp $L/libegfem.so /tmp/libegfem_default.so
for rep in 1 2; do for v in "$@"; do
cp $L/variants/$v.so $L/libegfem.so
for c in "cfg4" "cfg4 f32"; do timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"lib\": \"$v\", /" >> $O/ab.jsonl 2>> $O/err; done
done; done
cp /tmp/libegfem_default.so $L/libegfem.so
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
