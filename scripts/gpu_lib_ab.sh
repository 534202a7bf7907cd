#!/bin/bash
# A/B of a variant build (lib/libegfem_exp.so) against lib/libegfem.so: step_sweep base variants
cd $GRAFT_REPO_ROOT
O=gpurun_out/libab; mkdir -p $O; : > $O/a.jsonl; : > $O/b.jsonl
for c in "cfg4 f64" "cfg4 f32" "cfg3 f64"; do timeout 300 python scripts/step_sweep.py $c 30 - >> $O/a.jsonl 2>> $O/err; done
cp paper_2005_06193_b200/lib/libegfem_exp.so paper_2005_06193_b200/lib/libegfem.so
for c in "cfg4 f64" "cfg4 f32" "cfg3 f64"; do timeout 300 python scripts/step_sweep.py $c 30 - >> $O/b.jsonl 2>> $O/err; done
