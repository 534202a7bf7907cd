#!/bin/bash
# fp64 geometry-class interp at 5 / 6 / 8 CTAs per SM (lib variants geo6 / geo8) vs the gathering kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/geominb; mkdir -p $O; : > $O/ab.jsonl
L=paper_2005_06193_b200/lib
cp $L/libegfem.so /tmp/libegfem_default.so
cp /tmp/libegfem_default.so $L/variants/geo1.so
for v in geo1 geo6 geo8; do
  cp $L/variants/$v.so $L/libegfem.so
  GEO_F64=1 timeout 600 python scripts/geo_ab.py | sed "s/^{/{\"lib\": \"$v\", /" >> $O/ab.jsonl 2>> $O/err
done
cp /tmp/libegfem_default.so $L/libegfem.so
