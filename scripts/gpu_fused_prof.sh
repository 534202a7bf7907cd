#!/bin/bash
# one ncu --set full capture of the cfg4 fp64 fused k_cell launch; raw metrics + per-SASS source table
cd $GRAFT_REPO_ROOT
O=gpurun_out/fp; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cell --launch-skip 3 -c 1 -o $O/fused -f python scripts/profile_cfg4_jac.py > $O/ncu.log 2>&1
ncu -i $O/fused.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/fused.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
ls -la $O
