#!/bin/bash
# ncu of the four k_cell launches (apply, Picard, Newton, fused) with the packed words; fused staged.
cd $GRAFT_REPO_ROOT
O=gpurun_out/words3; mkdir -p $O
EGFEM_CELLS_WORDS=1 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$' -c 4 -o $O/pm -f python scripts/profile_cfg4_jac.py > $O/ncu_pm.log 2>&1
python scripts/ncu_summary.py $O/pm.ncu-rep > $O/pm.txt 2>&1
EGFEM_CELLS_WORDS=0 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_cell$' --launch-skip 3 -c 1 -o $O/st -f python scripts/profile_cfg4_jac.py > $O/ncu_st.log 2>&1
python scripts/ncu_summary.py $O/st.ncu-rep > $O/st.txt 2>&1
ncu -i $O/pm.ncu-rep --page raw --csv > $O/raw_pm.csv 2>/dev/null
ncu -i $O/st.ncu-rep --page raw --csv > $O/raw_st.csv 2>/dev/null
ncu -i $O/pm.ncu-rep --page source --csv --print-source sass --launch-skip 3 > $O/sass_pm_fused.csv 2>/dev/null
python scripts/sass_stalls.py $O/sass_pm_fused.csv 30 > $O/stalls_pm_fused.txt 2>&1
rm -f $O/*.ncu-rep
