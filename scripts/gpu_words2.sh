#!/bin/bash
# Packed row words: bitwise test, carveout A/B, ncu of the fused kernel with and without words.
cd $GRAFT_REPO_ROOT
O=gpurun_out/words2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "packed_words" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
: > $O/ab.jsonl
for rep in 1 2; do
for v in "1 -1" "0 -1" "1 0" "1 28" "1 45" "1 58" "0 58"; do set -- $v
EGFEM_CELLS_WORDS=$1 EGFEM_CELLS_CARVE=$2 timeout 300 python scripts/rows_sweep.py cfg4 | sed "s/^{/{\"words\": $1, \"carve\": $2, /" >> $O/ab.jsonl 2>> $O/err
done; done
for wv in 1 0; do
EGFEM_CELLS_WORDS=$wv timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cell --launch-skip 3 -c 1 -o $O/fused_w$wv -f python scripts/profile_cfg4_jac.py > $O/ncu_w$wv.log 2>&1
python scripts/ncu_summary.py $O/fused_w$wv.ncu-rep > $O/fused_w$wv.txt 2>&1
ncu -i $O/fused_w$wv.ncu-rep --page raw --csv > $O/raw_w$wv.csv 2>/dev/null
ncu -i $O/fused_w$wv.ncu-rep --page source --csv --print-source sass > $O/sass_w$wv.csv 2>/dev/null
python scripts/sass_stalls.py $O/sass_w$wv.csv 30 > $O/stalls_w$wv.txt 2>&1
rm -f $O/fused_w$wv.ncu-rep
done
ls -la $O
