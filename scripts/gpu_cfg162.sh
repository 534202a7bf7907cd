#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/cfg162; mkdir -p $O; : > $O/ab.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "packed_words" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1
for rep in 1 2; do for c in "8,3" "16,2"; do for dt in f64 f32; do
EGFEM_CELLS_CFG=$c timeout 300 python scripts/rows_sweep.py cfg4 $dt | sed "s/^{/{\"G_CPL\": \"$c\", /" >> $O/ab.jsonl 2>> $O/err
done; done; done
