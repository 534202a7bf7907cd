#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/rows5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "row_partition or batched or partition" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python scripts/emulate_cfg5_rows.py 1,2,4,8 20 > $O/emu.jsonl 2> $O/emu.err
