#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/rk; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_step_gpu.py -q -k "packed_words or w_null or cfg4 or cfg3 or fused or kernel_paths" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
bash scripts/gpu_ab_libs.sh rk dg0
