#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/wnull; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_step_gpu.py -q -k "w_null or packed_words or step or fused" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
