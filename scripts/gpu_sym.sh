#!/bin/bash
# cfg5 symmetrized compiled groups (U == W): parity tests, bench with / without
cd $GRAFT_REPO_ROOT
O=gpurun_out/sym; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "batched or cfg5 or group or kernel_paths" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for rep in 1 2; do
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_sym$rep.json 2> $O/bench_sym$rep.err
EGFEM_GROUP_SYM=0 timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_nosym$rep.json 2> $O/bench_nosym$rep.err
done
