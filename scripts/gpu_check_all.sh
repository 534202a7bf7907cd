#!/bin/bash
# Full check: smoke, pytest -m gpu, default bench line, cell-kernel A/B (words on / off).
cd $GRAFT_REPO_ROOT
O=gpurun_out/all; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
: > $O/ab.jsonl
for wv in 1 0; do for c in "cfg4" "cfg4 f32" "cfg3"; do EGFEM_CELLS_WORDS=$wv timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"words\": $wv, /" >> $O/ab.jsonl 2>> $O/err; done; done
