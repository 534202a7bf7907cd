#!/bin/bash
# Packed row words (PM) vs staged slices: parity tests, kernel A/B, bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/words; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "packed_words or kernel_paths or cfg4 or cfg3 or fused" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
: > $O/ab.jsonl
for rep in 1 2; do
for wv in 1 0; do
for c in "cfg4" "cfg4 f32" "cfg3"; do EGFEM_CELLS_WORDS=$wv timeout 300 python scripts/rows_sweep.py $c | sed "s/^{/{\"words\": $wv, /" >> $O/ab.jsonl 2>> $O/err; done
done; done
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
EGFEM_CELLS_WORDS=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_w0.json 2>> $O/bench.err
