#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/sym2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "batched or cfg5 or group or kernel_paths" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
: > $O/b.txt
for rep in 1 2; do for B in 256 128 64 32; do
timeout 900 python bench.py --config cfg5 --batch $B --no-cpu-baseline > $O/b_$B.json 2> $O/b_$B.err
python -c "import json; d=json.loads(open('$O/b_$B.json').read().strip().splitlines()[-1]); print($B, round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))" >> $O/b.txt 2>&1 || tail -3 $O/b_$B.err >> $O/b.txt
done; done
