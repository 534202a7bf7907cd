#!/bin/bash
# symmetrized cfg5 with relabeled (descending) stencil order: lazy W loads on / off; parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/sym3; mkdir -p $O; : > $O/b.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "batched or cfg5 or group" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for rep in 1 2; do for lz in 1 0; do for B in 256 128; do
EGFEM_GROUP_SYM_LAZY=$lz timeout 900 python bench.py --config cfg5 --batch $B --no-cpu-baseline > $O/b_${lz}_$B.json 2> $O/b_${lz}_$B.err
python -c "import json; d=json.loads(open('$O/b_${lz}_$B.json').read().strip().splitlines()[-1]); print('lazy', $lz, $B, round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))" >> $O/b.txt 2>&1 || tail -3 $O/b_${lz}_$B.err >> $O/b.txt
done; done; done
