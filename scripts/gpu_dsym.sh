#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/dsym; mkdir -p $O; : > $O/b.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "identity_newton or cfg1 or cfg2 or dense or fused or bench_line" --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for rep in 1 2; do for sy in 1 0; do for c in cfg2 cfg1; do
EGFEM_DENSE_SYM=$sy timeout 600 python bench.py --config $c --no-cpu-baseline > $O/b_${sy}_$c.json 2> $O/b_${sy}_$c.err
python -c "import json; d=json.loads(open('$O/b_${sy}_$c.json').read().strip().splitlines()[-1]); print('sym', $sy, '$c', round(d['ms_per_step'],5), 'frac', round(d['roofline']['frac'],3), round(d['roofline']['time_ms'],5))" >> $O/b.txt 2>&1 || tail -3 $O/b_${sy}_$c.err >> $O/b.txt
done; done; done
timeout 600 python bench.py --config cfg2 > $O/b_cfg2_full.json 2> $O/b_cfg2_full.err
