#!/bin/bash
# F2 3D I_2 on the cell-major kernel (G = 32 lanes per row): parity + bench vs the row-group path.
cd $GRAFT_REPO_ROOT
O=gpurun_out/f2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "plap3d or cell or cfg4 or quad or newton" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in plap3d_i2 quadratic_i4 biochem_i2 plap_i1 cfg4; do
  EGFEM_DEBUG= timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  EGFEM_PATH=rows timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_rows.json 2> $O/bench_${c}_rows.err
done
