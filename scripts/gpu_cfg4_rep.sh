#!/bin/bash
# Repeat cfg4 bench lines for a list of env settings (A/B with repeats):
#   CFGS="EGFEM_CELLS_PF=0 EGFEM_CELLS_PF=2" REPS=2 ARGS="--dtype f64" scripts/gpu_cfg4_rep.sh
for rep in $(seq 1 ${REPS:-2}); do
  for c in $CFGS; do
    env ${c//,/ } python bench.py --no-cpu-baseline --steps 50 $ARGS > gpurun_out/rep4.json 2> gpurun_out/rep4.err
    python -c "import json; d=json.loads(open('gpurun_out/rep4.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$c', round(d['ms_per_step'],4), 'fused', round(k['apply_jacobian_fused']['ms'],4), 'interp', round(k['interp']['ms'],4), 'apply', round(k['apply']['ms'],4), 'newton', round(k['jacobian_newton']['ms'],4))" || tail -3 gpurun_out/rep4.err
  done
done
