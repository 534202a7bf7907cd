#!/bin/bash
# Repeat cfg5 bench lines for a list of env settings (A/B comparison with repeats):
#   CFGS="EGFEM_GROUP_PF=0 EGFEM_GROUP_PF=2" REPS=3 scripts/gpu_cfg5_rep.sh
for rep in $(seq 1 ${REPS:-2}); do
  for c in $CFGS; do
    env ${c//,/ } python bench.py --config cfg5 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/rep.json 2> gpurun_out/rep.err
    python -c "import json; d=json.loads(open('gpurun_out/rep.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4))" || tail -3 gpurun_out/rep.err
  done
done
