#!/bin/bash
# cfg5 batched-action sweep on the GPU box: parity tests, then bench lines per (P, run, IL, PF).
python -m pytest tests -m gpu -x -q -k "batched" > gpurun_out/t_b.log 2>&1; tail -2 gpurun_out/t_b.log
for P in ${PS:-4}; do for RUN in ${RUNS:-2}; do for IL in ${ILS:-4}; do for PF in ${PFS:-1}; do
  tag=p${P}_r${RUN}_i${IL}_f$PF
  EGFEM_GROUP_STAGED=${STAGED:-0} EGFEM_GROUP_PF=$PF EGFEM_GROUP_IL=$IL EGFEM_GROUP_RUN=$RUN EGFEM_GROUP_P=$P python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b5_$tag.json 2> gpurun_out/b5_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/b5_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['ms_per_step'],4), 'ms fp64', round(d['roofline']['frac'],3), 'hbm', round(d['roofline_hbm']['frac'],3))" || tail -5 gpurun_out/b5_$tag.err
done; done; done; done
