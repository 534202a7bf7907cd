#!/bin/bash
# cfg5 batched-action sweep on the GPU box: parity tests, then bench lines per (P, run).
python -m pytest tests -m gpu -x -q -k "batched" > gpurun_out/t_b.log 2>&1; tail -2 gpurun_out/t_b.log
for P in ${PS:-2 4}; do for RUN in ${RUNS:-4}; do
  EGFEM_GROUP_RUN=$RUN EGFEM_GROUP_P=$P python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b5_p${P}_r$RUN.json 2> gpurun_out/b5_p${P}_r$RUN.err
  python -c "import json; d=json.loads(open('gpurun_out/b5_p${P}_r$RUN.json').read().strip().splitlines()[-1]); print('P=$P run=$RUN', round(d['ms_per_step'],4), 'ms fp64', round(d['roofline']['frac'],3), 'hbm', round(d['roofline_hbm']['frac'],3), 'build', round(d['build_s'],1))" || tail -5 gpurun_out/b5_p${P}_r$RUN.err
done; done
