#!/bin/bash
# cfg5 with the symmetrized patterns: P / register cap / interleave / run sweep (bench lines)
cd $GRAFT_REPO_ROOT
O=gpurun_out/symsw; mkdir -p $O; : > $O/sweep.txt
IFS=";" read -ra VV <<< "$VARS"; for v in "${VV[@]}"; do set -- $v
  tag=p$1_m$2_i$3_r$4
  EGFEM_GROUP_P=$1 EGFEM_GROUP_MAXREG=$2 EGFEM_GROUP_IL=$3 EGFEM_GROUP_RUN=$4 timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > $O/b_$tag.json 2> $O/b_$tag.err
  python -c "import json; d=json.loads(open('$O/b_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))" >> $O/sweep.txt 2>&1 || tail -3 $O/b_$tag.err >> $O/sweep.txt
done
