#!/bin/bash
# The two arms as the driver runs them (reference first), with wall-clock around each.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2v12; mkdir -p $O
for K in 20 50; do
  s=$(date +%s.%N)
  timeout 900 python bench.py --impl reference --gpus 1 --steps $K --warmup 5 > $O/bench_ref_k$K.json 2> $O/bench_ref_k$K.err
  e=$(date +%s.%N); echo "reference K=$K rc=$? wall_s=$(echo "$e - $s" | bc)" >> $O/ref_wall.log
done
s=$(date +%s.%N)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_k20.json 2> $O/bench_k20.err
e=$(date +%s.%N); echo "ours K=20 rc=$? wall_s=$(echo "$e - $s" | bc)" >> $O/ref_wall.log
