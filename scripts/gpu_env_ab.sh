#!/bin/bash
# A/B of an env switch on the step kernels: gpu_env_ab.sh VAR "v1 v2 ..." [config dtype]
cd $GRAFT_REPO_ROOT
O=gpurun_out/envab; mkdir -p $O; : > $O/ab.jsonl
VAR=$1; VALS=$2; CFG=${3:-cfg4}; DT=${4:-f64}
for v in $VALS; do
  env $VAR=$v timeout 300 python scripts/step_sweep.py $CFG $DT 30 - | sed "s/^/{\"$VAR\": \"$v\", \"r\": /; s/$/}/" >> $O/ab.jsonl 2>> $O/err
done
last=$(echo $VALS | awk '{print $NF}')
env $VAR=$last timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "small or fused or cfg4_full" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
