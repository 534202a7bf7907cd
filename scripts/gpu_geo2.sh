#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/geo3; mkdir -p $O
timeout 600 python scripts/geo_ab.py > $O/geo_ab.json 2> $O/geo_ab.err
timeout 900 python -m pytest tests/test_geo_gpu.py -q --timeout 600 > $O/pytest_geo.log 2>&1; echo "rc=$?" >> $O/pytest_geo.log
