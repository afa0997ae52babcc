#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ck7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "column_kernel or batched or config2 or csc or shared_gather" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2 3; do timeout 300 python scripts/stress_v3.py 150 >> $O/stress.log 2>&1; echo "rc=$?" >> $O/stress.log; done
