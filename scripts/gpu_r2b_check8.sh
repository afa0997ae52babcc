#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ck8
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "column_kernel or batched or config2 or csc or shared_gather" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SRHT_LIB=libcp0.so timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "column_kernel" > $O/pytest_cp0.log 2>&1; echo "rc=$?" >> $O/pytest_cp0.log
