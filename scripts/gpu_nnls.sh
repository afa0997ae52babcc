#!/bin/bash
# NNLS solvers: parity tests, then Algorithm 1 stage timings (configs 4 and 2).
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sketch.py -x -q -k "nnls" > gpurun_out/nn_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nn_pytest.log
timeout 600 python scripts/pipeline_bench.py 4 > gpurun_out/pipe4.json 2>&1
timeout 600 python scripts/pipeline_bench.py 2 > gpurun_out/pipe2.json 2>&1
