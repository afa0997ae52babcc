#!/bin/bash
# End-to-end NNLS gate at full size (configs 4 and 5) + the full GPU test suite.
cd $GRAFT_REPO_ROOT
timeout 1500 python scripts/e2e_gate.py 5 > gpurun_out/r2_e2e_c5.json 2> gpurun_out/r2_e2e_c5.err
timeout 900 python scripts/e2e_gate.py 4 > gpurun_out/r2_e2e_c4.json 2> gpurun_out/r2_e2e_c4.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_all.log
