#!/bin/bash
# Round-2 check: GPU tests, smoke, a short default bench (incl. the all-cores cpu_baseline).
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench.log
