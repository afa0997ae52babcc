#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python scripts/fp64_mode_time.py"
$CMD > gpurun_out/ncu64_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma64 -s 1 -c 1 -o gpurun_out/ncu64 $CMD > gpurun_out/ncu64.log 2>&1
