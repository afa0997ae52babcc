#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sketch_tiles -s 3 -c 1 -o gpurun_out/ncuc3 $CMD > gpurun_out/ncuc3.log 2>&1
