#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python scripts/gram_probe.py 4 2"
$CMD > gpurun_out/gram_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gram_mma -s 1 -c 1 -o gpurun_out/ncugram $CMD > gpurun_out/ncugram.log 2>&1
