#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python scripts/nnls_probe.py bpp 2"
$CMD > gpurun_out/bpp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_nnls_bpp_cl -s 1 -c 1 -o gpurun_out/ncubpp $CMD > gpurun_out/ncubpp.log 2>&1
