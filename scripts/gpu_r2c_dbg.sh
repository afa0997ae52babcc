#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_dbg
mkdir -p $O
for L in libsrht.so libprev.so; do
SRHT_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size python scripts/gram_probe.py 4 2 > $O/ncu_$L.txt 2>&1
done
