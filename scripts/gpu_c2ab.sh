#!/bin/bash
# Config-2 A/B of the whole-column kernel build variants (bench line per variant).
cd $GRAFT_REPO_ROOT
for L in $LIBS; do
  SRHT_LIB=$L timeout 300 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/c2_$L.json 2>/dev/null
done
