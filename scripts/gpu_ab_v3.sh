#!/bin/bash
# Kernel-v3 variant A/B (alternating, two repetitions): scripts/ab_time.py per library.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab
mkdir -p $O
for rep in 1 2; do
for L in $LIBS; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done
done
