#!/bin/bash
# Consumer pacing: __nanosleep between gather chunks (V3_CSLEEP ns) vs none.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab12
mkdir -p $O
for rep in 1 2; do for L in libsrht.so libcs50.so libcs150.so libcs300.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done; done
